#!/bin/bash
# Full ncu captures of the loss, SGLD and pair-emission kernels at config 3.
mkdir -p gpurun_out
C3="python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --mcmc-every 1000"
$C3 > gpurun_out/misc_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"ssim_stats_kernel|ssim_grad_kernel|sgld_kernel|emit_pairs_kernel|gauss_write_kernel" -s 15 -c 5 \
    -o gpurun_out/r2_misc_c3 -f $C3 > gpurun_out/ncu_misc.log 2>&1
tail -c 300 gpurun_out/ncu_misc.log
