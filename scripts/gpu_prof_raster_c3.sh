#!/bin/bash
# Full ncu captures of the raster kernels at config 3 (after the same command exited 0).
mkdir -p gpurun_out
C3="python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --mcmc-every 1000"
$C3 > gpurun_out/rc3_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"raster_fwd_kernel|raster_bwd_kernel|refine_kernel" -s 12 -c 4 \
    -o gpurun_out/r2_raster_c3 -f $C3 > gpurun_out/ncu_rc3.log 2>&1
tail -c 300 gpurun_out/ncu_rc3.log
