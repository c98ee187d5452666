#!/bin/bash
# Full ncu captures of the per-splat front end at config 3 (projection, depth
# / tile onesweep passes, pair-offset scan), after the same command exited 0.
mkdir -p gpurun_out
C3="python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --mcmc-every 1000"
$C3 > gpurun_out/proj_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"project_kernel|onesweep_kernel|scan_kernel|emit_pairs_kernel" -s 24 -c 8 \
    -o gpurun_out/r2_front_c3 -f $C3 > gpurun_out/ncu_front.log 2>&1
tail -c 400 gpurun_out/proj_plain.log; tail -c 400 gpurun_out/ncu_front.log
