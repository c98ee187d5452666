#!/bin/bash
# ncu --set full of the per-splat gradient kernels at config 1 (after the
# same command exited 0 without ncu).
D=gpurun_out/red; mkdir -p $D
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $D/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"splat_reduce_kernel|pull_back_kernel|sh_code_reduce|sr_code_reduce|gauss_write|emit_pairs_kernel|tile_scatter" -s 20 -c 7 \
    -o $D/full_reduce $CMD > $D/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $D/ncu.log
