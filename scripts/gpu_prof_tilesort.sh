#!/bin/bash
# Full ncu captures of the counting tile sort kernels at config 3.
mkdir -p gpurun_out
C3="python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --mcmc-every 1000"
$C3 > gpurun_out/ts_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"tile_count_kernel|tile_scatter_kernel|scan_kernel" -s 6 -c 4 \
    -o gpurun_out/ts_c3 -f $C3 > gpurun_out/ncu_ts.log 2>&1
tail -c 400 gpurun_out/ts_plain.log; tail -c 400 gpurun_out/ncu_ts.log
