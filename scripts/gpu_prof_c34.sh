#!/bin/bash
# Round-2 launch lists at configs 3 and 4 (each ncu run after the same
# command exited 0 without ncu).
mkdir -p gpurun_out
C3="python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --mcmc-every 1000"
C4="python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --views-per-frame 16"
$C3 > gpurun_out/c3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 150 --csv \
    --log-file gpurun_out/r2_launches_config3.csv $C3 > gpurun_out/ncu_c3.log 2>&1
$C4 > gpurun_out/c4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 120 --csv \
    --log-file gpurun_out/r2_launches_config4.csv $C4 > gpurun_out/ncu_c4.log 2>&1
tail -c 600 gpurun_out/c3_plain.log; tail -c 600 gpurun_out/c4_plain.log
