#!/bin/bash
# Round-2 profiles: live kernel times, the ncu launch list and one ncu --set
# full capture of the raster kernels at config 1 (each ncu command only after
# the same command exited 0 without ncu).
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 160 --csv \
    --log-file gpurun_out/r2_launches_config1.csv $CMD > gpurun_out/ncu_l.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"raster_fwd_kernel|raster_bwd_kernel|refine_kernel" \
    -s 12 -c 4 -o gpurun_out/r2_full_raster $CMD > gpurun_out/ncu_f.log 2>&1
ls -la gpurun_out/r2_full_raster* gpurun_out/r2_launches_config1.csv
