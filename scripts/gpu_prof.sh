mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain8.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"raster_" -s 4 -c 2 -o gpurun_out/prof_r1f $CMD > gpurun_out/ncu8.log 2>&1; echo ncu=$?
