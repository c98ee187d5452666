#!/bin/bash
# ncu --set full captures of several kernels (one each) of the bench step.
mkdir -p gpurun_out
TAG=${TAG:-m}
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1; echo "plain rc=$?"
for K in $KERNS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-4} -c 1 -o gpurun_out/full_${TAG}_${K//[^a-zA-Z0-9_]/} $CMD > gpurun_out/ncu_${TAG}_${K//[^a-zA-Z0-9_]/}.log 2>&1; echo "ncu $K rc=$?"
done
