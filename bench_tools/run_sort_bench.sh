#!/bin/bash
# Build and run the sort microbenchmark for several items:lookback variants.
mkdir -p gpurun_out
for cfg in ${CFGS:-16:32}; do
  it=${cfg%%:*}; lb=${cfg##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DCGS_SORT_ITEMS=$it -DCGS_SORT_LOOKBACK=$lb bench_tools/sort_bench.cu -o /tmp/sb_$it_$lb || exit 1
  echo "== items=$it lookback=$lb"
  timeout 120 /tmp/sb_$it_$lb
done
