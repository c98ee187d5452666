#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include bench_tools/sort_bench.cu -o /tmp/sb || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KERN:-onesweep} -s ${SKIP:-4} -c 1 -o gpurun_out/full_sb${TAG} /tmp/sb ${CASE:-5} > gpurun_out/ncu_sb.log 2>&1; echo rc=$?
