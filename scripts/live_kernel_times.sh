#!/bin/bash
# Live (not under ncu) per-kernel average launch durations at config 1: one
# bench run per kernel with --profile-kernel (CUDA events on the launch
# stream), graphs off so every launch is bracketed.
mkdir -p gpurun_out
for k in ${KERNELS:-raster_bwd_kernel raster_fwd_kernel project_kernel emit_pairs_kernel onesweep_kernel scan_kernel pull_back_kernel splat_reduce_kernel sh_code_reduce_kernel sr_code_reduce_kernel ssim_stats_kernel ssim_grad_kernel sgld_kernel}; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-graphs ${BENCH_ARGS} --profile-kernel $k 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(f\"{r['kernel']:28s} {1000*r['avg_launch_ms']:8.1f} us x {r['launches']/d['steps']:.1f}/step  (step {d['ms_per_step']:.3f} ms)\")"
done
