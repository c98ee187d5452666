#!/bin/bash
# Live per-kernel launch durations of one bench configuration (graphs off,
# CUDA events on the launch stream, one kernel profiled per run).
# usage: BENCH_ARGS="--config 3" bash scripts/live_all.sh
KS="project_kernel onesweep_kernel depth_tie_fix_kernel scan_kernel emit_pairs_kernel tile_count_kernel tile_scatter_kernel raster_fwd_kernel
refine_fwd_kernel ssim_stats_kernel ssim_grad_kernel raster_bwd_kernel refine_bwd_kernel splat_reduce_kernel
pull_back_kernel gauss_write_kernel sh_code_reduce_kernel sr_code_reduce_kernel sr_precompute_kernel sgld_kernel"
for k in $KS; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-graphs ${BENCH_ARGS} --profile-kernel $k 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
n=r['launches']/d['steps']; us=1000*r['avg_launch_ms']
print(f\"{r['kernel']:24s} {us:9.1f} us x {n:4.1f}/step = {us*n:8.1f} us/step  (step {1000*d['ms_per_step']:.0f} us)\")"
done
