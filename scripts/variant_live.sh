#!/bin/bash
# Live per-kernel launch durations (graphs off, CUDA events on the launch
# stream) for the default library and every variants/lib_*.so.
for lib in default variants/lib_*.so; do
  if [ "$lib" = default ]; then unset CGS_LIB_PATH; else export CGS_LIB_PATH=$PWD/$lib; fi
  for k in ${KERNS:-raster_fwd_kernel raster_bwd_kernel}; do
    timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-graphs ${BENCH_ARGS} --profile-kernel $k 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(f\"{'$lib':28s} {r['kernel']:24s} {1000*r['avg_launch_ms']:8.1f} us x {r['launches']/d['steps']:.1f}/step  (step {d['ms_per_step']:.3f} ms)\")"
  done
done
