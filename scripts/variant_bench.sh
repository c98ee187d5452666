#!/bin/bash
# Bench the default library and every variants/lib_*.so (tuning experiments,
# built with build.build(defines=..., out=...)): config-1 value and the live
# duration of one kernel per run (KERN, default raster_bwd_kernel).
for lib in default variants/lib_*.so; do
  if [ "$lib" = default ]; then unset CGS_LIB_PATH; else export CGS_LIB_PATH=$PWD/$lib; fi
  for k in ${KERNS:-raster_bwd_kernel}; do
    timeout 300 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} --profile-kernel $k 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(f\"{'$lib':28s} {d['value']:8.1f} it/s  p50 {d['step_ms']['p50']:.3f} ms  {r['kernel']} {1000*r['avg_launch_ms']:.1f} us\")"
  done
done
