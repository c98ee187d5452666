#!/bin/bash
# Config-4 render-only: live per-kernel times and the bench line, default
# library and every variants/lib_*.so.
D=gpurun_out/c4; mkdir -p $D
for lib in default variants/lib_*.so; do
  if [ "$lib" = default ]; then unset CGS_LIB_PATH; else export CGS_LIB_PATH=$PWD/$lib; fi
  echo "== $lib"
  timeout 600 python scripts/live_c4.py 1 2>&1 | tail -12
  timeout 600 python bench.py --config 4 --steps ${C4_STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | cut -c1-200
done
