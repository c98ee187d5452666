#!/bin/bash
D=gpurun_out/scan; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest.log
KERNS="scan_kernel project_kernel" bash scripts/variant_live.sh
BENCH_ARGS="--config 3" KERNS="scan_kernel project_kernel" bash scripts/variant_live.sh
for lib in default variants/lib_*.so; do
  if [ "$lib" = default ]; then unset CGS_LIB_PATH; else export CGS_LIB_PATH=$PWD/$lib; fi
  echo "== $lib"; timeout 600 python scripts/live_c4.py 1 2>&1 | tail -10
done
