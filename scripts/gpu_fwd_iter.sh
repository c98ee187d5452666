#!/bin/bash
# raster_fwd iteration: GPU parity tests, then live times of the default
# library and every variants/lib_*.so at configs 1, 3 (and 4 with C4=1).
D=gpurun_out/fwd; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest.log
KERNS="${KERNS:-raster_fwd_kernel}" bash scripts/variant_live.sh
BENCH_ARGS="--config 3" KERNS="${KERNS:-raster_fwd_kernel}" bash scripts/variant_live.sh
