#!/bin/bash
# raster_bwd iteration: parity tests of the backward, then live times of the
# default library and every variants/lib_*.so at configs 1 and 3.
timeout 900 python -m pytest tests -m gpu -q -x -k "backward or giants or deep_stack or config1_full or strip or gradcheck or train_loop or staged" 2>&1 | tail -3
KERNS="raster_bwd_kernel" bash scripts/variant_live.sh
BENCH_ARGS="--config 3" KERNS="raster_bwd_kernel" bash scripts/variant_live.sh
