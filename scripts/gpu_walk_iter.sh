#!/bin/bash
D=gpurun_out/walk; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -q -x -k "backward or giants or deep_stack or config1_full or strip or gradcheck or train_loop or staged or knife" > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest.log
KERNS="splat_reduce_kernel" bash scripts/variant_live.sh
BENCH_ARGS="--config 3" KERNS="splat_reduce_kernel" bash scripts/variant_live.sh
