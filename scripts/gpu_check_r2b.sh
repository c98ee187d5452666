#!/bin/bash
# Re-entry check: GPU tests, smoke, config-1 bench and config-3 MCMC bench on the current tree.
D=gpurun_out/chk; mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $D/bench_config1.json 2> $D/bench_config1.err; echo "bench rc=$?"; cat $D/bench_config1.json | cut -c1-300
timeout 1200 python bench.py --config 3 --steps 200 --warmup 5 --mcmc-every 100 --no-cpu-baseline > $D/bench_config3_mcmc.json 2> $D/bench_config3.err; echo "c3 rc=$?"; cut -c1-300 $D/bench_config3_mcmc.json
