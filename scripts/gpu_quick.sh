#!/bin/bash
# GPU tests + config-1 bench line (no CPU baseline) on the current tree.
D=gpurun_out/quick; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $D/bench1.json 2>$D/bench1.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$D/bench1.json').read().strip().splitlines()[-1]); print(d['value'], d['step_ms'], d['e2e']['value'], d['clocks']['sm_mhz'], d['gpu_launches']/d['steps'])"
