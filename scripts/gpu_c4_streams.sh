#!/bin/bash
D=gpurun_out/c4s; mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_output.py -m gpu -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest.log
for S in 1 2 3 4; do
  timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --render-streams $S 2>$D/err_$S.log | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('streams $S', round(d['value'],1), 'Mpix/s e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
