#!/bin/bash
# Counting tile sort check: parity tests touching tile lists, live kernel times, config 1/4 bench.
D=gpurun_out/cs; mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest_gpu.log
timeout 300 python scripts/live_c4.py 1 > $D/live_c4.txt 2>&1; cat $D/live_c4.txt
for k in onesweep_kernel scan_kernel tile_count_kernel tile_scatter_kernel emit_pairs_kernel; do
 for cfg in 1 3; do
  timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-graphs --profile-kernel $k 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
n=r['launches']/d['steps']; us=1000*r['avg_launch_ms']
print(f\"cfg $cfg {r['kernel']:24s} {us:9.1f} us x {n:4.1f}/step = {us*n:8.1f} us/step  (step {1000*d['ms_per_step']:.0f} us)\")"
 done
done
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $D/bench_c1.json 2>&1; cut -c1-200 $D/bench_c1.json
timeout 900 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > $D/bench_c4.json 2>&1; cut -c1-200 $D/bench_c4.json
