#!/bin/bash
# Closing bench lines on the final tree (configs 1-3 and the reference arm;
# config 4 and the ncu captures are unchanged since gpu_evidence_r2c.sh / r2b.sh
# except for the memset nodes), live config-1 list and launch list.
D=gpurun_out/ev4; mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $D/bench_config1.json 2> $D/bench_config1.err; echo "bench rc=$?"
timeout 900 python bench.py --config 2 --steps 50 --mcmc-every 100 --no-cpu-baseline > $D/bench_config2.json 2> $D/bench_config2.err; echo "c2 rc=$?"
timeout 1200 python bench.py --config 3 --steps 200 --warmup 5 --mcmc-every 100 --no-cpu-baseline > $D/bench_config3_mcmc.json 2> $D/bench_config3.err; echo "c3 rc=$?"
timeout 1200 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > $D/bench_config4.json 2> $D/bench_config4.err; echo "c4 rc=$?"
bash scripts/live_all.sh > $D/live_kernels_config1.txt 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $D/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 160 --csv \
    --log-file $D/launches_config1.csv $CMD > $D/ncu_l.log 2>&1; echo "ncu launches rc=$?"
