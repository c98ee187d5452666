#!/bin/bash
# Round-2 final evidence refresh (same steps as gpu_evidence_r2.sh plus
# configs 2/4 lines, config-3/4 launch lists, config-4 live list and the
# config-3 front-end capture).  Every ncu command runs after the same
# command exited 0 without ncu.  Outputs under gpurun_out/ev2/.
D=gpurun_out/ev2; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $D/bench_config1.json 2> $D/bench_config1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $D/reference_arm_config1.json 2> $D/reference_arm.err; echo "ref rc=$?"
timeout 900 python bench.py --config 2 --steps 50 --mcmc-every 100 --no-cpu-baseline > $D/bench_config2.json 2> $D/bench_config2.err; echo "c2 rc=$?"
timeout 1200 python bench.py --config 3 --steps 200 --warmup 5 --mcmc-every 100 --no-cpu-baseline > $D/bench_config3_mcmc.json 2> $D/bench_config3.err; echo "c3 rc=$?"
timeout 1200 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > $D/bench_config4.json 2> $D/bench_config4.err; echo "c4 rc=$?"
bash scripts/live_all.sh > $D/live_kernels_config1.txt 2>&1
BENCH_ARGS="--config 3" bash scripts/live_all.sh > $D/live_kernels_config3.txt 2>&1
timeout 600 python scripts/live_c4.py 1 > $D/live_kernels_config4.txt 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $D/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 160 --csv \
    --log-file $D/launches_config1.csv $CMD > $D/ncu_l.log 2>&1; echo "ncu launches rc=$?"
C3="python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --mcmc-every 1000"
$C3 > $D/c3_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 150 --csv \
    --log-file $D/launches_config3.csv $C3 > $D/ncu_c3.log 2>&1; echo "ncu c3 launches rc=$?"
C4="python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$C4 > $D/c4_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 120 --csv \
    --log-file $D/launches_config4.csv $C4 > $D/ncu_c4.log 2>&1; echo "ncu c4 launches rc=$?"
$CMD > $D/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"raster_fwd_kernel|raster_bwd_kernel|refine_kernel" \
    -s 12 -c 4 -o $D/full_raster $CMD > $D/ncu_f.log 2>&1; echo "ncu full rc=$?"
C3P="python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --mcmc-every 1000"
$C3P > $D/c3p_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"project_kernel|onesweep_kernel|scan_kernel|tile_scatter_kernel" -s 24 -c 8 \
    -o $D/full_front_c3 $C3P > $D/ncu_front.log 2>&1; echo "ncu front rc=$?"
ls -la $D
