mkdir -p gpurun_out
python bench.py --config 3 --steps 20 --warmup 3 --mcmc-every 100 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo rc=$?
tail -5 gpurun_out/bench_c3.err
