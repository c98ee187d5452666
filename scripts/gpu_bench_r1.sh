mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo rc=$?
tail -3 gpurun_out/bench7.err
python scripts/host_profile.py --graphs 2>&1 | grep -E "span|raster_|tile_depth|pull_back|sh_code" | cut -c1-150
