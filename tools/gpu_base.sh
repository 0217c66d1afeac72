# Round-2 baseline: GPU tests, default bench, launch list of the default bench.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/gputest.log
cat gpurun_out/gputest.log
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json
cat gpurun_out/bench_default.json
timeout 600 python bench.py --steps 20 --warmup 5 2>&1 | tail -1 > gpurun_out/bench_s20.json
cat gpurun_out/bench_s20.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
