# Iteration: build, smoke, the GPU parity suite, per-kernel times and the default bench.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > gpurun_out/gputest_it.log; cat gpurun_out/gputest_it.log
timeout 300 python tools/ktime.py > gpurun_out/ktime.json 2>&1; cat gpurun_out/ktime.json
timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_it.json
python -c "import json; d=json.load(open('gpurun_out/bench_it.json')); print('BENCH', d['value'], d['ms_per_step']*1e3)"
