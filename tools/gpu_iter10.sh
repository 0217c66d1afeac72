# Max shared carve-out on every tiled kernel: launch overhead of empty kernels, kernel times, bench.
set -x
SF_BUILD_DEBUG=1 python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SF_DEBUG_SKIP=32 timeout 300 python tools/ktime2.py
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python tools/ktime2.py
timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_it10.json
python -c "import json; d=json.load(open('gpurun_out/bench_it10.json')); print('BENCH', d['value'], d['ms_per_step']*1e3)"
timeout 300 python bench.py --levels 2 --steps 1000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_it10_h2.json
python -c "import json; d=json.load(open('gpurun_out/bench_it10_h2.json')); print('BENCH H2', d['value'], d['ms_per_step']*1e3)"
