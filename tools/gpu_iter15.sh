# Transport regions flush with the grid border (rows: run-end replicate; columns: COLFIX).
set -x
SF_BUILD_DEBUG=1 python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SF_DEBUG_SKIP=8192 timeout 300 python tools/ktime.py --frames 12 --ring 8 2>&1 | grep 'SFPROF trans' | tail -2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_it15.json
python -c "import json; d=json.load(open('gpurun_out/bench_it15.json')); print('BENCH', d['value'], d['ms_per_step']*1e3)"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
