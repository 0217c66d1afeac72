# Launch overhead (empty kernels via SF_DEBUG_SKIP=32) vs real kernel times; transport shapes A/B.
set -x
SF_BUILD_DEBUG=1 python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SF_DEBUG_SKIP=32 timeout 300 python tools/ktime2.py
timeout 300 python tools/ktime2.py
for cfg in 0 1 3 4; do
  SF_TRANS_CFG=$cfg SF_DEBUG_SKIP=8192 timeout 300 python tools/ktime.py --frames 12 --ring 8 2>&1 | grep 'SFPROF trans' | tail -2
done
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for cfg in 0 1 3 4; do
  SF_TRANS_CFG=$cfg timeout 300 python tools/ktime2.py
  SF_TRANS_CFG=$cfg timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_it9_$cfg.json
  python -c "import json; d=json.load(open('gpurun_out/bench_it9_$cfg.json')); print('BENCH cfg $cfg', d['value'], d['ms_per_step']*1e3)"
done
