python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for c in 3 4 5; do
  timeout 1200 python bench.py --config $c --steps 40 --warmup 8 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c$c.json
  python -c "import json; d=json.load(open('gpurun_out/bench_c$c.json')); print($c, round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,1), 'us', d['device_flags'], d['config'].get('workload'))"
done
