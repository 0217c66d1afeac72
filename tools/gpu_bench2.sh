python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python bench.py --levels 2 --steps 1000 --warmup 40 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_h2.json
cat gpurun_out/bench_h2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), 'Hz', round(d['ms_per_step']*1000,2), 'us', d['device_flags'], d['gpu_launches']/d['steps'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches_h2.csv python bench.py --levels 2 --steps 16 --warmup 8 --ring 8 --no-cpu-baseline > /dev/null 2>&1
