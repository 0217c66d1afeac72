# H = 2 pyramid: GPU tests (pyramid, async, map, eval) and the bench (with and without mapping)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_async.py tests/test_gpu_map.py tests/test_gpu_eval.py -x -q 2>&1 | tail -1
for i in 1 2; do timeout 600 python bench.py --levels 2 --steps 1000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench H=2', round(d['ms_per_step']*1000,2), 'us', round(d['value']), 'Hz')"; done
timeout 600 python bench.py --levels 2 --map --steps 1000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench H=2 map', round(d['ms_per_step']*1000,2), 'us', round(d['value']), 'Hz')"
