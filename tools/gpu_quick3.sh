python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not config5" 2>&1 | tail -2
for i in 1 2; do
  SF_DEBUG_SKIP=0 timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us', d['device_flags'])"
done

