python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SF_DEBUG_SKIP=0 timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us', d['device_flags'])"
SF_BUILD_DEBUG=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SF_DEBUG_SKIP=256 timeout 600 python bench.py --steps 24 --warmup 8 --no-cpu-baseline 2>&1 | grep SFTIME > gpurun_out/sftime.txt
python - <<'PY'
import collections
d=collections.defaultdict(list)
for l in open('gpurun_out/sftime.txt'):
    k,v=l.split(':',1); d[k].append(v.strip())
for k in sorted(d): print(k, len(d[k]), '|', d[k][len(d[k])//2], '|', d[k][-1])
PY
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1  # back to the production build
