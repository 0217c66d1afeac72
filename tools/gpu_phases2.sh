python -c "import __graft_entry__ as g; g.build()"
for sk in 0 512 1024 1536 2; do
  echo -n "skip=$sk "; SF_DEBUG_SKIP=$sk timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us')"
done
SF_DEBUG_SKIP=768 timeout 600 python bench.py --steps 64 --warmup 8 --no-cpu-baseline 2>&1 | grep SFTIME | tail -2
