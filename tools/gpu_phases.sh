# phase timing experiment (results are wrong with SF_DEBUG_SKIP; timing only)
python -c "import __graft_entry__ as g; g.build()"
for sk in 0 2 66 130 194; do
  echo -n "skip=$sk "; SF_DEBUG_SKIP=$sk timeout 600 python bench.py --steps 1000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us')"
done
