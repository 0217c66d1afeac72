python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not config5" 2>&1 | tail -2
for cfg in 0 1; do
for sk in 0 2; do
  echo -n "cfg=$cfg skip=$sk "; SF_FUSED_CFG=$cfg SF_DEBUG_SKIP=$sk timeout 600 python bench.py --steps 1000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us')"
done; done
