# edge-CTA timing: current code (all, no column passes, no row passes), then the previous commit
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for sk in 256 320 384; do echo "== skip $sk"; SF_DEBUG_SKIP=$sk timeout 600 python bench.py --steps 16 --warmup 8 --no-cpu-baseline 2>&1 | grep SFTIME | tail -1; done
cp tools/old_sf_fused.cu paper_2406_18031_b200/csrc/sf_fused.cu
python paper_2406_18031_b200/build.py --force > /dev/null 2>&1
echo "== old"; SF_DEBUG_SKIP=0 timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us')"
for sk in 256 320 384; do echo "== old skip $sk"; SF_DEBUG_SKIP=$sk timeout 600 python bench.py --steps 16 --warmup 8 --no-cpu-baseline 2>&1 | grep SFTIME | tail -1; done
