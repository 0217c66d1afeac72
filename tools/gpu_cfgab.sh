# A/B of the fused kernel's region shapes (SF_FUSED_CFG): parity tests + bench + phase clocks per shape
set +e
python paper_2406_18031_b200/build.py --force > /dev/null
for cfg in "$@"; do
  echo "=== cfg $cfg"
  SF_FUSED_CFG=$cfg timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
  for i in 1 2; do SF_FUSED_CFG=$cfg timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['ms_per_step']*1000,2), 'us', round(d['value']), 'Hz')"; done
done
SF_BUILD_DEBUG=1 python paper_2406_18031_b200/build.py --force > /dev/null
for cfg in "$@"; do
  echo "=== phases cfg $cfg"
  SF_FUSED_CFG=$cfg SF_DEBUG_SKIP=256 timeout 600 python bench.py --steps 64 --warmup 8 --no-cpu-baseline 2>&1 | grep SFTIME | tail -4
done
python paper_2406_18031_b200/build.py --force > /dev/null
