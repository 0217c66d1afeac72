# One optimisation iteration on the GPU: parity (fused kernel tests), bench, per-phase clocks.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['ms_per_step']*1000,2), 'us', round(d['value']), 'Hz')"; done
SF_BUILD_DEBUG=1 python paper_2406_18031_b200/build.py --force > /dev/null
SF_DEBUG_SKIP=256 timeout 600 python bench.py --steps 64 --warmup 8 --no-cpu-baseline 2>&1 | grep SFTIME | tail -4
python paper_2406_18031_b200/build.py --force > /dev/null
