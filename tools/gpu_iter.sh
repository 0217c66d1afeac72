# One optimisation iteration on the GPU: all GPU tests, bench x2 (+ H = 2), per-phase clocks.
set -x
[ -x tools/rcp/check_rcp ] && timeout 300 tools/rcp/check_rcp
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['ms_per_step']*1000,2), 'us', round(d['value']), 'Hz')"; done
timeout 600 python bench.py --levels 2 --steps 1000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench H=2', round(d['ms_per_step']*1000,2), 'us', round(d['value']), 'Hz')"
SF_BUILD_DEBUG=1 python paper_2406_18031_b200/build.py --force > /dev/null
SF_DEBUG_SKIP=256 timeout 600 python bench.py --steps 64 --warmup 8 --no-cpu-baseline 2>&1 | grep SFTIME | tail -4
SF_DEBUG_SKIP=2048 timeout 600 python bench.py --steps 24 --warmup 8 --ring 8 --no-cpu-baseline 2>&1 | grep SFGT > gpurun_out/gt_iter.txt
python tools/gt_classes.py gpurun_out/gt_iter.txt
python paper_2406_18031_b200/build.py --force > /dev/null
