# Phase profile (debug build, clock64 per phase, CTAs (0,0) and (3,3)) of k_trans and k_upd.
set -x
SF_BUILD_DEBUG=1 python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SF_DEBUG_SKIP=8192 timeout 300 python tools/ktime.py --frames 30 --ring 8 > gpurun_out/phases.log 2>&1
grep SFPROF gpurun_out/phases.log | tail -24
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python tools/ktime.py > gpurun_out/ktime.json 2>&1; cat gpurun_out/ktime.json
