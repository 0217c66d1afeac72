# A/B on one box: k_upd geometry from separate planes vs interleaved (SF_UPD_GS); spin-queued kernel
# timing in the bench; the banded substep-exchange tests.
set -x
SF_BUILD_DEBUG=1 python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for rep in 1 2; do
  SF_DEBUG_SKIP=8192 timeout 300 python tools/ktime.py --frames 12 --ring 8 2>&1 | grep 'SFPROF upd' | tail -2
  SF_UPD_GS=1 SF_DEBUG_SKIP=8192 timeout 300 python tools/ktime.py --frames 12 --ring 8 2>&1 | grep 'SFPROF upd' | tail -2
done
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for v in "" 1; do
  SF_UPD_GS=$v timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_it8_$v.json
  python -c "import json; d=json.load(open('gpurun_out/bench_it8_$v.json')); r=d['roofline']; print('BENCH GS=$v', d['value'], d['ms_per_step']*1e3, r.get('kernel_times'))"
done
timeout 900 python -m pytest tests/test_gpu_band_substep.py -m gpu -q -x 2>&1 | tail -15
