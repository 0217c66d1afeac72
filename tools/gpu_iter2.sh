# GPU suite + default bench line + interleaved A/B of the builds in LIBS.
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/gputest.log
cat gpurun_out/gputest.log
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_now.json
python -c "import json; d=json.load(open('gpurun_out/bench_now.json')); r=d['roofline']; print('bench', d['ms_per_step']*1e3, 'us', 'frac', r['frac'], 'traffic', r['traffic'], 'k_trans', r['kernel_ms'], 'k_upd', r['update_kernel']['kernel_ms'], 'single', r['kernel_times']['single_frame'])"
[ -n "$LIBS" ] && LIBS="$LIBS" bash tools/gpu_abn.sh
