# Split step (k_trans + k_upd): GPU tests, then A/B of the transport shapes against the monolithic kernel.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gputest_split.log
cat gpurun_out/gputest_split.log
for cfg in 0 1 2; do
  SF_TRANS_CFG=$cfg timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_split_$cfg.json
done
SF_FUSED_MODE=mono timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_mono.json
for f in gpurun_out/bench_split_*.json gpurun_out/bench_mono.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step']*1e3)"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
    --log-file gpurun_out/launches_split.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py --launches gpurun_out/launches_split.csv --tag r02split 2>&1 | tail -3; cat profiles/r02split_launches.md
