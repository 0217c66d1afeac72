# H = 2 breakdown: ncu launch list of the pyramid bench; bench H = 2 with the bottom update fused / per-pass.
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python bench.py --levels 2 --steps 1000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_h2_a.json
python -c "import json; d=json.load(open('gpurun_out/bench_h2_a.json')); print('BENCH H2', d['value'], d['ms_per_step']*1e3)"
SF_UPD_LOW_PASSES=1 timeout 300 python bench.py --levels 2 --steps 1000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_h2_b.json
python -c "import json; d=json.load(open('gpurun_out/bench_h2_b.json')); print('BENCH H2 passes-update', d['value'], d['ms_per_step']*1e3)"
SF_FUSED_MODE=mono timeout 300 python bench.py --levels 2 --steps 1000 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_h2_c.json
python -c "import json; d=json.load(open('gpurun_out/bench_h2_c.json')); print('BENCH H2 mono-top', d['value'], d['ms_per_step']*1e3)"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
    --log-file gpurun_out/launches_h2.csv python bench.py --levels 2 --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py --launches gpurun_out/launches_h2.csv --tag r02h2 2>&1 | tail -1; cat profiles/r02h2_launches.md
cp profiles/r02h2_launches.md gpurun_out/
