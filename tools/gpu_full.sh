# Full GPU round: build+smoke, parity tests, default bench (+cpu_baseline), passes bench,
# reference arm, ncu launch list + one --set full capture of the fused kernel.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json
cat gpurun_out/bench_default.json
timeout 600 python bench.py --steps 500 --warmup 20 --kernel passes --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_passes.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_reference.json
cat gpurun_out/bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --ring 8 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_passes.csv python bench.py --steps 5 --warmup 3 --ring 8 --kernel passes --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 10 -c 1 \
    -o gpurun_out/prof_fused python bench.py --steps 10 --warmup 5 --ring 8 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
