# End-of-round GPU pass: tests, every bench line kept under profiles/, ncu launch lists and the
# ncu --set full capture of k_fused, configs 3-5 and the paper's Table 2/3 sweeps.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json
cat gpurun_out/bench_default.json
timeout 600 python bench.py --steps 500 --warmup 20 --kernel passes --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_passes.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_reference.json
timeout 600 python bench.py --levels 2 --steps 1000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_h2.json
timeout 600 python bench.py --levels 2 --map --steps 1000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_h2_map.json
timeout 600 python bench.py --map --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_map.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --ring 8 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_h2.csv python bench.py --levels 2 --steps 20 --warmup 5 --ring 8 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 10 -c 1 \
    -o gpurun_out/prof_fused python bench.py --steps 10 --warmup 5 --ring 8 --no-cpu-baseline > /dev/null 2>&1
bash tools/gpu_configs.sh
bash tools/gpu_sweep.sh
ls gpurun_out
