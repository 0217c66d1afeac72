# End-of-round GPU pass: smoke, the GPU suite, every bench line kept under profiles/ (default,
# e2e, reference arm, per-pass, H = 2, input mapping, configs 3-5, the paper's Table 2/3 sweeps),
# the ncu launch lists of the default and H = 2 benches and the per-kernel ncu evidence.
#   TAG=r02 gpurun --timeout 3600 -- 'bash tools/gpu_round.sh'
set -x
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/${TAG}_gputest.txt; cat gpurun_out/${TAG}_gputest.txt
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/${TAG}_bench_default.json
cat gpurun_out/${TAG}_bench_default.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/${TAG}_bench_reference.json
timeout 600 python bench.py --steps 500 --warmup 20 --kernel passes --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/${TAG}_bench_passes.json
timeout 600 python bench.py --levels 2 --steps 1000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/${TAG}_bench_h2.json
timeout 600 python bench.py --map --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/${TAG}_bench_map.json
for c in 3 4 5; do
  timeout 1200 python bench.py --config $c --steps 40 --warmup 8 2>&1 | tail -1 > gpurun_out/${TAG}_bench_config$c.json
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 20 --warmup 5 --ring 8 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py --launches gpurun_out/${TAG}_launches.csv --tag ${TAG} > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/${TAG}_launches_h2.csv python bench.py --levels 2 --steps 20 --warmup 5 --ring 8 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py --launches gpurun_out/${TAG}_launches_h2.csv --tag ${TAG}_h2 > /dev/null 2>&1
cp profiles/${TAG}_launches.md profiles/${TAG}_h2_launches.md gpurun_out/ 2>/dev/null
TAG=$TAG bash tools/gpu_sweep.sh
ls gpurun_out
