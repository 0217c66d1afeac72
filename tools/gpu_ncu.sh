# ncu: launch list of a short bench run and one full capture of the fused kernel.
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --ring 8 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 10 -c 2 \
    -o gpurun_out/prof_fused python bench.py --steps 10 --warmup 5 --ring 8 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
