# quick GPU iteration: build, fused-vs-oracle tests, fused bench, ncu capture of the fused kernel
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 10 -c 1 \
    -o gpurun_out/prof_fused python bench.py --steps 10 --warmup 5 --ring 8 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
