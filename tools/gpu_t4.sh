bash tools/gpu_t2.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 10 -c 1 \
    -o gpurun_out/prof_box python bench.py --steps 10 --warmup 5 --ring 8 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
