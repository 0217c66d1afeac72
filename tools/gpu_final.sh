# Closing GPU pass of a session: compute-sanitizer over the kernels, the default bench line and
# its ncu launch list (TAG names the profiles).
#   TAG=r02 gpurun --timeout 3000 -- 'bash tools/gpu_final.sh'
set -x
TAG=${TAG:-r02}
bash tools/gpu_sanitize.sh > gpurun_out/${TAG}_sanitizer.txt 2>&1
cat gpurun_out/${TAG}_sanitizer.txt | grep -c "ERROR SUMMARY: 0"
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/${TAG}_bench_default.json
cat gpurun_out/${TAG}_bench_default.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 20 --warmup 5 --ring 8 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py --launches gpurun_out/${TAG}_launches.csv --tag ${TAG} > /dev/null 2>&1
cp profiles/${TAG}_launches.md gpurun_out/ 2>/dev/null
