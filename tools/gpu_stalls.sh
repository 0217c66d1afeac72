# Warp-stall profile of the split step's two kernels (config 2): one ncu --set full capture with
# source, the SASS source page per kernel and its per-region stall summary (tools/ncu_source.py).
#   TAG=r02s gpurun --timeout 1200 -- 'bash tools/gpu_stalls.sh'
set -x
TAG=${TAG:-r02s}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_trans|k_upd' -s 6 -c 2 \
    -o gpurun_out/${TAG}_cfg2 python bench.py --steps 6 --warmup 3 --ring 8 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
for k in k_trans k_upd; do
  ncu -i gpurun_out/${TAG}_cfg2.ncu-rep -k regex:"$k" --page source --csv --print-source sass > gpurun_out/${TAG}_${k}_src.csv 2>/dev/null
  python tools/ncu_source.py gpurun_out/${TAG}_${k}_src.csv > gpurun_out/${TAG}_${k}_regions.txt 2>&1
done
ncu -i gpurun_out/${TAG}_cfg2.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
ls -la gpurun_out
