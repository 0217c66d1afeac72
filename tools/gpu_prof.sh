# Per-kernel steady-state times (tools/ktime.py) and ncu --set full captures of k_trans and k_upd.
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python tools/ktime.py > gpurun_out/ktime.json 2>&1; cat gpurun_out/ktime.json
SF_TRANS_CFG=1 timeout 300 python tools/ktime.py > gpurun_out/ktime_c1.json 2>&1; cat gpurun_out/ktime_c1.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_trans|k_upd' -s 20 -c 2 \
    -o gpurun_out/prof_split python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
