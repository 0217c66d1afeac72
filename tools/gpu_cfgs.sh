# compare fused-kernel region configurations (bench only) + parity tests with the alternate config
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
for cfg in 0 1; do
  SF_FUSED_CFG=$cfg timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
done
SF_FUSED_CFG=1 timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in 0 1; do
SF_FUSED_CFG=$cfg timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 10 -c 1 \
    -o gpurun_out/prof_cfg$cfg python bench.py --steps 10 --warmup 5 --ring 8 --no-cpu-baseline > /dev/null 2>&1
done
