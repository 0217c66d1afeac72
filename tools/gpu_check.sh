# GPU-box check: build, smoke, parity tests, benches, ncu launch list + one full capture.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 2000 --warmup 50 2>&1 | tail -1
timeout 600 python bench.py --steps 500 --warmup 20 --kernel passes --no-cpu-baseline 2>&1 | tail -1
