set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -14
timeout 900 python bench.py --config 5 --steps 20 --warmup 3 2>&1 | tail -1 | cut -c1-600
