python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not config5" 2>&1 | tail -2
bash tools/gpu_t2.sh
