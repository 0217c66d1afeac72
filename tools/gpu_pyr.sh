python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_eval.py -q -x 2>&1 | tail -15
