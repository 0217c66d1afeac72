# lib A/B + the parity / pyramid GPU tests on the tree build.
bash tools/gpu_ab_lib.sh
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pyramid.py tests/test_gpu_band_substep.py -m gpu -q -x 2>&1 | tail -3
