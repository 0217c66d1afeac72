# Pyramid GPU tests on the tree's build, then an interleaved H = 2 A/B of the builds in LIBS.
set -x
timeout 900 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_parity.py -q -x -k "pyramid or config1 or random" 2>&1 | tail -2
ARGS="--levels 2 --steps 1000 --warmup 50 --ring 48 --no-cpu-baseline" LIBS="$LIBS" bash tools/gpu_abn.sh
