# H = 2 A/B of environment settings (ENVS), interleaved, 3 rounds; pyramid GPU tests first.
set -x
timeout 900 python -m pytest tests/test_gpu_pyramid.py -q -x 2>&1 | tail -2
ARGS="--levels 2 --steps 1000 --warmup 50 --ring 48 --no-cpu-baseline" ENVS="$ENVS" bash tools/gpu_abenv.sh
