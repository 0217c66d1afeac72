# Interleaved A/B/... of environment settings on the tree's build (ENVS="'' 'X=1' 'Y=2'"), default bench.
#   ENVS="..." gpurun --timeout 900 -- 'bash tools/gpu_abenv.sh'
set -x
ARGS=${ARGS:-"--steps 2000 --warmup 20 --ring 48 --no-cpu-baseline"}
eval "set -- $ENVS"
n=$#
for rep in 1 2 3; do
  i=0
  for E in "$@"; do
    env $E timeout 300 python bench.py $ARGS 2>&1 | tail -1 > gpurun_out/abe_${i}_$rep.json
    i=$((i+1))
  done
done
python - "$@" <<'PY'
import json, statistics, sys
for i, E in enumerate(sys.argv[1:]):
    v = []
    for r in (1, 2, 3):
        try:
            v.append(json.load(open(f'gpurun_out/abe_{i}_{r}.json'))['ms_per_step'] * 1e3)
        except Exception:
            v.append(float('nan'))
    print(f'{E or "(default)":32s}', [round(x, 2) for x in v], 'median', round(statistics.median(v), 2))
PY
