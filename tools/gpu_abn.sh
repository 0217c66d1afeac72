# Interleaved A/B/... of several builds of libsf (LIBS="ab_lib/libsf_a.so ab_lib/libsf_b.so ..."), default
# bench, 3 rounds; prints the per-build median us/frame.
#   LIBS="..." gpurun --timeout 900 -- 'bash tools/gpu_abn.sh'
set -x
ARGS=${ARGS:-"--steps 2000 --warmup 20 --ring 48 --no-cpu-baseline"}
for rep in 1 2 3; do
  i=0
  for L in $LIBS; do
    SF_LIB=$L timeout 300 python bench.py $ARGS 2>&1 | tail -1 > gpurun_out/abn_${i}_$rep.json
    i=$((i+1))
  done
done
python - "$LIBS" <<'PY'
import json, statistics, sys
libs = sys.argv[1].split()
for i, L in enumerate(libs):
    v = []
    for r in (1, 2, 3):
        try:
            v.append(json.load(open(f'gpurun_out/abn_{i}_{r}.json'))['ms_per_step'] * 1e3)
        except Exception as e:
            v.append(float('nan'))
    print(f'{L:32s}', [round(x, 2) for x in v], 'median', round(statistics.median(v), 2))
PY
