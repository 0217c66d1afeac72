# Interleaved A/B of two builds (A = ab_lib/libsf_a.so, B = the tree's libsf.so), default bench,
# plus the per-CTA phase profile of each when debug builds ab_lib/libsf_a_dbg.so / libsf_b_dbg.so exist.
set -x
for rep in 1 2 3; do
  SF_LIB=ab_lib/libsf_a.so timeout 300 python bench.py --steps 2000 --warmup 20 --ring 48 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/abl_a$rep.json
  timeout 300 python bench.py --steps 2000 --warmup 20 --ring 48 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/abl_b$rep.json
done
python - <<'PY'
import json, statistics
a=[json.load(open(f'gpurun_out/abl_a{i}.json'))['ms_per_step']*1e3 for i in (1,2,3)]
b=[json.load(open(f'gpurun_out/abl_b{i}.json'))['ms_per_step']*1e3 for i in (1,2,3)]
print('A (ab_lib/libsf_a.so)', [round(x,2) for x in a], 'median', round(statistics.median(a),2))
print('B (tree)             ', [round(x,2) for x in b], 'median', round(statistics.median(b),2))
PY
for v in a b; do
  if [ -f ab_lib/libsf_${v}_dbg.so ]; then
    SF_LIB=ab_lib/libsf_${v}_dbg.so SF_DEBUG_SKIP=8192 timeout 300 python tools/ktime.py --frames 12 --ring 8 2>&1 | grep SFPROF | tail -4 | sed "s/^/$v /"
  fi
done
