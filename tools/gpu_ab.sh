# Interleaved A/B of an environment switch on the default bench (3 runs each, same box).
#   AB_ENV="SF_NO_FLUSH=1" gpurun -- 'bash tools/gpu_ab.sh'
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 2000 --warmup 20 --ring 48 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/ab_a$rep.json
  env $AB_ENV timeout 300 python bench.py --steps 2000 --warmup 20 --ring 48 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/ab_b$rep.json
done
python - <<'PY'
import json, statistics
a=[json.load(open(f'gpurun_out/ab_a{i}.json'))['ms_per_step']*1e3 for i in (1,2,3)]
b=[json.load(open(f'gpurun_out/ab_b{i}.json'))['ms_per_step']*1e3 for i in (1,2,3)]
print('A (default)', [round(x,2) for x in a], 'median', round(statistics.median(a),2))
print('B (env)    ', [round(x,2) for x in b], 'median', round(statistics.median(b),2))
PY
