# The paper's Tables 2 (H = 1) and 3 (H = 2) sweeps at 512^2 (max flow 1, 2, 4, 8 px), with the
# Spherepix input mapping inside the step (the paper's timed region).
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for lv in 1 2; do for mf in 1 2 4 8; do
  timeout 900 python bench.py --levels $lv --max-flow $mf --map --ring 48 --steps 1000 --warmup 40 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/${TAG}_sweep_${lv}_${mf}.json
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_sweep_${lv}_${mf}.json')); print('H=$lv', 'maxflow=$mf', round(d['value']), 'Hz', round(d['ms_per_step']*1000,1), 'us', d['device_flags'])"
done; done
