python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for a in "--map" "--levels 2 --map"; do
timeout 900 python bench.py $a --steps 1000 --warmup 40 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_tmp.json
python -c "import json,sys; d=json.load(open('gpurun_out/bench_tmp.json')); print('$a', round(d['value']), 'Hz', round(d['ms_per_step']*1000,2), 'us', d['device_flags'], d['gpu_launches']/d['steps'])"
cp gpurun_out/bench_tmp.json "gpurun_out/bench_$(echo $a | tr -d ' -').json"
done
