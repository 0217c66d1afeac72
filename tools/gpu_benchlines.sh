# The bench lines kept under profiles/ (the default line, the reference arm, per-pass, H = 2,
# input mapping, configs 3-5 with their CPU baselines), each printed to the log as well.
#   TAG=r02 gpurun --timeout 3000 -- 'bash tools/gpu_benchlines.sh'
set -x
TAG=${TAG:-r02}
run() { name=$1; shift; timeout 1200 python bench.py "$@" 2>&1 | tail -1 > gpurun_out/${TAG}_bench_$name.json; cat gpurun_out/${TAG}_bench_$name.json; }
run default
run reference --impl reference --steps 20 --warmup 3
run passes --steps 500 --warmup 20 --kernel passes --no-cpu-baseline
run h2 --levels 2 --steps 1000 --warmup 50
run map --map --steps 2000 --warmup 50 --no-cpu-baseline
for c in 3 4 5; do run config$c --config $c --steps 40 --warmup 8; done
