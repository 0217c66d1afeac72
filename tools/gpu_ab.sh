# A/B timing of fused-kernel variants: tmp_ab/<name>.cu replaces csrc/sf_fused.cu in turn.
# Usage: bash tools/gpu_ab.sh name1 name2 ...   (each: GPU parity + pyramid tests, bench x2, H=2 bench, phases)
set +e
CS=paper_2406_18031_b200/csrc/sf_fused.cu
cp $CS /tmp/sf_fused_orig.cu
for v in "$@"; do
  echo "=== $v"
  cp tmp_ab/$v.cu $CS
  python paper_2406_18031_b200/build.py --force > /dev/null || { echo build failed; continue; }
  timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
  for i in 1 2; do timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['ms_per_step']*1000,2), 'us', round(d['value']), 'Hz')"; done
  timeout 600 python bench.py --levels 2 --steps 1000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench H=2', round(d['ms_per_step']*1000,2), 'us', round(d['value']), 'Hz')"
  SF_BUILD_DEBUG=1 python paper_2406_18031_b200/build.py --force > /dev/null
  SF_DEBUG_SKIP=256 timeout 600 python bench.py --steps 64 --warmup 8 --no-cpu-baseline 2>&1 | grep SFTIME | tail -4
done
cp /tmp/sf_fused_orig.cu $CS
python paper_2406_18031_b200/build.py --force > /dev/null
