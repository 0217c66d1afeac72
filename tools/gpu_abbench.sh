# bench-only A/B of fused-kernel variants (tmp_ab/<name>.cu), 3 runs each, interleaved
CS=paper_2406_18031_b200/csrc/sf_fused.cu
cp $CS /tmp/sf_fused_orig.cu
for v in "$@"; do
  cp tmp_ab/$v.cu $CS; python paper_2406_18031_b200/build.py --force > /dev/null && cp paper_2406_18031_b200/libsf.so /tmp/libsf_$v.so
done
for rep in 1 2 3; do for v in "$@"; do
  cp /tmp/libsf_$v.so paper_2406_18031_b200/libsf.so
  echo -n "$v "; timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us')"
done; done
cp /tmp/sf_fused_orig.cu $CS; python paper_2406_18031_b200/build.py --force > /dev/null
