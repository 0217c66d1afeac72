# which part of the edge transport instantiation costs time: every CTA on the EDGE path
# (SF_DEBUG_SKIP=6144), with parts compiled out (timing only: results are wrong with these)
for ex in "" "-DSF_EXP_NO_COLREP" "-DSF_EXP_NO_ROWREP" "-DSF_EXP_NO_IN1" "-DSF_EXP_NO_COLREP -DSF_EXP_NO_ROWREP -DSF_EXP_NO_IN1"; do
  SF_BUILD_DEBUG=1 SF_NVCC_EXTRA="$ex" python paper_2406_18031_b200/build.py --force > /dev/null
  SF_DEBUG_SKIP=6144 timeout 600 python bench.py --steps 24 --warmup 8 --ring 8 --no-cpu-baseline 2>&1 | grep SFGT > gpurun_out/gt_iter.txt
  echo "== extra: $ex"; python tools/gt_classes.py gpurun_out/gt_iter.txt | grep -E "interior|left|top"
done
python paper_2406_18031_b200/build.py --force > /dev/null
