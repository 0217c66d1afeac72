# per-CTA-class timing (debug build): default, and with every CTA on the edge transport instantiation
SF_BUILD_DEBUG=1 python paper_2406_18031_b200/build.py --force > /dev/null
for k in 2048; do
SF_DEBUG_SKIP=$k timeout 600 python bench.py --steps 24 --warmup 8 --ring 8 --no-cpu-baseline 2>&1 | grep SFGT > gpurun_out/gt_iter.txt
echo "SF_DEBUG_SKIP=$k"; python tools/gt_classes.py gpurun_out/gt_iter.txt
done
