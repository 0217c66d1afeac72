# per-CTA globaltimer trace of consecutive fused launches (debug build, SF_DEBUG_SKIP=2048):
# entry, griddep release, exit, e planes landed; with TMA staging and with cp.async staging
SF_BUILD_DEBUG=1 python paper_2406_18031_b200/build.py --force > /dev/null
SF_DEBUG_SKIP=2048 timeout 600 python bench.py --steps 24 --warmup 8 --ring 8 --no-cpu-baseline 2>&1 | grep SFGT > gpurun_out/gt.txt
SF_NO_TMA=1 SF_DEBUG_SKIP=2048 timeout 600 python bench.py --steps 24 --warmup 8 --ring 8 --no-cpu-baseline 2>&1 | grep SFGT > gpurun_out/gt_notma.txt
python paper_2406_18031_b200/build.py --force > /dev/null
SF_NO_TMA=1 timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench no-TMA', round(d['ms_per_step']*1000,2), 'us')"
