python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py fused 2>&1 | grep -E "SUMMARY|bitwise|Race" | head
SF_NO_TMA=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py fused 2>&1 | grep -E "SUMMARY|bitwise|Race" | head
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['ms_per_step']*1000,2), 'us', round(d['value']), 'Hz')"; done
