# compute-sanitizer over the fused / per-pass / pyramid paths (tools/sanitize_run.py):
# memcheck (out-of-bounds, misaligned), racecheck (shared-memory hazards), synccheck (barriers),
# initcheck (reads of uninitialised global memory).  Summary lines -> gpurun_out/sanitize.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for tool in memcheck racecheck synccheck initcheck; do
  for w in fused passes pyramid; do
    echo "== $tool $w"
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py $w 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|bitwise ok|Error|error|Hazard|hazard" | head -12
  done
done
