# Per-CTA phase clocks (debug build ab_lib/libsf_dbg.so, SF_DEBUG_SKIP=8192) of k_trans and k_upd on
# the bench workload, plus the timing knobs given in KNOBS (each added to 8192).
#   KNOBS="16 1024" gpurun --timeout 600 -- 'bash tools/gpu_phases.sh'
set -x
for k in 0 $KNOBS; do
  echo "== knob $k"
  SF_LIB=ab_lib/libsf_dbg.so SF_DEBUG_SKIP=$((8192 + k)) timeout 300 python tools/ktime.py --frames 12 --ring 8 2>&1 | grep -E "SFPROF|median" | tail -6
done
