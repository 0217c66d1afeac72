# One iteration: GPU suite (-x) on the shipped build, interleaved A/B of ab_lib/libsf_a.so vs the
# tree's build, and the phase clocks of the debug build ab_lib/libsf_dbg.so.
#   gpurun --timeout 1800 -- 'bash tools/gpu_iter.sh'
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/gputest.log
cat gpurun_out/gputest.log
LIBS="ab_lib/libsf_a.so paper_2406_18031_b200/libsf.so" bash tools/gpu_abn.sh
KNOBS="$KNOBS" bash tools/gpu_phases.sh
SF_LIB=ab_lib/libsf_dbg.so SF_DEBUG_SKIP=16384 timeout 300 python tools/cta_trace.py 2>&1 | tail -12
