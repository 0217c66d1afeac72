# GPU suite on the shipped build, then the interleaved A/B of ab_lib/libsf_a.so vs the tree's build.
#   gpurun --timeout 1500 -- 'bash tools/gpu_test_ab.sh'
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/gputest.log
cat gpurun_out/gputest.log
bash tools/gpu_ab_lib.sh
