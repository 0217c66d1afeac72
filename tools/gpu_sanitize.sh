# memcheck the smoke run (fused kernel, TMA path)
python -c "import __graft_entry__ as g; g.build()"
CUDA_LAUNCH_BLOCKING=1 timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | grep -v "Host Frame" | head -40
