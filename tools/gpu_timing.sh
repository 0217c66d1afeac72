python -c "import __graft_entry__ as g; g.build()"
SF_BUILD_DEBUG=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SF_DEBUG_SKIP=256 timeout 600 python bench.py --steps 64 --warmup 8 --no-cpu-baseline 2>&1 | grep SFTIME | sort | tail -8
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1  # back to the production build
