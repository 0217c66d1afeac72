# k_upd solve experiments: no in-loop fetches (16), no LDL^T (1024), both.
set -x
SF_BUILD_DEBUG=1 python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for k in 8192 8208 9216 9232; do
  SF_DEBUG_SKIP=$k timeout 300 python tools/ktime.py --frames 12 --ring 8 2>&1 | grep 'SFPROF upd' | tail -2
done
