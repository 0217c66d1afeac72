# ncu --set full evidence for every kernel of the hot path and the NEXT rows (DESIGN.md section 8,
# profiles/r02_evidence.md): captures steady-state launches, summarises them on the box
# (tools/ncu_evidence.py) and keeps the small reports of the headline kernels.
set -x
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
NCU="timeout 900 ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 6 --warmup 3 --ring 8 --no-cpu-baseline"
PX2=262144
rm -f profiles/${TAG}_evidence.md
# config 2, split fused step
$NCU -k regex:'k_trans|k_upd' -s 6 -c 2 -o gpurun_out/${TAG}_cfg2 $B > /dev/null 2>&1
python tools/ncu_evidence.py gpurun_out/${TAG}_cfg2.ncu-rep --kernel k_trans --pixels $PX2 --algo-bytes 32 --algo-ops 416 --tag $TAG --name cfg2_k_trans --label "cfg2 512^2 N=8"
python tools/ncu_evidence.py gpurun_out/${TAG}_cfg2.ncu-rep --kernel 'k_upd\(' --pixels $PX2 --algo-bytes 52 --algo-ops 163 --tag $TAG --name cfg2_k_upd --label "cfg2 512^2 S=2"
# config 2, per-pass kernels
$NCU -k regex:'k_pass' -s 40 -c 4 -o gpurun_out/${TAG}_passes $B --kernel passes > /dev/null 2>&1
$NCU -k regex:'k_update|k_box' -s 9 -c 3 -o gpurun_out/${TAG}_passes_u $B --kernel passes > /dev/null 2>&1
python tools/ncu_evidence.py gpurun_out/${TAG}_passes.ncu-rep --kernel 'k_pass<0>' --pixels $PX2 --algo-bytes 32 --algo-ops 26 --tag $TAG --label "cfg2 passes"
python tools/ncu_evidence.py gpurun_out/${TAG}_passes.ncu-rep --kernel 'k_pass<1>' --pixels $PX2 --algo-bytes 32 --algo-ops 26 --tag $TAG --label "cfg2 passes"
python tools/ncu_evidence.py gpurun_out/${TAG}_passes_u.ncu-rep --kernel 'k_update' --pixels $PX2 --algo-bytes 56 --algo-ops 109 --tag $TAG --label "cfg2 passes"
python tools/ncu_evidence.py gpurun_out/${TAG}_passes_u.ncu-rep --kernel 'k_box' --pixels $PX2 --algo-bytes 32 --algo-ops 27 --tag $TAG --label "cfg2 passes"
# config 2 through the two-level pyramid (NEXT #1)
$NCU -k regex:'k_low|k_down2|k_up2_add|k_trans|k_update|k_box' -s 30 -c 12 -o gpurun_out/${TAG}_h2 $B --levels 2 > /dev/null 2>&1
python tools/ncu_evidence.py gpurun_out/${TAG}_h2.ncu-rep --kernel k_low --pixels $PX2 --algo-bytes 64 --algo-ops 672 --tag $TAG --label "H=2 bottom 512^2 N=8"
python tools/ncu_evidence.py gpurun_out/${TAG}_h2.ncu-rep --kernel k_trans --pixels 65536 --algo-bytes 32 --algo-ops 208 --tag $TAG --name h2top_k_trans --label "H=2 top 256^2 N=4"
# k_upd launches alternate top (256^2, S = 4) / bottom (512^2 [dU] + reconstruction) per frame: one capture each
$NCU -k regex:'k_upd' -s 6 -c 1 -o gpurun_out/${TAG}_h2u_top $B --levels 2 > /dev/null 2>&1
$NCU -k regex:'k_upd' -s 7 -c 1 -o gpurun_out/${TAG}_h2u_bot $B --levels 2 > /dev/null 2>&1
python tools/ncu_evidence.py gpurun_out/${TAG}_h2u_top.ncu-rep --kernel 'k_upd\(' --pixels 65536 --algo-bytes 52 --algo-ops 217 --tag $TAG --name h2top_k_upd --label "H=2 top 256^2 S=4"
python tools/ncu_evidence.py gpurun_out/${TAG}_h2u_bot.ncu-rep --kernel 'k_upd\(' --pixels $PX2 --algo-bytes 68 --algo-ops 163 --tag $TAG --name h2bot_k_upd --label "H=2 bottom 512^2 [dU] + reconstruction"
python tools/ncu_evidence.py gpurun_out/${TAG}_h2.ncu-rep --kernel k_down2 --pixels $PX2 --algo-bytes 10 --tag $TAG --label "H=2"
python tools/ncu_evidence.py gpurun_out/${TAG}_h2.ncu-rep --kernel k_up2_add --pixels $PX2 --algo-bytes 36 --tag $TAG --label "H=2"
# input mapping (NEXT #2)
$NCU -k regex:'k_map' -s 6 -c 2 -o gpurun_out/${TAG}_map $B --map > /dev/null 2>&1
python tools/ncu_evidence.py gpurun_out/${TAG}_map.ncu-rep --kernel k_map --pixels $PX2 --algo-bytes 8 --tag $TAG --label "cfg2 --map"
# config 4 (batch 64, HBM-sized) and config 3 (1024^2, N = 16: two transport launches)
$NCU -k regex:'k_trans' -s 4 -c 1 -o gpurun_out/${TAG}_cfg4 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
$NCU -k regex:'k_upd$' -s 4 -c 1 -o gpurun_out/${TAG}_cfg4u python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_evidence.py gpurun_out/${TAG}_cfg4.ncu-rep --kernel k_trans --pixels 16777216 --algo-bytes 32 --algo-ops 416 --tag $TAG --name cfg4_k_trans --label "cfg4 64x512^2"
python tools/ncu_evidence.py gpurun_out/${TAG}_cfg4u.ncu-rep --kernel 'k_upd\(' --pixels 16777216 --algo-bytes 52 --algo-ops 163 --tag $TAG --name cfg4_k_upd --label "cfg4 64x512^2"
$NCU -k regex:'k_trans|k_upd' -s 9 -c 3 -o gpurun_out/${TAG}_cfg3 python bench.py --config 3 --steps 3 --warmup 3 --ring 4 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_evidence.py gpurun_out/${TAG}_cfg3.ncu-rep --kernel k_trans --pixels 1048576 --algo-bytes 32 --algo-ops 416 --tag $TAG --name cfg3_k_trans --label "cfg3 1024^2 N=16 (8 substeps per launch)"
python tools/ncu_evidence.py gpurun_out/${TAG}_cfg3.ncu-rep --kernel 'k_upd\(' --pixels 1048576 --algo-bytes 52 --algo-ops 163 --tag $TAG --name cfg3_k_upd --label "cfg3 1024^2"
cp profiles/${TAG}_evidence.md profiles/${TAG}_cfg*_*.json profiles/${TAG}_h2*_*.json profiles/${TAG}_k_*.json gpurun_out/ 2>/dev/null
rm -f gpurun_out/${TAG}_passes*.ncu-rep gpurun_out/${TAG}_h2.ncu-rep gpurun_out/${TAG}_map.ncu-rep gpurun_out/${TAG}_cfg4*.ncu-rep gpurun_out/${TAG}_cfg3.ncu-rep
rm -f profiles/${TAG}_evidence.md.bak
ls -la gpurun_out | tail -30
cat profiles/${TAG}_evidence.md
