set -x
TAG=r02
timeout 1200 python bench.py --config 5 --steps 40 --warmup 8 2>&1 | tail -1 > gpurun_out/r02_bench_config5.json
cat gpurun_out/r02_bench_config5.json
NCU="timeout 900 ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 6 --warmup 3 --ring 8 --no-cpu-baseline"
PX2=262144
$NCU -k regex:'k_upd' -s 6 -c 1 -o gpurun_out/${TAG}_h2u_top $B --levels 2 > /dev/null 2>&1
$NCU -k regex:'k_upd' -s 7 -c 1 -o gpurun_out/${TAG}_h2u_bot $B --levels 2 > /dev/null 2>&1
rm -f profiles/${TAG}_evidence.md
python tools/ncu_evidence.py gpurun_out/${TAG}_h2u_top.ncu-rep --kernel 'k_upd\(' --pixels 65536 --algo-bytes 52 --algo-ops 217 --tag $TAG --name h2top_k_upd --label "H=2 top 256^2 S=4"
python tools/ncu_evidence.py gpurun_out/${TAG}_h2u_bot.ncu-rep --kernel 'k_upd\(' --pixels $PX2 --algo-bytes 68 --algo-ops 163 --tag $TAG --name h2bot_k_upd --label "H=2 bottom 512^2 [dU] + reconstruction"
cp profiles/${TAG}_evidence.md gpurun_out/r02_evidence_h2upd.md; cp profiles/${TAG}_h2*_k_upd.json gpurun_out/
rm -f gpurun_out/*.ncu-rep
