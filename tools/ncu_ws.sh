# ncu --set full of the fused CholQR2 pass on the weak config in both forms (consumer-side refill,
# the default for one output tile, and the warp-specialised form forced with PQR_S2_WS=1): kernel
# summary, per-line and per-SASS-instruction stall samples.  usage: bash tools/ncu_ws.sh TAG
TAG=${1:-ws}; O=gpurun_out
C="python bench.py --variant cholqr2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
for ws in 0 1; do
  PQR_S2_WS=$ws timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream2 -s 3 -c 1 -o $O/${TAG}_ws$ws $C > $O/${TAG}_ws$ws.log 2>&1
  python tools/ncu_summary.py $O/${TAG}_ws$ws.ncu-rep > $O/${TAG}_ws${ws}_ncu.json 2> $O/${TAG}_ws${ws}_summary.err
  ncu -i $O/${TAG}_ws$ws.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py 30 > $O/${TAG}_ws${ws}_lines.txt
  python tools/ncu_sass_stalls.py $O/${TAG}_ws$ws.ncu-rep 60 > $O/${TAG}_ws${ws}_sass.txt 2>&1
done
rm -f $O/${TAG}_ws*.ncu-rep
