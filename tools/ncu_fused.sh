# ncu capture of the CholQR2 fused second-pass kernel on the weak config (usage: bash tools/ncu_fused.sh TAG)
TAG=${1:-f}
CMD="python bench.py --variant cholqr2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/${TAG}_plain.json 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update_gram_pair -s 2 -c 1 -o gpurun_out/${TAG}_fused $CMD > gpurun_out/${TAG}_fused.log 2>&1
