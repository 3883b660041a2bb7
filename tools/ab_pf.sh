# A/B of the fused pass's L2 prefetch distance (PQR_S2_PF rounds of 8 units) and one ncu capture
# of the fused kernel on the weak config; results in gpurun_out/ab1.txt, gpurun_out/s2f_*
rm -f gpurun_out/ab1.txt
AB_CFGS="PQR_S2_PF=0;PQR_S2_PF=1;PQR_S2_PF=2;PQR_S2_PF=4;PQR_S2_PF=8;PQR_S2_PF=0" bash tools/ab_s2.sh
cat gpurun_out/ab1.txt
bash tools/ncu_one.sh s2f k_stream2 1 python bench.py --variant cholqr2 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline
head -c 3000 gpurun_out/s2f_summary.json
