# ncu --set full of the leaf stage-1 kernel with chains on and off (weak config), summaries + per-line stalls
B="python bench.py --variant tsqr --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
PQR_CHAINS=on timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_wy_upILi4ELi1ELi8ELb0ELi2ELb1" -s 17 -c 1 -o gpurun_out/ch_on $B > gpurun_out/ch_on.log 2>&1
PQR_CHAINS=off timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_wy_upILi4ELi1ELi8ELb0ELi2ELb0" -s 17 -c 1 -o gpurun_out/ch_off $B > gpurun_out/ch_off.log 2>&1
python tools/ncu_summary.py gpurun_out/ch_on.ncu-rep gpurun_out/ch_off.ncu-rep > gpurun_out/ch_summary.json
for k in on off; do
  ncu -i gpurun_out/ch_$k.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py 30 > gpurun_out/ch_${k}_lines.txt
  ncu -i gpurun_out/ch_$k.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/ch_${k}_raw.csv
done
rm -f gpurun_out/ch_on.ncu-rep gpurun_out/ch_off.ncu-rep
