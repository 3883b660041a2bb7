# Round evidence (round 2 layout): GPU tests, every workload's bench line, the default bench
# command's launch list, ncu --set full of the dominant kernels (fused CholQR2 pass k_stream2, the
# Gram and update passes, the TSQR leaf kernels), summaries.  usage: bash tools/profile_round2.sh TAG
TAG=${1:-r}
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
for w in tiny single deflation arnoldi; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/${TAG}_bench_$w.json 2>> $O/${TAG}_bench.err
done
timeout 600 python bench.py --impl reference > $O/${TAG}_bench_reference.json 2>> $O/${TAG}_bench.err
B="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $B > $O/${TAG}_bench_short.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv $B > $O/${TAG}_launch.log 2>&1
python tools/launch_summary.py $O/${TAG}_launches.csv > $O/${TAG}_launches_summary.csv 2>/dev/null
C="python bench.py --variant cholqr2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream2 -s 3 -c 1 -o $O/${TAG}_fused $C > $O/${TAG}_fused.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_cpa|k_update_cpa" -s 6 -c 2 -o $O/${TAG}_cholqr $C > $O/${TAG}_cholqr.log 2>&1
T="python bench.py --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_wy_upILi4ELi1ELi8ELb0ELi2ELb0" -s 19 -c 1 -o $O/${TAG}_wy_up $T > $O/${TAG}_wy_up.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_wy_downILi4ELi1ELi8ELi2ELb0" -s 3 -c 1 -o $O/${TAG}_wy_down $T > $O/${TAG}_wy_down.log 2>&1
python tools/ncu_summary.py $O/${TAG}_fused.ncu-rep $O/${TAG}_cholqr.ncu-rep $O/${TAG}_wy_up.ncu-rep $O/${TAG}_wy_down.ncu-rep > $O/${TAG}_ncu_full.json 2> $O/${TAG}_ncu_summary.err
for k in fused wy_up wy_down; do
  ncu -i $O/${TAG}_$k.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py 40 > $O/${TAG}_${k}_lines.txt
done
rm -f $O/${TAG}_*.ncu-rep $O/${TAG}_launches.csv
ls -la $O | grep ${TAG}
