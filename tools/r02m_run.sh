# r02m: validation of the final build (fused pass without the dead unrolled-copy and prefetch code
# in its loop): smoke(), whole GPU suite, default bench line + short line, configs[1]/[3] lines,
# launch list and ncu --set full of the fused pass
O=gpurun_out
timeout 300 python __graft_entry__.py smoke > $O/r02m_smoke.log 2>&1; echo "rc=$?" >> $O/r02m_smoke.log; tail -2 $O/r02m_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/r02m_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02m_pytest.log; tail -3 $O/r02m_pytest.log
timeout 600 python bench.py > $O/r02m_bench.json 2> $O/r02m_bench.err; head -c 200 $O/r02m_bench.json; echo
for w in single deflation arnoldi tiny; do timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/r02m_bench_$w.json 2>> $O/r02m_bench.err; done
B="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $B > $O/r02m_bench_short.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02m_launches.csv $B > $O/r02m_launch.log 2>&1
python tools/launch_summary.py $O/r02m_launches.csv > $O/r02m_launches_summary.csv 2>/dev/null
C="python bench.py --variant cholqr2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream2 -s 3 -c 1 -o $O/r02m_fused $C > $O/r02m_fused.log 2>&1
python tools/ncu_summary.py $O/r02m_fused.ncu-rep > $O/r02m_ncu_fused.json 2> $O/r02m_ncu_summary.err
ncu -i $O/r02m_fused.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py 40 > $O/r02m_fused_lines.txt
rm -f $O/r02m_*.ncu-rep $O/r02m_launches.csv
timeout 700 python tools/stress_parity.py 300 303 > $O/r02m_stress_parity.txt 2>&1; tail -n 1 $O/r02m_stress_parity.txt
