set -x
CMD="python bench.py --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/p1_plain.json 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wy_up -s 119 -c 2 -o gpurun_out/p1_up $CMD > gpurun_out/p1_up.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wy_down -s 12 -c 2 -o gpurun_out/p1_down $CMD > gpurun_out/p1_down.log 2>&1
python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/p1_bench2.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/p1_launch.log 2>&1
ls -la gpurun_out
