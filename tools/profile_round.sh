# Round evidence: bench line, launch list (cold/serialised) and one ncu --set full capture of
# the dominant kernel (leaf stage-1 TSQR kernel), all for the default bench command.
# usage: bash tools/profile_round.sh TAG
TAG=${1:-r}
B="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err || exit 1
timeout 300 $B > gpurun_out/${TAG}_bench_short.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wy_up -s 119 -c 1 -o gpurun_out/${TAG}_wy_up python bench.py --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_wy_up.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update_gram|k_gram_cpa|k_update_cpa" -s 3 -c 3 -o gpurun_out/${TAG}_cholqr python bench.py --variant cholqr2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_cholqr.log 2>&1
ls -la gpurun_out | grep ${TAG}
