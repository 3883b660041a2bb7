# ncu capture of the TSQR leaf kernels on the weak config (usage: bash tools/ncu_tsqr.sh TAG)
set -x
TAG=${1:-p}
CMD="python bench.py --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.json 2>&1 || exit 1
cat gpurun_out/${TAG}_plain.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wy_up -s 119 -c 1 -o gpurun_out/${TAG}_up $CMD > gpurun_out/${TAG}_up.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wy_down -s 13 -c 1 -o gpurun_out/${TAG}_down $CMD > gpurun_out/${TAG}_down.log 2>&1
ls -la gpurun_out
