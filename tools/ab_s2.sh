# A/B of the stream2 fused kernel variants (env) on CholQR2 bench lines; results in gpurun_out/ab1.txt
line() {
  env $2 timeout ${AB_TO:-300} python bench.py --workload $1 --variant cholqr2 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab_line.json 2>/dev/null || { echo "$1 $2 FAILED" >> gpurun_out/ab1.txt; return; }
  python -c "
import json,sys; d=json.load(open('gpurun_out/ab_line.json'))
print('$1 $2', round(d['value'],1), round(d['ms_per_step'],3), {k:(round(v['avg_launch_ms'],3), round(v['frac'],3)) for k,v in d['roofline_by_kernel'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/ab1.txt
}
IFS=';'
for cfg in ${AB_CFGS:-"PQR_S2=0;PQR_S2=1"}; do IFS=' '; line ${AB_WL:-weak} "$cfg"; IFS=';'; done
