# A/B: k_stream2 in Gram / update mode (PQR_S2_GRAM=1, PQR_S2_UPD=1) against the default
# k_gram_cpa / k_update_cpa passes, after the code-size cuts of k_stream2.
O=gpurun_out/s2modes_ab.txt
run() {  # workload env...
  w=$1; shift
  env "$@" timeout 300 python bench.py --workload $w --variant cholqr2 --steps 8 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/_ab.json 2>/dev/null
  python -c "
import json
d = json.load(open('gpurun_out/_ab.json'))
r = d.get('roofline_by_kernel') or {}
print('$w', '$*', round(d['value'], 1), round(d['ms_per_step'], 3), {k: (round(v['avg_launch_ms'], 3), round(v['frac'], 3)) for k, v in r.items()}, d['clocks']['sm_mhz'])
" >> $O
}
for rep in 1 2; do
  run weak PQR_X=0
  run weak PQR_S2_GRAM=1
  run weak PQR_S2_UPD=1
done
run single PQR_X=0
run single PQR_S2_GRAM=1
run single PQR_S2_UPD=1
cat $O
