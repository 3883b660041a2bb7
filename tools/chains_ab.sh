# TSQR with FlatTSPQR leaf chains on / off (PQR_CHAINS), interleaved: usage: bash tools/chains_ab.sh "weak deflation"
for rep in 1 2; do
  for w in $1; do
    for c in off on; do
      PQR_CHAINS=$c timeout 200 python bench.py --workload $w --variant tsqr --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('chains=$c', '$w', round(d['variant_ms_per_call']['tsqr'],3), {k:round(v['avg_launch_ms'],3) for k,v in d['roofline_by_kernel'].items()}, 'tree', round(d['kernel_share'].get('tsqr_tree',0)*d['ms_per_step'],3), d['clocks']['sm_mhz'])
"
    done
  done
done
