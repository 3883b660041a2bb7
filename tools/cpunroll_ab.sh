# A/B of the slot-copy issue loop's unroll factor in the fused CholQR2 pass (variant libraries
# build/cpuN/libpqr.so = -DPQR_S2_CPUNROLL=N, tools/build_variant.py) against the in-tree library.
O=gpurun_out/cpunroll_ab.txt
run() {  # workload lib env...
  w=$1; lib=$2; shift 2
  env PQR_LIB=$lib "$@" timeout 300 python bench.py --workload $w --variant cholqr2 --steps 8 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/_ab.json 2>/dev/null
  python -c "
import json
d = json.load(open('gpurun_out/_ab.json'))
r = d.get('roofline_by_kernel') or {}
print('$w', '$lib', '$*', round(d['value'], 1), round(d['ms_per_step'], 3), {k: (round(v['avg_launch_ms'], 3), round(v['frac'], 3)) for k, v in r.items()}, d['clocks']['sm_mhz'])
" >> $O
}
D=paper_2204_13393_b200/libpqr.so
for rep in 1 2; do
  run weak $D
  for u in 2 4 8; do run weak build/cpu$u/libpqr.so; done
  run weak $D PQR_S2_LOOP=0
done
for u in 0 2 4 8; do
  lib=build/cpu$u/libpqr.so; [ $u = 0 ] && lib=$D
  run single $lib
  run single $lib PQR_S2_IL=0
  run deflation $lib
done
cat $O
