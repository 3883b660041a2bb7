# A/B of the G-phase tile group (PQR_S2_TG) and U-phase chains (PQR_S2_UCH) with and without the
# run-time k test (PQR_S2_KTEST): variant libraries build/<name>/libpqr.so vs the in-tree library.
O=gpurun_out/tg_ab.txt
run() {  # workload lib
  w=$1; lib=$2
  env PQR_LIB=$lib timeout 300 python bench.py --workload $w --variant cholqr2 --steps 8 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/_ab.json 2>/dev/null
  python -c "
import json
d = json.load(open('gpurun_out/_ab.json'))
r = d.get('roofline_by_kernel') or {}
print('$w', '$lib', round(d['value'], 1), round(d['ms_per_step'], 3), {k: (round(v['avg_launch_ms'], 3), round(v['frac'], 3)) for k, v in r.items()}, d['clocks']['sm_mhz'])
" >> $O
}
N=paper_2204_13393_b200/libpqr.so
for rep in 1 2; do
  run weak $N
  for v in kt0tg1 kt0tg4 kt1tg1 kt1tg4 kt0uc4; do run weak build/$v/libpqr.so; done
done
for v in kt1tg1 kt1tg4; do run single build/$v/libpqr.so; run deflation build/$v/libpqr.so; done
run single $N; run deflation $N
cat $O
