# A/B of the G-phase tile-group separator (PQR_S2_GBAR) and the run-time k test (PQR_S2_KTEST) of
# the fused pass: in-tree (GBAR=2, KTEST=0) vs build/base (previous build), gbar0, gbar1, kt1.
O=gpurun_out/gbar_ab.txt
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
N=paper_2204_13393_b200/libpqr.so
for rep in 1 2; do
  for lib in build/base/libpqr.so $N build/gbar1/libpqr.so build/kt1/libpqr.so; do run weak $lib; done
done
run weak build/gbar0/libpqr.so
for lib in build/base/libpqr.so $N build/kt1/libpqr.so; do run single $lib; run deflation $lib; done
cat $O
PQR_LIB=$N timeout 900 python -m pytest tests/test_gpu_cholqr.py tests/test_gpu_pqr.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/gbar_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gbar_tests.log
tail -3 gpurun_out/gbar_tests.log
