# A/B of the deferred refill of the fused CholQR2 pass (PQR_S2_DEFER): each setting runs the
# cholqr2-only bench; the line shows value, ms/step, per-kernel (ms, frac), SM clock.
# usage: bash tools/defer_ab.sh [OUT]
O=${1:-gpurun_out/defer_ab.txt}
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
# correctness first: the CholQR2 GPU tests with the option forced on
PQR_S2_DEFER=1 timeout 900 python -m pytest tests/test_gpu_cholqr.py tests/test_gpu_pqr.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/defer_tests.log 2>&1; echo "rc=$?" >> gpurun_out/defer_tests.log
tail -3 gpurun_out/defer_tests.log
for rep in 1 2; do
  run weak PQR_S2_DEFER=0
  run weak PQR_S2_DEFER=1
  run weak PQR_S2_DEFER=1 PQR_S2_NSL=13
  run weak PQR_S2_DEFER=1 PQR_S2_NSL=11
done
run single PQR_S2_DEFER=0
run single PQR_S2_IL=0 PQR_S2_DEFER=0
run single PQR_S2_IL=0 PQR_S2_DEFER=1
run single PQR_S2_IL=0 PQR_S2_DEFER=1 PQR_S2_NSL=16
run deflation PQR_S2_DEFER=0
run deflation PQR_S2_WS=0 PQR_S2_IL=0 PQR_S2_DEFER=1
run deflation PQR_S2_WS=0 PQR_S2_DEFER=0
cat $O
