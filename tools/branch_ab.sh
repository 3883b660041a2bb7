# A/B of the fused pass with its run-time options compiled out of the MMA stream (in-tree library)
# against the previous build (build/base/libpqr.so), after the CholQR2 parity tests.
O=gpurun_out/branch_ab.txt
timeout 900 python -m pytest tests/test_gpu_cholqr.py tests/test_gpu_pqr.py tests/test_gpu_fullsize.py tests/test_gpu_vranks.py -m gpu -q -x > gpurun_out/branch_tests.log 2>&1; echo "rc=$?" >> gpurun_out/branch_tests.log
tail -3 gpurun_out/branch_tests.log
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
N=paper_2204_13393_b200/libpqr.so; B=build/base/libpqr.so
for rep in 1 2 3; do run weak $B; run weak $N; done
run weak $N PQR_S2_NSL=13
run weak $N PQR_S2_NSL=11
for w in single deflation arnoldi; do run $w $B; run $w $N; done
run single $N PQR_S2_IL=0
run deflation $N PQR_S2_WS=0
run deflation $B PQR_S2_WS=0
cat $O
