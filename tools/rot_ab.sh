# TSQR leaf kernels of A/B builds with chains off and on (weak): usage: bash tools/rot_ab.sh v1 v2 ...
for c in off on; do for v in "$@"; do
  PQR_CHAINS=$c PQR_LIB=$PWD/build/$v/libpqr.so timeout 200 python bench.py --workload ${W:-weak} --variant tsqr --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v chains=$c', round(d['variant_ms_per_call']['tsqr'],3), {k:round(v['avg_launch_ms'],3) for k,v in d['roofline_by_kernel'].items()}, 'tree', round(d['kernel_share'].get('tsqr_tree',0)*d['ms_per_step'],3))
"
done; done
