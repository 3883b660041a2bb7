# chained-kernel ablation timings (stage 2 and stage 1 leaf kernels, weak config, chains on)
for v in "$@"; do
  PQR_CHAINS=on PQR_LIB=$PWD/build/$v/libpqr.so timeout 200 python bench.py --workload weak --variant tsqr --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', {k:round(v['avg_launch_ms'],3) for k,v in d['roofline_by_kernel'].items()})
"
done
