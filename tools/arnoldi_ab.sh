# Arnoldi workload A/B of libpqr builds ("cur" = in-tree): per-kernel-kind ms per step
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = cur ]; then LIB=""; else LIB=$PWD/build/$v/libpqr.so; fi
  PQR_LIB=$LIB timeout 300 python bench.py --workload arnoldi --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); T=d['ms_per_step']
print('$v', round(T,1), 'op', round(d['config']['operator_ms_per_step'],1), {k: round(v*T,1) for k,v in d['kernel_share'].items()}, d['clocks']['sm_mhz'])
"
done; done
