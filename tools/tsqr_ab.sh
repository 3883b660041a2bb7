# Interleaved A/B of libpqr builds (build/<v>/libpqr.so; "cur" = the in-tree library) on the TSQR
# variant: per-call time, leaf kernels, tree.  usage: bash tools/tsqr_ab.sh "weak deflation" v1 v2 ...
WLS=$1; shift
for rep in 1 2; do
  for w in $WLS; do
    for v in "$@"; do
      if [ "$v" = cur ]; then LIB=""; else LIB=$PWD/build/$v/libpqr.so; fi
      PQR_LIB=$LIB timeout 200 python bench.py --workload $w --variant tsqr --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$w', round(d['variant_ms_per_call']['tsqr'],3), {k:round(v['avg_launch_ms'],3) for k,v in d['roofline_by_kernel'].items()}, 'tree', round(d['kernel_share'].get('tsqr_tree',0)*d['ms_per_step'],3), d['clocks']['sm_mhz'])
"
    done
  done
done
