# phase traces (PQR_WY_TRACE) of trace builds build/<v>/libpqr.so: the leaf k_wy_up launch of a workload
# usage: bash tools/tsqr_trace.sh WORKLOAD NBLOCKS v1 v2 ...
W=$1; NB=$2; shift 2
for v in "$@"; do
  PQR_LIB=$PWD/build/$v/libpqr.so PQR_WY_TRACE=1 timeout 300 python bench.py --workload $W --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 >/dev/null | grep "\"up\", \"nblocks\": $NB," | tail -1 | sed "s/^/$v /"
done
