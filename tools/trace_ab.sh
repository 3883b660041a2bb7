# phase traces (leaf level of k_wy_up) of alternative trace builds build/<v>/libpqr.so, TSQR variant, weak config
for v in "$@"; do
  PQR_LIB=$PWD/build/$v/libpqr.so PQR_WY_TRACE=1 timeout 300 python bench.py --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 >/dev/null | grep '"up", "nblocks": 32768' | tail -1 | sed "s/^/$v /"
done
