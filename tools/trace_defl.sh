# phase traces of the TSQR level kernels on the deflation config (s = 16), trace build
PQR_LIB=$PWD/build/vtrace/libpqr.so PQR_WY_TRACE=1 timeout 300 python bench.py --workload deflation --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_defl.json 2> gpurun_out/trace_defl.err
grep -c wy_trace gpurun_out/trace_defl.err; grep -v wy_trace gpurun_out/trace_defl.err | tail -5
