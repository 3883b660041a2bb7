# A/B of whole default bench lines across variant builds (build/<v>/libpqr.so), interleaved twice;
# prints value, per-variant ms per call, median SM clock and power (the bench is power-capped)
for rep in 1 2; do for v in "$@"; do PQR_LIB=$PWD/build/$v/libpqr.so timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), d['variant_ms_per_call'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"; done; done
