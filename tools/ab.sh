# A/B correctness+timing of alternative libpqr builds (build/<v>/libpqr.so)
for v in "$@"; do PQR_LIB=$PWD/build/$v/libpqr.so timeout 300 python bench.py --variant tsqr --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['t'], d['variant_ms_per_call'], d['kernel_share'])"; done
