# correctness + timing of the fused CholQR2 pass variants (PQR_FUSE_PAIR=1 pair form, 0 block form)
timeout 300 python -m pytest tests -m gpu -x -q -k "cholqr" 2>&1 | tail -2
for v in 1 0; do PQR_FUSE_PAIR=$v timeout 120 python bench.py --variant cholqr2 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pair=$v', d['config']['t'], d['variant_ms_per_call'], {k:round(v*d['ms_per_step'],3) for k,v in d['kernel_share'].items()}, d['clocks']['sm_mhz'])"; done
