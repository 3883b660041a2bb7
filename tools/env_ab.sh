# timing A/B over environment knobs of the CholQR2 kernels (weak config)
for envs in "" "PQR_FUSE_CTAS=1" "PQR_NO_FUSE=1"; do
  env $envs timeout 120 python bench.py --variant cholqr2 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$envs]', d['variant_ms_per_call'], {k:round(v*d['ms_per_step'],3) for k,v in d['kernel_share'].items()}, d['clocks']['sm_mhz'])"
done
