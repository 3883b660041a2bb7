timeout 600 python -m pytest tests/test_gpu_nccl_path.py -x -q > gpurun_out/r02g_nccl.log 2>&1; echo nccl_rc=$?
tail -30 gpurun_out/r02g_nccl.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream2" -s 1 -c 1 -o gpurun_out/r02g_fused python bench.py --variant cholqr2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02g_fused.log 2>&1; echo ncu_rc=$?
python tools/ncu_summary.py gpurun_out/r02g_fused.ncu-rep > gpurun_out/r02g_fused_ncu.json 2>&1
ncu -i gpurun_out/r02g_fused.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py 40 > gpurun_out/r02g_fused_lines.txt
ncu -i gpurun_out/r02g_fused.ncu-rep --page raw --csv > gpurun_out/r02g_fused_raw.csv 2>/dev/null
rm -f gpurun_out/r02g_fused.ncu-rep
