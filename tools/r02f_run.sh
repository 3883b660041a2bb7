set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02f_pytest.log 2>&1; echo pytest_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo smoke_rc=$?
bash tools/profile_round.sh r02f; echo prof_rc=$?
for w in tiny single deflation arnoldi; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r02f_bench_$w.json 2> gpurun_out/r02f_bench_$w.err; echo $w rc=$?; done
