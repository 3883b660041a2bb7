O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $O/r02i_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02i_pytest.log
tail -2 $O/r02i_pytest.log
for e in "PQR_S2_NSL=0" "" "PQR_S2_NSL=0" ""; do
  env $e timeout 300 python bench.py --workload arnoldi --steps 3 --warmup 3 --no-cpu-baseline > $O/arn_ab.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/arn_ab.json')); print('arnoldi [$e]', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" >> $O/arn_ab.txt
done
cat $O/arn_ab.txt
timeout 600 python bench.py > $O/r02i_bench.json 2> $O/r02i_bench.err
timeout 600 python bench.py --workload deflation --no-cpu-baseline > $O/r02i_bench_deflation.json 2>> $O/r02i_bench.err
head -c 400 $O/r02i_bench.json
