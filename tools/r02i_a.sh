O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > $O/r02i_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02i_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r02i_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r02i_smoke.log
timeout 600 python bench.py > $O/r02i_bench.json 2> $O/r02i_bench.err
tail -3 $O/r02i_pytest.log; tail -2 $O/r02i_smoke.log; head -c 600 $O/r02i_bench.json
