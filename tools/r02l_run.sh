# r02l: last validation of the final sources — smoke(), the whole GPU suite, the default bench
# line, the stability sweep and the heatmap on the final build
O=gpurun_out
timeout 300 python __graft_entry__.py smoke > $O/r02l_smoke.log 2>&1; echo "rc=$?" >> $O/r02l_smoke.log; tail -2 $O/r02l_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/r02l_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02l_pytest.log; tail -3 $O/r02l_pytest.log
timeout 600 python bench.py > $O/r02l_bench.json 2> $O/r02l_bench.err; head -c 300 $O/r02l_bench.json
timeout 600 python tools/stability_sweep.py > $O/r02l_stability_sweep.jsonl 2> $O/r02l_stab.err; tail -n 3 $O/r02l_stability_sweep.jsonl
timeout 900 python tools/heatmap.py > $O/r02l_heatmap.jsonl 2> $O/r02l_heat.err; tail -n 1 $O/r02l_heatmap.jsonl | head -c 400
