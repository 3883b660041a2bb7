# r02k: the column-graded TSQR tolerance test, then a randomised parity sweep of the final build
# (the sweep of r02_stress_parity_b predates the warp-specialised fused pass and the slot cap)
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_pqr.py -m gpu -q -k "deflation_small" > $O/r02k_deflation_tests.log 2>&1; echo "rc=$?" >> $O/r02k_deflation_tests.log
tail -15 $O/r02k_deflation_tests.log
timeout 1000 python tools/stress_parity.py 420 101 > $O/r02k_stress_parity_a.txt 2>&1; tail -3 $O/r02k_stress_parity_a.txt
timeout 1000 python tools/stress_parity.py 420 202 > $O/r02k_stress_parity_b.txt 2>&1; tail -3 $O/r02k_stress_parity_b.txt
