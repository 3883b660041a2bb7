# A/B of the warp-specialised fused CholQR2 pass (PQR_S2_WS) + its parity tests; gpurun_out/ws_ab.txt
O=gpurun_out
rm -f $O/ab1.txt
AB_WL=weak AB_CFGS="PQR_S2_WS=1;PQR_S2_WS=0;PQR_S2_WS=1;PQR_S2_WS=0" bash tools/ab_s2.sh
cat $O/ab1.txt
grep -q "weak PQR_S2_WS=1 FAILED" $O/ab1.txt && exit 3
AB_WL=single AB_CFGS="PQR_S2_WS=0;PQR_S2_WS=1" bash tools/ab_s2.sh
AB_WL=deflation AB_CFGS="PQR_S2_WS=0;PQR_S2_WS=1" bash tools/ab_s2.sh
mv $O/ab1.txt $O/ws_ab.txt; cat $O/ws_ab.txt
PQR_S2_WS=1 timeout 600 python -m pytest tests/test_gpu_pqr.py tests/test_gpu_cholqr.py tests/test_gpu_fullsize.py -q -x > $O/ws_pytest.log 2>&1; echo "pytest rc=$?" >> $O/ws_pytest.log
tail -2 $O/ws_pytest.log
