O=gpurun_out
rm -f $O/ab1.txt
AB_WL=weak AB_CFGS="PQR_S2_NSL=13;PQR_S2_NSL=12;PQR_S2_NSL=11;PQR_S2_NSL=10;PQR_S2_NSL=13;PQR_S2_NSL=12;PQR_S2_NSL=13;PQR_S2_NSL=12" bash tools/ab_s2.sh
AB_WL=deflation AB_CFGS="PQR_S2_NSL=15 PQR_S2_WS=0;PQR_S2_NSL=12 PQR_S2_WS=0;PQR_S2_NSL=15;PQR_S2_NSL=12;PQR_S2_NSL=8" bash tools/ab_s2.sh
AB_WL=single AB_CFGS="PQR_S2_NSL=24;PQR_S2_NSL=16;PQR_S2_NSL=20;PQR_S2_NSL=12" bash tools/ab_s2.sh
mv $O/ab1.txt $O/nsl_ab.txt; cat $O/nsl_ab.txt
