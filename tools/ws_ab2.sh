O=gpurun_out
rm -f $O/ab1.txt
AB_WL=weak AB_CFGS="PQR_S2_WS=0;PQR_S2_WS=1 PQR_S2_NSL=12;PQR_S2_WS=1 PQR_S2_NSL=9;PQR_S2_WS=0 PQR_S2_NSL=12;PQR_S2_WS=1;PQR_S2_WS=0" bash tools/ab_s2.sh
AB_WL=single AB_CFGS="PQR_S2_WS=0;PQR_S2_WS=1 PQR_S2_NSL=12;PQR_S2_WS=1 PQR_S2_NSL=16" bash tools/ab_s2.sh
AB_WL=deflation AB_CFGS="PQR_S2_WS=0;PQR_S2_WS=1;PQR_S2_WS=1 PQR_S2_NSL=12" bash tools/ab_s2.sh
mv $O/ab1.txt $O/ws_ab2.txt; cat $O/ws_ab2.txt
