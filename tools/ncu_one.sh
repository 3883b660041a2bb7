# one ncu --set full capture of the first launch (after SKIP) of kernels matching REGEX in CMD
# usage: bash tools/ncu_one.sh TAG REGEX SKIP CMD...
TAG=$1; RX=$2; SKIP=$3; shift 3
timeout 600 "$@" > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed" >> gpurun_out/${TAG}_plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SKIP -c 1 -o gpurun_out/${TAG} "$@" > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}.ncu-rep > gpurun_out/${TAG}_summary.json 2> gpurun_out/${TAG}_summary.err
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py 40 > gpurun_out/${TAG}_lines.txt
