# ncu --set full of the TSQR leaf kernels of the timed step of the weak bench (leaf stage 1 = the
# 58th launch of the mangled <4,1,8,0,2,0> kernel: 16 LOR-build sweeps + 3 warm-up solves x 3
# levels of that shape; leaf stage 2 = the 12th of <4,1,8,2,0>).  usage: bash tools/ncu_tsqr_leaf.sh TAG
TAG=$1; O=gpurun_out
T="python bench.py --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_wy_upILi4ELi1ELi8ELb0ELi2ELb0" -s 57 -c 1 -o $O/${TAG}_wy_up $T > $O/${TAG}_wy_up.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_wy_downILi4ELi1ELi8ELi2ELb0" -s 11 -c 1 -o $O/${TAG}_wy_down $T > $O/${TAG}_wy_down.log 2>&1
python tools/ncu_summary.py $O/${TAG}_wy_up.ncu-rep $O/${TAG}_wy_down.ncu-rep > $O/${TAG}_ncu_tsqr.json 2> $O/${TAG}_ncu_summary.err
for k in wy_up wy_down; do
  ncu -i $O/${TAG}_$k.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py 40 > $O/${TAG}_${k}_lines.txt
done
rm -f $O/${TAG}_*.ncu-rep
