# A/B of one kernel across variant builds (build/<v>/libpqr.so) under ncu with its default
# clock control (clocks locked to base: removes power-cap variance from the comparison).
# usage: tools/ncu_ab.sh KERNEL_REGEX VARIANT(cholqr2|tsqr) v1 v2 ...
kre=$1; var=$2; shift 2
for v in "$@"; do
  PQR_LIB=$PWD/build/$v/libpqr.so timeout 300 ncu --clock-control none -k "regex:$kre" -s 2 -c 3 --csv \
    --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum \
    python bench.py --variant $var --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null \
    | grep -E '^"[0-9]' | awk -F'","' -v v=$v '{print v, $5, $(NF-2), $NF}' | tr -d '"'
done
