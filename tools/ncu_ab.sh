# A/B of one kernel across variant builds (build/<v>/libpqr.so) under ncu, clocks unlocked
# (single serialised launches draw less power than the bench's steady state).
# usage: tools/ncu_ab.sh KERNEL_REGEX VARIANT(cholqr2|tsqr) MIN_MS v1 v2 ...   (prints launches >= MIN_MS)
kre=$1; var=$2; minms=$3; shift 3
for v in "$@"; do
  PQR_LIB=$PWD/build/$v/libpqr.so timeout 300 ncu --clock-control none -k "regex:$kre" -s ${SKIP:-0} -c 30 --csv \
    --metrics gpu__time_duration.sum \
    python bench.py --variant $var --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null \
    | grep -E '^"[0-9]' | python3 -c "
import csv, sys
for r in csv.reader(sys.stdin):
    unit, val = r[-2], float(r[-1].replace(',', ''))
    ms = val * {'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1.0}.get(unit, 1e-6)
    if ms >= $minms: print('$v', r[4][:40], round(ms, 4))
"
done
