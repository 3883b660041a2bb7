# phase traces (CTA 0, group 0) of the leaf k_wy_up / k_wy_down launches with chains off / on
# usage: bash tools/chains_trace.sh TRACEBUILD [WORKLOAD]
for c in off on; do
  PQR_CHAINS=$c PQR_LIB=$PWD/build/$1/libpqr.so PQR_WY_TRACE=1 timeout 300 python bench.py --workload ${2:-weak} --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 >/dev/null | python -c "
import json, sys
last = {}
for line in sys.stdin:
    if 'wy_trace' not in line: continue
    d = json.loads(line)
    key = d['wy_trace']
    if key not in last or d['nblocks'] >= last[key]['nblocks']: last[key] = d
for k, d in last.items():
    print('chains=$c', k, d['nblocks'], d['rows'], 'w0', d['w0'][:14], 'sum', sum(d['w0']))
"
done
