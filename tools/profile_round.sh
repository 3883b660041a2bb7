# Round evidence: bench line, launch list (cold/serialised) and one ncu --set full capture of
# the dominant kernel (leaf stage-1 TSQR kernel), all for the default bench command.
# usage: bash tools/profile_round.sh TAG
TAG=${1:-r}
B="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err || exit 1
timeout 300 $B > gpurun_out/${TAG}_bench_short.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wy_up -s 119 -c 1 -o gpurun_out/${TAG}_wy_up python bench.py --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_wy_up.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream2|k_gram_cpa|k_update_cpa" -s 3 -c 3 -o gpurun_out/${TAG}_cholqr python bench.py --variant cholqr2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_cholqr.log 2>&1
# leaf stage-2 launch: the first k_wy_down launch of the timed step that runs > 3 ms
T="python bench.py --variant tsqr --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_wy_down $T 2>/dev/null > gpurun_out/${TAG}_down_list.csv
SKIP=$(python - gpurun_out/${TAG}_down_list.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5 and r[0].isdigit()]
ms = [float(r[-1].replace(",", "")) for r in rows]
unit = rows[0][-2] if rows else "ns"
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
big = [i for i, v in enumerate(ms) if v * scale > 3.0]
print(big[-1] if big else 0)
PY
)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wy_down -s $SKIP -c 1 -o gpurun_out/${TAG}_wy_down $T > gpurun_out/${TAG}_wy_down.log 2>&1
# summaries on the box (the .ncu-rep files are large: gpurun copies back <= 64 MiB)
python tools/ncu_summary.py gpurun_out/${TAG}_wy_up.ncu-rep gpurun_out/${TAG}_wy_down.ncu-rep gpurun_out/${TAG}_cholqr.ncu-rep > gpurun_out/${TAG}_ncu_full.json 2> gpurun_out/${TAG}_ncu_summary.err
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.csv 2>/dev/null
for k in wy_up wy_down; do
  ncu -i gpurun_out/${TAG}_$k.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py 40 > gpurun_out/${TAG}_${k}_lines.txt
done
rm -f gpurun_out/${TAG}_cholqr.ncu-rep gpurun_out/${TAG}_launches.csv
ls -la gpurun_out | grep ${TAG}
