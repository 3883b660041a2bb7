"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) over the last N library
launches (the timed steps of bench.py; setup/input-generation launches are dropped)."""
import collections, csv, sys

path, nlast = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 60
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
lib = []
for r in rows[start + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum" or "pqr::" not in r[ki]:
        continue
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] == "us" else (v / 1e6 if r[ui] == "ns" else v)
    lib.append((r[ki].split("(")[0].replace("void ", "").replace("pqr::", ""), v))
lib = lib[-nlast:]
agg = collections.OrderedDict()
for name, v in lib:
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print("kernel,launches,total_ms,avg_ms,share")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k},{n},{t:.3f},{t / n:.4f},{t / tot:.4f}")
