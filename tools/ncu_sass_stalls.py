"""Per-SASS-instruction stall breakdown from `ncu -i REP --page source --csv --print-source sass` (tuning aid).
usage: python tools/ncu_sass_stalls.py REP [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
out = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        v = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    st = {k[6:]: int(d[k]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k and d[k].isdigit() and int(d[k]) > 0}
    out.append((v, d["Address"], d["Source"][:60], sorted(st.items(), key=lambda x: -x[1])[:3]))
tot = sum(o[0] for o in out) or 1
out.sort(key=lambda o: -o[0])
for v, a, s, st in out[:n]:
    print("%5.1f%% %s %-60s %s" % (100.0 * v / tot, a, s, st))
