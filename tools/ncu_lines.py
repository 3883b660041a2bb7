"""Per-source-line stall samples from `ncu --page source --csv --print-source cuda,sass` (tuning aid)."""
import csv, sys
rows = list(csv.reader(sys.stdin))
out, cur_file = [], None
tot = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) > 5 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            v = int(r[4])
        except ValueError:
            continue
        out.append((v, cur_file, r[0], r[1].strip()[:100]))
        tot += v
out.sort(reverse=True)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for v, f, l, src in out[:n]:
    print("%5.1f%% %s:%s  %s" % (100.0 * v / tot, f, l, src))
