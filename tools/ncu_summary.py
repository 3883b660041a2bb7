"""Key metrics of every kernel in an ncu --set full report (json to stdout)."""
import csv, io, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second"]
out = {}
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] + " grid " + r[hdr.index("launch__grid_size")]
        d = {}
        for k in KEYS:
            if k in hdr:
                d[k] = [r[hdr.index(k)], units[hdr.index(k)]]
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if v > 0:
                    stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = v
        tot = sum(stalls.values()) or 1.0
        d["stall_samples_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
        out[name] = d
json.dump(out, sys.stdout, indent=1)
