#!/usr/bin/env python
"""Benchmark of the PQR hot path (BASELINE.json metric:
"PQR effective HBM GB/s (fraction of roofline) at 1/2/4/8 B200, fp64").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload weak|single|deflation|tiny]
                  [--variant cholqr2|tsqr|both] [--impl pqr|reference]

One step = one pqr_project_normalize call per selected variant (default: both, so a step
covers every row of SURVEY.md §8(a): CholQR2 a1-a5 and TSQR a6-a8) with PQR_NO_APPEND, so
the basis and all inputs are identical every step.  --workload arnoldi instead times the
32 PQR calls of one block-Arnoldi run (configs[2]; the stencil is timed separately).
Default workload = configs[4] ("weak": 2^25 rows per GPU, k=128, s=8), the config the
metric is quoted on at 1/2/4/8 GPUs; per-GPU work is fixed, so scaling is "weak".

value = whole-job effective GB/s = sum over ranks of the MANDATORY bytes of a call
(Q and X read once, U written once: 8 n_local (k + 2s)) x calls / max-over-ranks time.
--impl reference times the CPU oracle (oracle/, plain C fp64 Householder) on a bounded
row sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 2204133930
WORKLOADS = {
    "tiny": dict(n=10_000, k=32, s=4, cfg_index=0),
    "arnoldi": dict(n=256 ** 3, k=128, s=4, grid=256, steps=32, cfg_index=2),
    "single": dict(n=2 ** 24, k=64, s=8, cfg_index=1),
    "deflation": dict(n=2 ** 22, k=96, s=16, cfg_index=3),
    "weak": dict(n=2 ** 25, k=128, s=8, cfg_index=4),
}
METRIC = "PQR effective HBM GB/s (fraction of roofline) at 1/2/4/8 B200, fp64"


# The JSON line is the only thing this script writes to stdout: C-level output of the libraries
# (e.g. NCCL's version banner from the communicator the library builds) is redirected to
# stderr at start-up, and the line goes to a saved duplicate of the original stdout.
_JSON_FD = None


def _claim_stdout():
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line: dict):
    out = (json.dumps(line) + "\n").encode()
    os.write(_JSON_FD if _JSON_FD is not None else 1, out)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def mandatory_bytes(n, k, s):
    return 8.0 * n * (k + 2 * s)


# --------------------------------------------------------------------------
# clocks sampler (nvml) — runs during the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples = []
        self.power = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.hd = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.hd, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.hd, self.nv.NVML_CLOCK_SM))
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.hd) / 1000.0)
                fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    getattr(self.nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
                r = fn(self.hd)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        out = {"sm_mhz": statistics.median(self.samples), "sm_min_mhz": min(self.samples), "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.power:
            out["power_w"] = round(statistics.median(self.power), 1)
        return out


# --------------------------------------------------------------------------
# CPU oracle baseline (rank 0, bounded sample)
# --------------------------------------------------------------------------
def oracle_sample(w, target_s=15.0, max_rows=None):
    """Time the oracle (as it stands) on a row sample of the workload; returns (GB/s, info)."""
    import numpy as np

    import oracle
    from paper_2204_13393_b200 import inputs

    k, s = w["k"], w["s"]
    n_full = w["n"]
    # calibration run: large enough for the oracle's threads to scale as on the real sample
    rows = min(n_full, 2 ** 14 if target_s < 2 else 2 ** 17)
    Q = inputs.orthonormal(SEED + 11, rows, k)
    X = inputs.gaussian(SEED + 12, rows, s)
    t0 = time.perf_counter()
    oracle.householder_pqr(Q, X)
    dt = time.perf_counter() - t0
    # scale the sample to ~target_s seconds (the oracle is O(n) per call); at most 2^23 rows
    rows2 = int(min(n_full, 2 ** 23, max(rows, rows * target_s / max(dt, 1e-3) * 0.9)))
    if max_rows:
        rows2 = min(rows2, max_rows)
    if rows2 > rows:
        rows = rows2
        Q = inputs.orthonormal(SEED + 11, rows, k)
        X = inputs.gaussian(SEED + 12, rows, s)
        t0 = time.perf_counter()
        oracle.householder_pqr(Q, X)
        dt = time.perf_counter() - t0
    gbs = mandatory_bytes(rows, k, s) / dt / 1e9
    info = {"value": gbs, "unit": "GB/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"one Householder PQR of [Q X] with {rows} of the workload's {n_full} rows "
                      f"(k={k}, s={s}), {dt:.2f} s; GB/s = 8*rows*(k+2s)/time"}
    return gbs, info, dt


def host_info():
    """CPU model and core counts of the box (the oracle's machine)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def single_thread_oracle():
    """The oracle with one OpenMP thread (a subprocess: the thread count is fixed at load) on
    configs[0] in full and on a 2^18-row sample of configs[1]'s shape."""
    import subprocess

    code = ("import json,time,sys; sys.path.insert(0, %r)\n"
            "import oracle\nfrom paper_2204_13393_b200 import inputs\nout = {}\n"
            "for name, n, k, s in (('tiny', 10000, 32, 4), ('single_sample', 2**18, 64, 8)):\n"
            "    Q = inputs.orthonormal(7, n, k); X = inputs.gaussian(8, n, s)\n"
            "    t0 = time.perf_counter(); oracle.householder_pqr(Q, X); dt = time.perf_counter() - t0\n"
            "    out[name] = {'rows': n, 'k': k, 's': s, 'seconds': dt, 'GB/s': 8.0 * n * (k + 2 * s) / dt / 1e9}\n"
            "out['threads'] = oracle.num_threads()\nprint(json.dumps(out))\n") % ROOT
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                           env=dict(os.environ, OMP_NUM_THREADS="1"))
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    w = WORKLOADS[args.workload]
    _, info, dt1 = oracle_sample(w, target_s=min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    # the steps: repeat the same bounded sample
    import numpy as np

    import oracle
    from paper_2204_13393_b200 import inputs

    rows = int(info["sample"].split(" with ")[1].split(" of ")[0])
    Q = inputs.orthonormal(SEED + 11, rows, w["k"])
    X = inputs.gaussian(SEED + 12, rows, w["s"])
    for _ in range(args.warmup):
        oracle.householder_pqr(Q, X)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.householder_pqr(Q, X)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = mandatory_bytes(rows, w["k"], w["s"]) * args.steps / tot / 1e9
    info["value"] = val
    line = {"metric": METRIC, "value": val, "unit": "GB/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "n_local": w["n"], "k": w["k"], "s": w["s"],
                       "sample_rows": rows, "parallelism": f"dp{world}"},
            "cpu_baseline": info,
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="weak", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default="both", choices=["cholqr2", "tsqr", "both"])
    ap.add_argument("--impl", default="pqr", choices=["pqr", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-serial", action="store_true", help="e2e: the variants one after the other only")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "RANK" not in os.environ:
        world = 1
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2204_13393_b200 import inputs, pqr

    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=device)
    if args.workload == "arnoldi":
        return run_arnoldi(args, rank, world, local_rank, device)
    w = WORKLOADS[args.workload]
    n, k, s = w["n"], w["k"], w["s"]
    stream = torch.cuda.current_stream(device)

    # ---- inputs (seeded, synthetic, on the device) ----
    torch.cuda.synchronize()
    if args.workload == "weak":
        Q, X = inputs.device_weak_inputs(SEED + 4, n, k, s, device, rank=rank, world=world)
    elif args.workload == "single":
        Q, X = inputs.device_projected_inputs(SEED + 1, n, k, s, device)
    elif args.workload == "deflation":
        Q, X = inputs.device_deflation_inputs(SEED + 3, n, k, s, device)
    else:
        Qh, Xh = inputs.tiny_inputs(SEED, n, k, s)
        Q = torch.from_numpy(np.ascontiguousarray(Qh.T)).to(device).t()
        X = torch.from_numpy(np.ascontiguousarray(Xh.T)).to(device).t()
    U = inputs.colmajor_empty(n, s, device)
    Pm = inputs.colmajor_empty(k, s, device)
    Nm = inputs.colmajor_empty(s, s, device)
    torch.cuda.synchronize()

    from paper_2204_13393_b200 import dist as pdist

    # the weak workload is one global problem row-sharded over the ranks (the library's NCCL
    # exchange joins them); the other workloads run as independent replicas per rank
    sharded = args.workload == "weak" and world > 1
    variants = ["cholqr2", "tsqr"] if args.variant == "both" else [args.variant]
    handles = {}
    # one CUDA stream per variant's handle (the calls are host-synchronous, so the device loop
    # is sequential; the e2e leg runs the two handles from two host threads)
    hstreams = {v: torch.cuda.Stream(device) for v in variants}
    for v in variants:
        # one ncclUniqueId per communicator (each handle owns one)
        nccl_id = pdist.nccl_id_for_library(world) if sharded else None
        handles[v] = pqr.PQR(n, k, s, Q, variant=v, stream=hstreams[v], rank=rank if sharded else 0,
                             nranks=world if sharded else 1, nccl_id=nccl_id)
    del Q
    torch.cuda.empty_cache()

    var_ms = {v: 0.0 for v in variants}
    timing = {"on": False}

    def step():
        ts = []
        for v in variants:
            if timing["on"]:
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(hstreams[v])
            ts.append(handles[v].solve(X, U=U, P=Pm, N=Nm, flags=pqr.PQR_NO_APPEND))
            if timing["on"]:
                b.record(hstreams[v])
                b.synchronize()
                var_ms[v] += a.elapsed_time(b)
        return ts

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])

    for _ in range(args.warmup):
        t_vals = step()
    launches0 = sum(h.stats()["kernel_launches"] for h in handles.values())
    for h in handles.values():
        h.profile(True)
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    timing["on"] = True
    with ClockSampler(local_rank) as clk:
        ev0.record(hstreams[variants[0]])
        for _ in range(args.steps):
            t_vals = step()
        ev1.record(hstreams[variants[-1]])  # after the last (host-synchronous) call
        torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    launches = sum(h.stats()["kernel_launches"] for h in handles.values()) - launches0
    prof = {v: h.profile() for v, h in handles.items()}
    tmax = torch.tensor([ms], device=device, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    ms_step = ms_max / args.steps

    mand = mandatory_bytes(n, k, s) * world * len(variants)  # per step, whole job
    value = mand / (ms_step * 1e-3) / 1e9
    hbm, peak_kind = peaks()

    # ---- roofline of the dominant kernel (device events per launch, in the timed region) ----
    kinds = {}
    for v, p in prof.items():
        for kind, d in p.items():
            if d["launches"]:
                kk = kinds.setdefault(kind, dict(ms=0.0, launches=0))
                kk["ms"] += d["ms"]
                kk["launches"] += d["launches"]
    dom = max(kinds.items(), key=lambda kv: kv[1]["ms"])[0] if kinds else None
    per_launch_bytes = {
        "gram": 8.0 * n * (k + s),             # read Q, X (or Q, U1)
        "update": 8.0 * n * (k + s) + 8.0 * n * s,  # read Q, X; write U
        "update_gram": 8.0 * n * (k + s) + 8.0 * n * s,  # read Q, X; write U1 (W2 on chip)
        "tsqr_local": 8.0 * n * (k + s) + 8.0 * n * s,  # read Y (reflectors) and X, write new reflectors
        "tsqr_apply": 8.0 * n * (k + s) + 8.0 * n * s,  # read Y, write U
    }
    roof = None
    if dom in per_launch_bytes:
        avg_ms = kinds[dom]["ms"] / kinds[dom]["launches"]
        ach = per_launch_bytes[dom] / (avg_ms * 1e-3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tr = json.load(f)
            traffic = tr.get(f"{args.workload}:{dom}")
        except Exception:
            traffic = None
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": ach / hbm, "traffic": traffic, "algorithmic_bytes": per_launch_bytes[dom],
                "avg_launch_ms": avg_ms}
    # the same figure for every streaming kernel kind of the step (device events, this run's clocks)
    roof_all = {}
    for kd, d in kinds.items():
        if kd in per_launch_bytes and d["launches"]:
            am = d["ms"] / d["launches"]
            roof_all[kd] = {"avg_launch_ms": am, "achieved": per_launch_bytes[kd] / (am * 1e-3) / 1e9,
                            "frac": per_launch_bytes[kd] / (am * 1e-3) / 1e9 / hbm}
    share = {kd: (d["ms"] / (ms * 1.0)) for kd, d in kinds.items()}
    # north_star roofline: mandatory bytes / HBM + the measured latency of the small exchanges
    # (device time of the collectives in this run, per step; 0 on one GPU without NCCL)
    nccl_ms_step = kinds.get("nccl", {}).get("ms", 0.0) / args.steps
    t_roof = mandatory_bytes(n, k, s) / (hbm * 1e9) * 1e3 * len(variants) + nccl_ms_step
    frac_whole = t_roof / ms_step

    # ---- e2e through the C-ABI with HOST buffers (pinned), copies inside the timed region ----
    # Every step uploads X and downloads U (and P, N) per variant.  Default: the step's two
    # independent solves run from two host threads (one per variant), so one solve's U download
    # overlaps the other's X upload on the full-duplex link; "serial" runs them one after the
    # other (also reported).
    e2e = None
    if args.e2e_steps > 0:
        Xh = torch.empty((s, n), dtype=torch.float64, pin_memory=True).t()
        Xh.copy_(X)
        outs = {}
        for v in variants:
            outs[v] = (torch.empty((s, n), dtype=torch.float64, pin_memory=True).t(),
                       torch.empty((s, k), dtype=torch.float64, pin_memory=True).t(),
                       torch.empty((s, s), dtype=torch.float64, pin_memory=True).t())

        def solve_host(v):
            Uh, Ph, Nh = outs[v]
            handles[v].solve(Xh, U=Uh, P=Ph, N=Nh, flags=pqr.PQR_NO_APPEND)

        def run_serial(steps):
            for _ in range(steps):
                for v in variants:
                    solve_host(v)

        def run_threads(steps):
            errs = []

            def worker(v):
                try:
                    torch.cuda.set_device(local_rank)  # a new host thread starts on device 0
                    for _ in range(steps):
                        solve_host(v)
                except Exception as e:  # pragma: no cover
                    errs.append(e)

            ths = [threading.Thread(target=worker, args=(v,)) for v in variants]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            if errs:
                raise errs[0]

        def timed(fn):
            fn(1)  # warm-up (staging buffers, copy streams)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(args.e2e_steps)
            torch.cuda.synchronize()
            dt = torch.tensor([time.perf_counter() - t0], device=device, dtype=torch.float64)
            if world > 1:
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            return float(dt.item()) / args.e2e_steps

        serial_step = timed(run_serial)
        # (sharded runs stay serial: two NCCL communicators driven from two threads could
        # interleave their collectives differently on different ranks)
        conc = len(variants) > 1 and not args.e2e_serial and not sharded
        e2e_step = timed(run_threads) if conc else serial_step
        e2e = {"value": mand / e2e_step / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": 8 * n * s * len(variants),
               "d2h_bytes_per_step": (8 * n * s + 8 * k * s + 8 * s * s) * len(variants),
               "ms_per_step": e2e_step * 1e3,
               "mode": "concurrent: one host thread per variant" if conc else "serial",
               "serial": {"value": mand / serial_step / 1e9, "ms_per_step": serial_step * 1e3}}
        del Xh, outs

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            _, cpu, _ = oracle_sample(w, target_s=25.0)
            cpu.update(host_info())
            cpu["single_thread"] = single_thread_oracle()
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "error": str(e)}

    for h in handles.values():
        h.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "baseline_config": w["cfg_index"], "n_local": n, "k": k, "s": s,
                       "global_rows": n * world if sharded or world == 1 else n, "variants": variants,
                       "parallelism": f"dp{world}" if sharded or world == 1 else f"replicas{world}",
                       "l2": "inputs exceed L2 (no flush needed)" if mandatory_bytes(n, k, s) > 2 * 126e6
                       else "inputs fit in L2 (latency-bound config)",
                       "t": t_vals},
            "frac_of_roofline": frac_whole,
            "roofline_terms_ms": {"hbm": t_roof - nccl_ms_step, "nccl": nccl_ms_step},
            "roofline": roof,
            "roofline_by_kernel": roof_all,
            "kernel_share": share,
            "variant_ms_per_call": {v: var_ms[v] / args.steps for v in variants},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_arnoldi(args, rank, world, local_rank, device):
    """configs[2]: block Arnoldi on the 256^3 7-point Laplacian, s = 4, 32 PQR calls with
    k = 4..128 (after the k = 0 start).  Each rank runs its own replica (the Arnoldi operator
    is not sharded here: "replicas only" for this workload).  Timed: the PQR calls only."""
    import torch
    import torch.distributed as dist

    from paper_2204_13393_b200 import arnoldi, inputs, pqr
    from paper_2204_13393_b200 import dist as pdist

    w = WORKLOADS["arnoldi"]
    g, s, steps = w["grid"], w["s"], w["steps"]
    n = g ** 3
    stream = torch.cuda.current_stream(device)
    R = inputs.device_gaussian(SEED + 2 + 1000 * rank, n, s, device)
    variants = ["cholqr2", "tsqr"] if args.variant == "both" else [args.variant]
    acc = {"pqr": 0.0, "op": 0.0}
    evs = []

    def timer(kind, fn):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = fn()
        b.record(stream)
        evs.append((kind, a, b))
        return r

    def one_step(prof=False):
        out = {}
        for v in variants:
            res = arnoldi.block_arnoldi(g, g, g, R, steps, variant=v, stream=stream, timer=timer, profile=prof)
            out[v] = (res["t_list"], res["h"].profile() if prof else None)
            res["h"].close()
        return out

    for _ in range(args.warmup):
        one_step()
    evs.clear()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        profs = [one_step(prof=True) for _ in range(args.steps)]
        torch.cuda.synchronize()
    for kind, a, b in evs:
        acc[kind] += a.elapsed_time(b)
    pqr_ms = pdist.max_over_ranks(acc["pqr"] / args.steps, device)
    op_ms = acc["op"] / args.steps
    # mandatory bytes of the calls: k = 0 (start), then k = 4, 8, ..., 4*steps
    mand = sum(mandatory_bytes(n, k, s) for k in range(0, s * steps + 1, s)) * len(variants) * world
    value = mand / (pqr_ms * 1e-3) / 1e9
    hbm, peak_kind = peaks()
    kinds = {}
    for pr in profs:
        for v, (tl, p) in pr.items():
            for kind, d in (p or {}).items():
                if d["launches"]:
                    kk = kinds.setdefault(kind, dict(ms=0.0, launches=0))
                    kk["ms"] += d["ms"]
                    kk["launches"] += d["launches"]
    tot = sum(d["ms"] for d in kinds.values()) or 1.0
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": pqr_ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "arnoldi", "baseline_config": 2, "grid": g, "n_local": n, "s": s,
                           "pqr_calls": steps + 1, "k_range": [0, s * steps], "variants": variants,
                           "parallelism": f"replicas{world}", "operator_ms_per_step": op_ms,
                           "pqr_plus_operator_ms_per_step": pqr_ms + op_ms,
                           "l2": "inputs exceed L2 (no flush needed)"},
                "frac_of_roofline": (mand / world / (hbm * 1e9) * 1e3) / pqr_ms,
                "kernel_share": {k: d["ms"] / tot for k, d in kinds.items()},
                "cpu_baseline": None, "e2e": None,
                "gpu_launches": sum(d["launches"] for d in kinds.values()) // max(1, args.steps),
                "clocks": clk.summary()}
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    _claim_stdout()
    sys.exit(main())
