"""Per-call latency of configs[0] (n = 10,000, k = 32, s = 4) through the C-ABI with device buffers
and PQR_NO_APPEND: median over many calls, both variants (PQR_NO_GRAPH=1 disables graph replay)."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2204_13393_b200 import inputs, pqr
dv = torch.device("cuda", 0)
n, k, s = 10_000, 32, 4
Qh, Xh = inputs.tiny_inputs(n=n, k=k, s=s)
Q = torch.from_numpy(Qh.T.copy()).to(dv).t()
X = torch.from_numpy(Xh.T.copy()).to(dv).t()
out = {}
for v in ("cholqr2", "tsqr"):
    U, P, N = inputs.colmajor_empty(n, s, dv), inputs.colmajor_empty(k, s, dv), inputs.colmajor_empty(s, s, dv)
    with pqr.PQR(n, k, s, Q, variant=v) as h:
        for _ in range(20):
            h.solve(X, U=U, P=P, N=N, flags=pqr.PQR_NO_APPEND)
        ts = []
        for _ in range(300):
            t0 = time.perf_counter()
            h.solve(X, U=U, P=P, N=N, flags=pqr.PQR_NO_APPEND)
            ts.append(time.perf_counter() - t0)
        st = h.stats()
    out[v] = {"us_median": 1e6 * statistics.median(ts), "us_min": 1e6 * min(ts), "launches_per_call": None}
out["graph"] = os.environ.get("PQR_NO_GRAPH") is None
print(json.dumps(out))
