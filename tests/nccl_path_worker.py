"""Run in a subprocess with PQR_FORCE_NCCL=1: single-rank handles that still build their NCCL
communicator and run every cross-GPU step (Gram allgathers, the replicated cross-GPU TSQR
node).  Prints one JSON line with the errors against the oracle and the collective counters."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from gpu_util import dev, empty, host, rel  # noqa: E402
from paper_2204_13393_b200 import inputs, pqr  # noqa: E402

exchange = os.environ.get("PQR_TEST_EXCHANGE", "collective")
out = {}
n, k, s = 300_007, 64, 8
Q = inputs.orthonormal(5, n, k)
X = inputs.gaussian(6, n, s)
ref = oracle.householder_pqr(Q, X)
Xd = dev(X)
for variant, kw in (("cholqr2", {}), ("tsqr", {}), ("tsqr_pip2", dict(reduction="pip2"))):
    U, Pm, Nm = empty(n, s), empty(k, s), empty(s, s)
    with pqr.PQR(n, k, s, dev(Q), variant=variant.split("_")[0], exchange=exchange, **kw) as h:
        # three calls: the device-API exchange alternates its window halves (odd exchange counts)
        res = []
        for _ in range(3):
            t = h.solve(Xd, U=U, P=Pm, N=Nm, flags=pqr.PQR_NO_APPEND)
            res.append((t, host(U), host(Pm), host(Nm)))
        st = h.stats()
    torch.cuda.synchronize()
    same = all(np.array_equal(a, b) for r in res[1:] for a, b in zip(r[1:], res[0][1:]))
    out[variant] = dict(t=res[0][0], P=rel(res[0][2], ref["P"]), N=rel(res[0][3], ref["N"]),
                        U=rel(res[0][1], ref["U"]), collectives=int(st["collectives"]), exchange=int(st["exchange"]),
                        repeat_bitwise=bool(same))
    if os.environ.get("PQR_TEST_DUMP"):
        np.savez(os.environ["PQR_TEST_DUMP"] + f"_{variant}.npz", U=res[0][1], P=res[0][2], N=res[0][3])
print(json.dumps(out))
