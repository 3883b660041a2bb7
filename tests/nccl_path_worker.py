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

out = {}
n, k, s = 300_007, 64, 8
Q = inputs.orthonormal(5, n, k)
X = inputs.gaussian(6, n, s)
ref = oracle.householder_pqr(Q, X)
for variant in ("cholqr2", "tsqr"):
    U, Pm, Nm = empty(n, s), empty(k, s), empty(s, s)
    with pqr.PQR(n, k, s, dev(Q), variant=variant) as h:
        t = h.solve(dev(X), U=U, P=Pm, N=Nm, flags=pqr.PQR_NO_APPEND)
        st = h.stats()
    torch.cuda.synchronize()
    out[variant] = dict(t=t, P=rel(host(Pm), ref["P"]), N=rel(host(Nm), ref["N"]), U=rel(host(U), ref["U"]),
                        collectives=int(st["collectives"]))
print(json.dumps(out))
