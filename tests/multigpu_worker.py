"""torchrun worker of tests/test_gpu_multigpu.py: one process per GPU, the library's NCCL
exchange, one global problem row-sharded over the ranks; rank 0 prints a JSON line."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

from gpu_util import dev, empty, host, rel  # noqa: E402
from paper_2204_13393_b200 import dist, inputs, pqr  # noqa: E402

rank, world, local = dist.env_rank_world()
torch.cuda.set_device(local)
dist.init("nccl", torch.device("cuda", local))
n, k, s = 200_003, 64, 8
Q = inputs.orthonormal(5, n, k)
X = inputs.gaussian(6, n, s)
off, nl = dist.row_shard(n, world, rank)
out = {}
for variant in ("cholqr2", "tsqr"):
    nid = dist.nccl_id_for_library(world)
    U, Pm, Nm = empty(nl, s), empty(k, s), empty(s, s)
    with pqr.PQR(nl, k, s, dev(Q[off:off + nl]), variant=variant, rank=rank, nranks=world, nccl_id=nid) as h:
        t = h.solve(dev(X[off:off + nl]), U=U, P=Pm, N=Nm, flags=pqr.PQR_NO_APPEND)
    torch.cuda.synchronize()
    parts = [None] * world
    tdist.all_gather_object(parts, dict(t=t, U=host(U)[:, :t], P=host(Pm), N=host(Nm)))
    if rank == 0:
        import oracle

        ref = oracle.householder_pqr(Q, X)
        Ug = np.vstack([p["U"] for p in parts])
        out[variant] = dict(t=[p["t"] for p in parts], P=rel(parts[0]["P"], ref["P"]), N=rel(parts[0]["N"], ref["N"]),
                            U=rel(Ug, ref["U"]),
                            replicated=all(np.array_equal(p["P"], parts[0]["P"]) and np.array_equal(p["N"], parts[0]["N"])
                                           for p in parts))
if rank == 0:
    print(json.dumps(out))
tdist.destroy_process_group()
