"""Worker bodies for the world-size-2 gloo tests (spawned processes; CPU only)."""
import os
import sys
import traceback

import numpy as np


def _setup(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"] = str(rank)
    os.environ["WORLD_SIZE"] = str(world)
    from paper_2204_13393_b200 import dist

    dist.init("gloo")
    return dist


def sharded_pqr_worker(rank, world, port, outdir):
    try:
        import torch.distributed as tdist

        import oracle
        from paper_2204_13393_b200 import inputs

        dist = _setup(rank, world, port)
        res = {}
        n, k, s = 4003, 24, 6
        # (1) row shards tile [0, n)
        offs = [dist.row_shard(n, world, r) for r in range(world)]
        res["shards_ok"] = offs[0][0] == 0 and all(offs[i][0] + offs[i][1] == offs[i + 1][0] for i in range(world - 1)) \
            and offs[-1][0] + offs[-1][1] == n
        off, nl = dist.row_shard(n, world, rank)
        # (2) library NCCL-id plumbing: a 128-byte token from rank 0 reaches every rank
        token = bytes(range(128)) if rank == 0 else None
        res["bcast_ok"] = dist.broadcast_bytes(token) == bytes(range(128))
        # global problem (every rank draws the same seeded matrices, keeps its shard)
        Q = inputs.orthonormal(7, n, k)
        X = inputs.projected_inputs(8, n, k, s, ratio=1e-1)[1]
        Qs, Xs = np.asfortranarray(Q[off:off + nl]), np.asfortranarray(X[off:off + nl])
        # (3) a1 + a2: per-shard Gram, allgather, fixed-order sum == full Gram; replicas identical
        Wsum, parts = dist.allgather_fixed_order_sum(oracle.gram(Qs, Xs))
        Wfull = oracle.gram(Q, X)
        res["gram_rel"] = float(np.linalg.norm(Wsum - Wfull) / np.linalg.norm(Wfull))
        chk, _ = dist.allgather_fixed_order_sum(Wsum)
        res["gram_replicated"] = bool(np.array_equal(chk, world * Wsum) or np.allclose(chk, world * Wsum, rtol=0, atol=0))
        # (4) a3 + a4 on the replicated W: N and this shard's U equal the full solve's
        N, t, piv = oracle.cholesky_deflate(Wsum, k)
        U_shard = oracle.update(Qs, Xs, Wsum[:k], N, t, piv)
        ref = oracle.bcgs_pip(Q, X)
        res["pip_N_rel"] = float(np.linalg.norm(N - ref["N"]) / np.linalg.norm(ref["N"]))
        res["pip_U_rel"] = float(np.linalg.norm(U_shard - ref["U"][off:off + nl]) / np.linalg.norm(ref["U"][off:off + nl]))
        # (5) TSQR cross-GPU level (reading R12): allgather each shard's R of [Q_g X_g]; the QR of
        # the stacked R's has the global R (up to row signs)
        A = np.asfortranarray(np.hstack([Qs, Xs]))
        V, rd = oracle.hh_local(A)
        m = k + s
        Rg = np.triu(V[:m])
        np.fill_diagonal(Rg, rd)
        _, Rparts = dist.allgather_fixed_order_sum(Rg)
        Rstack = np.vstack(Rparts)
        V2, rd2 = oracle.hh_local(Rstack)
        R2 = np.triu(V2[:m])
        np.fill_diagonal(R2, rd2)
        full = oracle.householder_pqr(Q, X)
        sg = np.sign(np.diag(R2))
        Rc = sg[:, None] * R2
        res["tsqr_P_rel"] = float(np.linalg.norm(Rc[:k, k:] - full["P"]) / np.linalg.norm(full["P"]))
        res["tsqr_N_rel"] = float(np.linalg.norm(Rc[k:, k:] - full["N"]) / np.linalg.norm(full["N"]))
        # (6) max over ranks (timing rule)
        res["max_ok"] = dist.max_over_ranks(float(rank + 1)) == float(world)
        tdist.barrier()
        tdist.destroy_process_group()
        np.save(os.path.join(outdir, f"rank{rank}.npy"), res, allow_pickle=True)
    except Exception:
        with open(os.path.join(outdir, f"rank{rank}.err"), "w") as f:
            f.write(traceback.format_exc())
        raise
