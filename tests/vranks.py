"""Virtual ranks (pqr_vgroup_create): P library handles in this process on one GPU, each
driven from its own host thread and stream, exchanging their small matrices through device
copies instead of NCCL.  Marshalling helpers for the -m gpu tests only."""
import threading

import numpy as np

from gpu_util import dev, empty, host


def row_shard(n, world, rank):
    base = n // world
    return rank * base, base + (n - base * world if rank == world - 1 else 0)


def run(pqr, Q, X, nranks, variant, calls=None, k_max=None, s_max=None, apply_after=False, **kw):
    """Run the same sequence of solves on every virtual rank of a new group.

    Q (n x k, may have k = 0) and X (n x s) are global host arrays; rank r gets its
    contiguous row shard.  `calls`: list of (X_global, flags) (default one NO_APPEND solve of
    X).  Returns per rank: list of dicts (t, U shard, P, N) per call, stats, and (apply_after)
    the explicit basis shard from pqr_basis_apply(I)."""
    import torch

    n, k = Q.shape
    s = X.shape[1]
    calls = calls or [(X, pqr.PQR_NO_APPEND)]
    s_max = s_max or max(c[0].shape[1] for c in calls)
    k_max = k_max or k
    g = pqr.pqr_vgroup_create(nranks)
    out = [None] * nranks
    errs = []

    def worker(r):
        h = None
        try:
            torch.cuda.set_device(0)
            off, nl = row_shard(n, nranks, r)
            st = torch.cuda.Stream()
            Qd = dev(Q[off:off + nl]) if k else None
            Xs = [dev(c[0][off:off + nl]) for c in calls]
            torch.cuda.synchronize()
            h = pqr.PQR(nl, k_max, s_max, Qd, k=k, variant=variant, stream=st, rank=r, nranks=nranks, vgroup=g, **kw)
            res = []
            for (Xc, flags), Xd in zip(calls, Xs):
                sc = Xc.shape[1]
                kk = h.k
                U, Pm, Nm = empty(nl, sc), empty(max(kk, 1), sc), empty(sc, sc)
                t = h.solve(Xd, U=U, P=Pm if kk else None, N=Nm, flags=flags)
                st.synchronize()
                res.append(dict(t=t, U=host(U)[:, :t], P=host(Pm)[:kk], N=host(Nm)))
            basis = None
            if apply_after:
                kk = h.k
                V = empty(nl, kk)
                h.apply(dev(np.eye(kk)), kk, V)
                st.synchronize()
                basis = host(V)
            out[r] = dict(calls=res, stats=h.stats(), basis=basis)
        except Exception as e:  # pragma: no cover - reported below
            errs.append((r, e))
        finally:
            if h is not None:
                h.close()

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    pqr.pqr_vgroup_destroy(g)
    if errs:
        r, e = min(errs, key=lambda x: x[0])
        raise RuntimeError(f"virtual rank {r} failed: {e!r} (all: {errs!r})") from e
    return out


def gather_u(out, ci=0):
    return np.vstack([o["calls"][ci]["U"] for o in out])


def block_qr(pqr, A, s, nranks, variant, **kw):
    """Alg. 2 (block column QR) of the global host matrix A (n x m) on
    `nranks` virtual ranks: rank r holds its row shard and appends every block's U.  Returns
    the gathered n x k basis (host) and the t of each block."""
    import torch

    n, m = A.shape
    g = pqr.pqr_vgroup_create(nranks)
    out = [None] * nranks
    errs = []

    def worker(r):
        h = None
        try:
            torch.cuda.set_device(0)
            off, nl = row_shard(n, nranks, r)
            st = torch.cuda.Stream()
            Ad = dev(A[off:off + nl])
            Qd = empty(nl, m)
            torch.cuda.synchronize()
            h = pqr.PQR(nl, m, s, None, k=0, variant=variant, stream=st, rank=r, nranks=nranks, vgroup=g, **kw)
            k, ts = 0, []
            for b in range(0, m, s):
                w = min(s, m - b)
                t = h.solve(Ad[:, b:b + w], U=Qd[:, k:k + w], s=w)
                k += t
                ts.append(t)
            st.synchronize()
            out[r] = dict(Q=host(Qd)[:, :k], t=ts)
        except Exception as e:  # pragma: no cover
            errs.append((r, e))
        finally:
            if h is not None:
                h.close()

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    pqr.pqr_vgroup_destroy(g)
    if errs:
        r, e = min(errs, key=lambda x: x[0])
        raise RuntimeError(f"virtual rank {r} failed: {e!r} (all: {errs!r})") from e
    return np.vstack([o["Q"] for o in out]), out[0]["t"]
