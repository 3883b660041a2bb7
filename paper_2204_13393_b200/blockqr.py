"""Block column QR (Alg. 2) on top of the PQR library — the driver of the
paper's stability experiments (§6, fig:kappa, Table 1).

    for each s-column block A_i of A (left to right):
        [Q A_i] = [Q U_i] [I P_i; 0 N_i]     (pqr_project_normalize, appending U_i)
        R[:, block i] = [P_i; N_i]

so A = Q R with Q the accumulated basis.  Every step runs in libpqr kernels (either variant,
or single-pass BCGS-PIP with PQR_SINGLE_PASS); this module only sequences the calls and
collects the small R blocks.  Reading G8 (Alg. 2's loop indices): block i
covers columns i*s .. i*s+s-1, i = 0 .. m/s - 1.
"""
from __future__ import annotations

import numpy as np


def block_column_qr(A, s, variant="cholqr2", single_pass=False, block_rows=0, defl_tol=0.0, gram_eta=0.0,
                    stream=None):
    """A: n x m column-major fp64 device tensor.  Returns dict(Q (n x k device tensor),
    R (k x m host array), t_list, stats).  Deflated columns (t < s) leave zero rows in R."""
    import torch

    from . import inputs, pqr

    n, m = A.shape
    dev = A.device
    Q = inputs.colmajor_empty(n, m, dev)
    R = np.zeros((m, m))
    Pb = inputs.colmajor_empty(max(1, m), s, dev)
    Nb = inputs.colmajor_empty(s, s, dev)
    flags = pqr.PQR_SINGLE_PASS if single_pass else 0
    t_list = []
    k = 0
    with pqr.PQR(n, m, s, None, k=0, variant=variant, block_rows=block_rows, defl_tol=defl_tol,
                 gram_eta=gram_eta, stream=stream) as h:
        for b in range(0, m, s):
            w = min(s, m - b)
            t = h.solve(A[:, b:b + w], U=Q[:, k:k + w], P=Pb[:max(k, 1)] if k > 0 else None, N=Nb, flags=flags, s=w)
            if k > 0:
                R[:k, b:b + w] = Pb[:k, :w].cpu().numpy()
            R[k:k + t, b:b + w] = Nb[:t, :w].cpu().numpy()
            k += t
            t_list.append(t)
        stats = h.stats()
    if stream is None:
        torch.cuda.synchronize()
    return dict(Q=Q[:, :k], R=R[:k], t_list=t_list, stats=stats)


def orthogonality_loss(Q):
    """e_perp = ||I - Q^T Q||_F (Eq. (4)), fp64 on the device."""
    import torch

    G = Q.t() @ Q
    return float(torch.linalg.matrix_norm(torch.eye(G.shape[0], dtype=G.dtype, device=G.device) - G))


def residual(A, Q, R):
    """||A - Q R||_F / ||A||_F (Table 1 header; normalisation per SPEC S:L293)."""
    import torch

    Rd = torch.as_tensor(R, dtype=A.dtype, device=A.device)
    return float(torch.linalg.matrix_norm(A - Q @ Rd) / torch.linalg.matrix_norm(A))
