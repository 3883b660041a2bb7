"""Block Arnoldi (Alg. 1) on top of the PQR library — the consumer of
BASELINE configs[2] (7-point Laplacian on a 256^3 grid, s = 4, 32 block iterations).

    V_0 = R H_0                         (PQR with k = 0)
    for i = 0..steps-1:
        X_{i+1} = A V_i                 (pqr_laplacian7_apply)
        [V X] = [V V_{i+1}] [I P; 0 N]  (pqr_project_normalize, appending V_{i+1})
        H_{i+1} = [H_i P; 0 N]

Every step runs in libpqr kernels; this module only sequences the calls and assembles the
(small, host) block-Hessenberg H.
"""
from __future__ import annotations

import numpy as np


def block_arnoldi(nx, ny, nz, R, steps, variant="cholqr2", device="cuda", stream=None, timer=None, profile=False):
    """Run Alg. 1.  R: n x s column-major device tensor.  Returns dict(H, k, t_list, handle_stats,
    V_last) and keeps the basis in the handle (returned open as 'h' for further queries).

    `timer`, if given, is called as timer('pqr'|'op', fn) to time each library call."""
    import torch

    from . import inputs, pqr

    n = nx * ny * nz
    s = R.shape[1]
    h = pqr.PQR(n, steps * s, s, None, k=0, variant=variant, stream=stream)
    if profile:
        h.profile(True)
    run = timer or (lambda kind, fn: fn())
    U = inputs.colmajor_empty(n, s, device)
    Nb = inputs.colmajor_empty(s, s, device)
    Pb = inputs.colmajor_empty(max(1, steps * s), s, device)
    X = inputs.colmajor_empty(n, s, device)
    t0 = run("pqr", lambda: h.solve(R, U=U, N=Nb))
    H0 = Nb.cpu().numpy()[:t0]
    H = np.zeros(((steps + 1) * s, steps * s))
    k = t0
    t_list = [t0]
    width = t0
    for i in range(steps):
        if width == 0:
            break
        run("op", lambda: pqr.pqr_laplacian7_apply(nx, ny, nz, width, U[:, :width], X[:, :width], stream=stream))
        Pk = Pb[:k] if k > 0 else None
        t = run("pqr", lambda: h.solve(X[:, :width], U=U, P=Pk, N=Nb, s=width))
        if k > 0:
            H[:k, i * s:i * s + width] = Pb[:k].cpu().numpy()[:, :width]
        H[k:k + t, i * s:i * s + width] = Nb.cpu().numpy()[:t, :width]
        k += t
        t_list.append(t)
        width = t
    torch.cuda.synchronize()
    return dict(H=H[:k, :sum(t_list[:-1])], H0=H0, k=k, t_list=t_list, h=h, V_last=U)
