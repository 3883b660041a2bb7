"""Block Arnoldi (Alg. 1) on top of the PQR library — the consumer of
BASELINE configs[2] (7-point Laplacian on a 256^3 grid, s = 4, 32 block iterations).

    V_0 = R H_0                         (PQR with k = 0)
    for i = 0..steps-1:
        X_{i+1} = A V_i                 (pqr_laplacian7_apply)
        [V X] = [V V_{i+1}] [I P; 0 N]  (pqr_project_normalize, appending V_{i+1})
        H_{i+1} = [H_i P; 0 N]

Every step runs in libpqr kernels on the device; this module only sequences the calls.  The
block-Hessenberg H lives on the device: each call writes its P and N straight into their
slices of H (column offset = the columns of H filled so far, row offset = the basis width),
so the loop moves no matrix data to the host — the one host value per call is the rank t
that pqr_project_normalize returns.
"""
from __future__ import annotations


def block_arnoldi(nx, ny, nz, R, steps, variant="cholqr2", device="cuda", stream=None, timer=None, profile=False):
    """Run Alg. 1.  R: n x s column-major device tensor.  Returns dict(H, H_dev, H0, k, t_list,
    h, V_last): H_dev is the k x (columns filled) block-Hessenberg matrix on the device (H a
    host copy taken after the loop), the basis stays in the handle `h` (returned open).

    `timer`, if given, is called as timer('pqr'|'op', fn) to time each library call."""
    import numpy as np
    import torch

    from . import inputs, pqr

    n = nx * ny * nz
    s = R.shape[1]
    h = pqr.PQR(n, steps * s, s, None, k=0, variant=variant, stream=stream)
    if profile:
        h.profile(True)
    run = timer or (lambda kind, fn: fn())
    U = inputs.colmajor_empty(n, s, device)
    X = inputs.colmajor_empty(n, s, device)
    H0 = inputs.colmajor_empty(s, s, device)
    Hd = inputs.colmajor_empty((steps + 1) * s, max(1, steps * s), device)
    Hd.zero_()
    t0 = run("pqr", lambda: h.solve(R, U=U, N=H0))
    k = t0
    c0 = 0          # columns of H filled so far (a deflated step adds width < s columns)
    t_list = [t0]
    width = t0
    for _ in range(steps):
        if width == 0:
            break
        run("op", lambda: pqr.pqr_laplacian7_apply(nx, ny, nz, width, U[:, :width], X[:, :width], stream=stream))
        Pk = Hd[:k, c0:c0 + width] if k > 0 else None
        Nk = Hd[k:k + width, c0:c0 + width]
        t = run("pqr", lambda: h.solve(X[:, :width], U=U, P=Pk, N=Nk, s=width))
        c0 += width
        k += t
        t_list.append(t)
        width = t
    torch.cuda.synchronize()
    H_dev = Hd[:k, :c0]
    return dict(H=np.asfortranarray(H_dev.cpu().numpy()), H_dev=H_dev, H0=H0[:t0].cpu().numpy(), k=k,
                t_list=t_list, h=h, V_last=U)
