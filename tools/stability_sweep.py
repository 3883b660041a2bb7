"""fig:kappa analogue on B200: block column QR (Alg. 2) of Stewart
matrices n = 2^16, m = 64, s = 4 for kappa = 1 .. 1e16 with single-pass BCGS-PIP, BCGS-PIP+
(CholQR2) and TreeTSPQR (Householder local + reduction, 256-row leaves).  Prints one JSON
object per (kappa, variant): e_perp = ||I - Q^T Q||_F (Eq. (4)), residual ||A - QR||_F/||A||_F,
total rank t, and the wall time of the QR."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2204_13393_b200 import blockqr, inputs

N, M, S = 1 << 16, 64, 4
for lk in range(0, 17, 2):
    kappa = 10.0 ** lk
    Ah = inputs.stewart(100 + lk, N, M, kappa)
    A = torch.from_numpy(np.ascontiguousarray(Ah.T)).cuda().t()
    for name, kw in (("bcgs_pip", dict(variant="cholqr2", single_pass=True)),
                     ("bcgs_pip_plus", dict(variant="cholqr2")),
                     ("tsqr_hh", dict(variant="tsqr", block_rows=256, defl_tol=1e-300))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = blockqr.block_column_qr(A, S, **kw)
        dt = time.perf_counter() - t0
        e = blockqr.orthogonality_loss(out["Q"])
        r = blockqr.residual(A, out["Q"], out["R"])
        print(json.dumps(dict(kappa=kappa, variant=name, e_perp=e, residual=r, rank=int(sum(out["t_list"])),
                              ms=round(dt * 1e3, 2))), flush=True)
