"""Small PQR calls for compute-sanitizer (memcheck / racecheck / synccheck): both variants,
several blocks per CTA (run with PQR_SMS=2 so the two-group TSQR kernels are exercised),
merge path (s = 4 twice) and host buffers."""
import numpy as np
import torch

from paper_2204_13393_b200 import inputs, pqr

n, k = 6 * 1024 + 37, 16
Q = inputs.orthonormal(5, n, k)
for variant in ("tsqr", "cholqr2"):
    h = pqr.PQR(n, k + 24, 8, torch.from_numpy(np.ascontiguousarray(Q.T)).cuda().t(), k=k, variant=variant)
    for s in (8, 4, 4):
        X = inputs.gaussian(10 + s, n, s)
        U = np.zeros((n, s), order="F")
        t = h.solve(X, U=U, s=s)
        assert t == s, (variant, s, t)
    h.close()
torch.cuda.synchronize()
print("sanitize_small ok")
