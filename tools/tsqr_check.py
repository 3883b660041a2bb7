"""Quick GPU check (tuning aid): TSQR vs CholQR2 results on device inputs at several sizes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_13393_b200 import inputs, pqr


def run(n, k, s, variant, Q, X):
    U = inputs.colmajor_empty(n, s, "cuda")
    P = inputs.colmajor_empty(max(k, 1), s, "cuda")
    N = inputs.colmajor_empty(s, s, "cuda")
    with pqr.PQR(n, k, s, Q, variant=variant) as h:
        t = h.solve(X, U=U, P=P, N=N, flags=pqr.PQR_NO_APPEND)
    torch.cuda.synchronize()
    return t, U, P, N


for n, k, s in [(300_007, 64, 8), (1 << 20, 64, 8), (1 << 22, 64, 8), (1 << 22, 128, 8), (1 << 21, 96, 16)]:
    Q = inputs.device_orthonormal(11, n, k, "cuda")
    X = inputs.device_gaussian(12, n, s, "cuda")
    a = run(n, k, s, "cholqr2", Q, X)
    b = run(n, k, s, "tsqr", Q, X)
    r = lambda x, y: float((x - y).norm() / y.norm())
    print(n, k, s, "t", a[0], b[0], "P %.2e N %.2e U %.2e" % (r(b[2][:k], a[2][:k]), r(b[3], a[3]), r(b[1], a[1])), flush=True)
