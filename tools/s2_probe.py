"""Probe: CholQR2 solve time over n (the fused pass uses the stream2 kernel), one size per process."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_13393_b200 import inputs, pqr
n, k, s = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dv = torch.device("cuda", 0)
Q = inputs.device_orthonormal(5, n, k, dv) if k else None
X = inputs.device_gaussian(6, n, s, dv)
U = inputs.colmajor_empty(n, s, dv)
h = pqr.PQR(n, k, s, Q, k=k, variant="cholqr2")
h.profile(True)
torch.cuda.synchronize()
t0 = time.time()
for _ in range(3):
    t = h.solve(X, U=U, flags=pqr.PQR_NO_APPEND)
torch.cuda.synchronize()
p = h.profile()
print(n, k, s, "t", t, "wall", round(time.time() - t0, 3), {kk: round(v["ms"] / max(1, v["launches"]), 3) for kk, v in p.items() if v["launches"]}, flush=True)
