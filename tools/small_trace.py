"""Phase timestamps (globaltimer, CTA 0) of the one-launch small CholQR2 kernel (trace build:
tools/build_variant.py smalltrace -DPQR_SMALL_TRACE; run with PQR_LIB=build/smalltrace/libpqr.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_13393_b200 import inputs, pqr
dv = torch.device("cuda", 0)
n, k, s = 10_000, 32, 4
Qh, Xh = inputs.tiny_inputs(n=n, k=k, s=s)
Q = torch.from_numpy(Qh.T.copy()).to(dv).t(); X = torch.from_numpy(Xh.T.copy()).to(dv).t()
U, P, N = inputs.colmajor_empty(n, s, dv), inputs.colmajor_empty(k, s, dv), inputs.colmajor_empty(s, s, dv)
lib = pqr.lib()
from cuda.bindings import runtime as rt  # noqa
with pqr.PQR(n, k, s, Q, variant="cholqr2") as h:
    for _ in range(5):
        h.solve(X, U=U, P=P, N=N, flags=pqr.PQR_NO_APPEND)
    torch.cuda.synchronize()
err, ptr = rt.cudaGetSymbolAddress if False else (None, None)
# read the trace through a tiny exported helper-free path: cudaMemcpyFromSymbol needs the symbol; use the
# module's device variable via cuModuleGetGlobal is not exposed -> the trace build exports pqr_small_trace()
buf = (ctypes.c_ulonglong * 16)()
lib.pqr_small_trace.argtypes = [ctypes.c_void_p]
lib.pqr_small_trace(buf)
t = [buf[i] for i in range(14)]
print({f"phase{i}": (t[i] - t[0]) / 1000.0 for i in range(9)})
print("last factor_body (pass 2), us from its start:", [(t[9 + i] - t[9]) / 1000.0 for i in range(5)])
