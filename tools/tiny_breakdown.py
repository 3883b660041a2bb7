"""Where the time of a configs[0] call goes: Python binding vs the C-ABI call vs device time."""
import ctypes, json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_13393_b200 import inputs, pqr
dv = torch.device("cuda", 0)
n, k, s = 10_000, 32, 4
Qh, Xh = inputs.tiny_inputs(n=n, k=k, s=s)
Q = torch.from_numpy(Qh.T.copy()).to(dv).t(); X = torch.from_numpy(Xh.T.copy()).to(dv).t()
out = {}
for v in ("cholqr2", "tsqr"):
    st = torch.cuda.Stream()
    U, P, N = inputs.colmajor_empty(n, s, dv), inputs.colmajor_empty(k, s, dv), inputs.colmajor_empty(s, s, dv)
    h = pqr.PQR(n, k, s, Q, variant=v, stream=st)
    L = pqr.lib()
    t = ctypes.c_int(0)
    args = (h.h, X.data_ptr(), n, s, pqr.PQR_NO_APPEND, U.data_ptr(), n, P.data_ptr(), k, N.data_ptr(), s, ctypes.byref(t))
    for _ in range(50):
        h.solve(X, U=U, P=P, N=N, flags=pqr.PQR_NO_APPEND)
    def tm(fn, it=500):
        ts = []
        for _ in range(it):
            t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
        return 1e6 * statistics.median(ts)
    res = {"python_solve_us": tm(lambda: h.solve(X, U=U, P=P, N=N, flags=pqr.PQR_NO_APPEND)),
           "cabi_call_us": tm(lambda: L.pqr_project_normalize(*args))}
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = []
    for _ in range(200):
        a.record(st); L.pqr_project_normalize(*args); b.record(st); b.synchronize(); ev.append(1e3 * a.elapsed_time(b))
    res["device_event_us"] = statistics.median(ev)
    out[v] = res
    h.close()
print(json.dumps(out))
