"""Randomised parity sweep (tuning/validation aid, not part of the suite): random (n, k, s,
variant, leaf block size, grid size), device buffers, against the CPU oracle.  Usage:
python tools/stress_parity.py SECONDS [SEED]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2204_13393_b200 import inputs, pqr  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


def host(t):
    return t.t().contiguous().cpu().numpy().T


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    t0 = time.time()
    cases = fails = 0
    while time.time() - t0 < budget:
        variant = ["cholqr2", "tsqr"][rng.integers(2)]
        s = int(rng.integers(1, 17))
        k = int(rng.integers(0, 120))
        n = int(rng.integers(max(1000, 2 * (k + s + 16)), 200_000))
        br = int(rng.choice([0, 0, 512, 768, 1024])) if variant == "tsqr" else 0
        if br and br < 2 * (k + s + 16):
            br = 0
        sms = str(int(rng.choice([0, 2, 3, 17])))
        if sms != "0":
            os.environ["PQR_SMS"] = sms
        else:
            os.environ.pop("PQR_SMS", None)
        seed = int(rng.integers(1 << 30))
        Q = inputs.orthonormal(seed, n, k)
        X = inputs.gaussian(seed + 1, n, s)
        try:
            U = torch.empty((s, n), dtype=torch.float64, device="cuda").t()
            Pm = torch.empty((s, max(k, 1)), dtype=torch.float64, device="cuda").t()
            Nm = torch.empty((s, s), dtype=torch.float64, device="cuda").t()
            with pqr.PQR(n, k, s, dev(Q) if k else None, k=k, variant=variant, block_rows=br) as h:
                t = h.solve(dev(X), U=U, P=Pm, N=Nm, flags=pqr.PQR_NO_APPEND)
            torch.cuda.synchronize()
            ref = oracle.householder_pqr(Q, X)
            e = max(rel(host(U)[:, :t], ref["U"]), rel(host(Nm), ref["N"]),
                    rel(host(Pm)[:k], ref["P"]) if k else 0.0)
            ok = t == ref["t"] and e < 1e-10
        except Exception as ex:  # noqa: BLE001
            ok, e, t = False, str(ex), None
            if "block plan" in e and br > 512 and s > 8:
                continue  # documented: 16-wide panels need leaf blocks of <= 512 rows
        cases += 1
        if not ok:
            fails += 1
            print("FAIL", dict(variant=variant, n=n, k=k, s=s, block_rows=br, sms=sms, seed=seed, t=t, err=e), flush=True)
    print(f"stress_parity: {cases} cases, {fails} failures, {time.time() - t0:.0f} s")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
