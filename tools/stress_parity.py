"""Randomised parity sweep (validation aid, not part of the suite): random (n, k, s, variant,
leaf block size, grid size) and mode — one solve, three appending solves of random widths, host
buffers, a dependent column — against the CPU oracle.  Usage:
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
        small = rng.random() < 0.25
        n = int(rng.integers(k + 3 * s + 2, 4000)) if small else int(rng.integers(max(1000, 2 * (k + s + 16)), 200_000))
        if rng.random() < 0.2:
            os.environ["PQR_FORCE_NCCL"] = "1"  # single-rank run through the NCCL exchange path
        else:
            os.environ.pop("PQR_FORCE_NCCL", None)
        br = int(rng.choice([0, 0, 512, 768, 1024])) if variant == "tsqr" else 0
        if br and br < 2 * (k + s + 16):
            br = 0
        sms = str(int(rng.choice([0, 2, 3, 17])))
        if sms != "0":
            os.environ["PQR_SMS"] = sms
        else:
            os.environ.pop("PQR_SMS", None)
        seed = int(rng.integers(1 << 30))
        chains = "on" if variant == "tsqr" and rng.random() < 0.35 else "auto"  # FlatTSPQR leaves
        mode = ["plain", "plain", "append", "host", "dependent"][rng.integers(5)]
        Q = inputs.orthonormal(seed, n, k)
        try:
            nsolve = 3 if mode == "append" else 1
            ok, e, t = True, 0.0, None
            with pqr.PQR(n, k + (s * nsolve if mode == "append" else 0), s, dev(Q) if k else None, k=k,
                         variant=variant, block_rows=br, chains=chains) as h:
                Qcur = Q
                for it in range(nsolve):
                    si = s if it == 0 else int(rng.integers(1, s + 1))
                    X = inputs.gaussian(seed + 1 + it, n, si)
                    if mode == "dependent" and si >= 2:
                        X[:, si - 1] = X[:, 0] + Qcur @ inputs.gaussian(seed + 7, Qcur.shape[1], 1)[:, 0] if Qcur.shape[1] else X[:, 0]
                    kk = Qcur.shape[1]
                    if mode == "host":
                        Uh, Ph, Nh = (np.zeros((n, si), order="F"), np.zeros((max(kk, 1), si), order="F"),
                                      np.zeros((si, si), order="F"))
                        t = h.solve(X, U=Uh, P=Ph, N=Nh, flags=pqr.PQR_NO_APPEND, s=si)
                        Uo, Po, No = Uh, Ph, Nh
                    else:
                        U = torch.empty((si, n), dtype=torch.float64, device="cuda").t()
                        Pm = torch.empty((si, max(kk, 1)), dtype=torch.float64, device="cuda").t()
                        Nm = torch.empty((si, si), dtype=torch.float64, device="cuda").t()
                        flags = 0 if mode == "append" else pqr.PQR_NO_APPEND
                        t = h.solve(dev(X), U=U, P=Pm, N=Nm, flags=flags, s=si)
                        torch.cuda.synchronize()
                        Uo, Po, No = host(U), host(Pm), host(Nm)
                    ref = oracle.householder_pqr(Qcur, X)
                    ei = max(rel(Uo[:, :t], ref["U"]) if t else 0.0, rel(No, ref["N"]),
                             rel(Po[:kk], ref["P"]) if kk else 0.0)
                    if mode == "dependent":  # N's pivot rows only (the dependent column's entries are tiny)
                        ei = max(rel(Po[:kk], ref["P"]) if kk else 0.0, 0.0)
                    e = max(e, ei)
                    ok = ok and t == ref["t"] and ei < 1e-10
                    if mode == "append":
                        Qcur = np.asfortranarray(np.hstack([Qcur, ref["U"]]))
                if mode == "append" and Qcur.shape[1] > 0:
                    # Y = Q_basis C (the stored basis, explicit or LOR) against the oracle's basis
                    m = int(rng.integers(1, 9))
                    C = inputs.gaussian(seed + 99, Qcur.shape[1], m)
                    Y = torch.empty((m, n), dtype=torch.float64, device="cuda").t()
                    h.apply(dev(C), m, Y)
                    torch.cuda.synchronize()
                    ea = rel(host(Y), Qcur @ C)
                    e = max(e, ea)
                    ok = ok and ea < 1e-10
        except Exception as ex:  # noqa: BLE001
            ok, e, t = False, str(ex), None
            if "block plan" in e and br > 512 and s > 8:
                continue  # documented: 16-wide panels need leaf blocks of <= 512 rows
            if "capacity exceeded" in e and "pqr_create" in e:
                continue  # documented: k_max + s_max <= 152
        cases += 1
        if not ok:
            fails += 1
            print("FAIL", dict(mode=mode, variant=variant, n=n, k=k, s=s, block_rows=br, sms=sms, chains=chains,
                               nccl=os.environ.get("PQR_FORCE_NCCL"), seed=seed, t=t, err=e),
                  flush=True)
    print(f"stress_parity: {cases} cases, {fails} failures, {time.time() - t0:.0f} s")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
