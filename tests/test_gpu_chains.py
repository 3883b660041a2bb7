"""FlatTSPQR leaf chains (§4.2, Alg. 10; pqr_config.chains):
chained leaf blocks solve [Q_i | P_{i-1}; N_{i-1}; X_i] and only the chains' last blocks reach
the tree.  Checked against the CPU oracle on every call of appending sequences (panel merges,
s = 16 rounds, deflation), against the pure tree (chains off) to rounding, through the host-buffer
pipeline (chunks are whole chain rounds; stage 2 walks them backwards), and for bitwise
reproducibility.  Grids are sized for 2-3 SMs (PQR_SMS) so that chains hold many blocks at
test sizes."""
import numpy as np
import pytest

from gpu_util import dev, empty, host, ortho_loss_2, rel
from paper_2204_13393_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_13393_b200 import pqr

    pqr.lib()
    return pqr


def run_sequence(P, orc, n, k0, widths, chains, seed, s_max=None, check=True):
    """Appending solves of the given widths; every call checked against the oracle on the growing
    basis.  Returns the per-call (U, P, N, t), the handle's stats and Y = Q_final (basis_apply)."""
    import torch

    s_max = s_max or max(widths)
    Q = inputs.orthonormal(seed, n, k0)
    outs = []
    with P.PQR(n, k0 + sum(widths), s_max, dev(Q), k=k0, variant="tsqr", chains=chains) as h:
        Qcur = Q
        for i, s in enumerate(widths):
            X = inputs.gaussian(seed + 1 + i, n, s)
            kc = h.k
            U, Pm, Nm = empty(n, s), empty(max(1, kc), s), empty(s, s)
            t = h.solve(dev(X), U=U, P=Pm, N=Nm, s=s)
            torch.cuda.synchronize()
            out = dict(U=host(U)[:, :t], P=host(Pm)[:kc], N=host(Nm), t=t)
            if check:
                ref = orc.householder_pqr(Qcur, X)
                assert t == ref["t"]
                assert rel(out["P"], ref["P"]) < 1e-10 and rel(out["N"], ref["N"]) < 1e-10
                assert rel(out["U"], ref["U"]) < 1e-10
                assert ortho_loss_2(dev(Qcur), U[:, :t]) < 1e-12
                Qcur = np.asfortranarray(np.hstack([Qcur, ref["U"]]))
            outs.append(out)
        st = h.stats()
        k = h.k
        Y = empty(n, k)
        h.apply(dev(np.eye(k)), k, Y)
        torch.cuda.synchronize()
    return outs, st, host(Y), Qcur


@pytest.mark.parametrize("sms", ["2", "3"])
@pytest.mark.parametrize("n,k0,widths", [
    (23 * 1024 + 41, 24, (8, 4, 4, 8)),   # 4-wide panels merged into one 8-wide panel
    (60_013, 0, (8, 8, 8)),               # basis built from nothing, odd n
    (31_000, 16, (16, 9, 16)),            # 16-column rounds (512-row blocks), ragged s
])
def test_chains_vs_oracle(P, orc, sms, n, k0, widths, monkeypatch):
    monkeypatch.setenv("PQR_SMS", sms)
    outs, st, Y, Qfin = run_sequence(P, orc, n, k0, widths, "on", 300 + n % 97)
    assert st["leaf_chains"] == 2 * int(sms)
    # the representation reproduces the basis it stores (LOR apply, stage 2 along the chains)
    assert rel(Y, Qfin) < 1e-10
    # bitwise reproducible (fixed chain and tree order, R7)
    outs2, _, _, _ = run_sequence(P, orc, n, k0, widths, "on", 300 + n % 97, check=False)
    for a, b in zip(outs, outs2):
        assert np.array_equal(a["U"], b["U"]) and np.array_equal(a["N"], b["N"])


@pytest.mark.parametrize("n,k0,widths,block_rows", [(138_329, 60, (1, 1), 512), (47_223, 21, (6, 6), 512),
                                                    (60_001, 30, (16, 3), 256)])
def test_chains_user_block_rows(P, orc, n, k0, widths, block_rows, monkeypatch):
    """Chains with a user leaf size below the kernel's register capacity: the chained blocks' carried
    pivot rows must still fit behind their own rows (regression: a 512-row leaf on an 8-column handle
    overlapped them; found by tools/stress_parity.py)."""
    import torch

    monkeypatch.setenv("PQR_SMS", "2")
    Q = inputs.orthonormal(801 + n % 7, n, k0)
    Qcur = Q
    with P.PQR(n, k0 + sum(widths), max(widths), dev(Q), k=k0, variant="tsqr", chains="on",
               block_rows=block_rows) as h:
        assert h.stats()["leaf_chains"] == 4
        for i, s in enumerate(widths):
            X = inputs.gaussian(810 + i, n, s)
            U, Pm, Nm = empty(n, s), empty(Qcur.shape[1], s), empty(s, s)
            t = h.solve(dev(X), U=U, P=Pm, N=Nm, s=s)
            torch.cuda.synchronize()
            ref = orc.householder_pqr(Qcur, X)
            assert t == ref["t"]
            assert rel(host(Pm), ref["P"]) < 1e-10 and rel(host(Nm), ref["N"]) < 1e-10
            assert rel(host(U)[:, :t], ref["U"]) < 1e-10
            Qcur = np.asfortranarray(np.hstack([Qcur, ref["U"]]))


@pytest.mark.parametrize("n,k0,widths", [(40_000, 32, (8, 8)), (33_333, 20, (12, 4))])
def test_chains_vs_tree(P, orc, n, k0, widths, monkeypatch):
    """Chains on and off are two locally orthogonal representations of the same basis: P, N, t and
    U agree to rounding on every call."""
    monkeypatch.setenv("PQR_SMS", "2")
    on, st_on, _, _ = run_sequence(P, orc, n, k0, widths, "on", 400, check=False)
    off, st_off, _, _ = run_sequence(P, orc, n, k0, widths, "off", 400, check=False)
    assert st_on["leaf_chains"] == 4 and st_off["leaf_chains"] == 0
    for a, b in zip(on, off):
        assert a["t"] == b["t"]
        for key in ("U", "P", "N"):
            assert rel(a[key], b[key]) < 1e-12, key


def test_chains_deflation(P, orc, monkeypatch):
    """A dependent column (X[:, 3] = Q c + X[:, 0] - 2 X[:, 1]) deflates at the top (t = s - 1) with
    the chained leaves, as in the oracle (reading R3)."""
    import torch

    monkeypatch.setenv("PQR_SMS", "2")
    n, k, s = 45_000, 40, 8
    Q = inputs.orthonormal(501, n, k)
    X = inputs.gaussian(502, n, s)
    X[:, 3] = Q @ inputs.gaussian(503, k, 1)[:, 0] + X[:, 0] - 2.0 * X[:, 1]
    X = np.asfortranarray(X)
    ref = orc.householder_pqr(Q, X)
    assert ref["t"] == s - 1
    U, Pm, Nm = empty(n, s), empty(k, s), empty(s, s)
    with P.PQR(n, k + s, s, dev(Q), k=k, variant="tsqr", chains="on") as h:
        t = h.solve(dev(X), U=U, P=Pm, N=Nm, flags=P.PQR_NO_APPEND)
        assert h.stats()["leaf_chains"] == 4
    torch.cuda.synchronize()
    assert t == ref["t"]
    assert rel(host(Pm), ref["P"]) < 1e-10 and rel(host(Nm), ref["N"]) < 1e-10
    assert rel(host(U)[:, :t], ref["U"]) < 1e-10


@pytest.mark.parametrize("chunks", ["3", "5"])
def test_chains_host_pipeline(P, orc, chunks, monkeypatch):
    """Host X and U: the leaf launches run chunk by chunk (whole chain rounds), the chains' carries
    crossing launch boundaries; stage 2 runs the chunks backwards.  Same results as the device
    path to rounding and the oracle's within tolerance."""
    import torch

    monkeypatch.setenv("PQR_SMS", "2")
    monkeypatch.setenv("PQR_HOST_CHUNKS", chunks)
    n, k, s = 70_001, 24, 8
    Q = inputs.orthonormal(601, n, k)
    X1 = inputs.gaussian(602, n, s)
    X2 = inputs.gaussian(603, n, s)
    ref = orc.householder_pqr(Q, X1)
    res = {}
    for mode in ("host", "device"):
        conv = (lambda a: a) if mode == "host" else dev
        mk = (lambda r, c: np.zeros((r, c), order="F")) if mode == "host" else empty
        get = (lambda a: np.array(a)) if mode == "host" else host
        U, Pm, Nm = mk(n, s), mk(k, s), mk(s, s)
        with P.PQR(n, k + 2 * s, s, dev(Q), k=k, variant="tsqr", chains="on") as h:
            t1 = h.solve(conv(X1), U=U, P=Pm, N=Nm)
            r1 = (get(U), get(Pm), get(Nm))
            t2 = h.solve(conv(X2), U=U, flags=P.PQR_NO_APPEND)
            r2 = get(U)
        torch.cuda.synchronize()
        res[mode] = (t1, t2, r1, r2)
    hst, dv = res["host"], res["device"]
    assert hst[0] == dv[0] == s and hst[1] == dv[1] == s
    assert rel(hst[2][0], ref["U"]) < 1e-10 and rel(hst[2][1], ref["P"]) < 1e-10 and rel(hst[2][2], ref["N"]) < 1e-10
    for a, b in zip(hst[2] + (hst[3],), dv[2] + (dv[3],)):
        assert rel(a, b) < 1e-12


def test_chains_plan(P):
    """Plan: AUTO keeps the pure tree (chains measure slower); ON chains 2 x SMs chains
    when there are more leaf blocks than chains; a leaf count at or below the chain count keeps the tree."""
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = 4 * 2 * sms * 1024 + 1000
    with P.PQR(n, 16, 8, None, k=0, variant="tsqr") as h:
        assert h.stats()["leaf_chains"] == 0
    with P.PQR(n, 16, 8, None, k=0, variant="tsqr", chains="on") as h:
        assert h.stats()["leaf_chains"] == 2 * sms
    with P.PQR(50_000, 16, 8, None, k=0, variant="tsqr", chains="on") as h:
        assert h.stats()["leaf_chains"] == 0
