"""GPU parity of pqr_project_normalize / pqr_basis_apply end to end (both variants,
all §8(a) rows through the C-ABI) against the CPU oracle.

Tolerances (BASELINE north_star): relative Frobenius error of U, P, N <= 1e-10 for
kappa <= 1e4 and ||I - [Q U]^T [Q U]||_2 <= 1e-12."""
import numpy as np
import pytest

from gpu_util import dev, empty, host, ortho_loss_2, rel
from paper_2204_13393_b200 import inputs

pytestmark = pytest.mark.gpu
VARIANTS = ["cholqr2", "tsqr"]


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_13393_b200 import pqr

    pqr.lib()
    return pqr


# ---------------------------------------------------------------------------
# end to end (a1-a5 through pqr_project_normalize)
# ---------------------------------------------------------------------------
def solve(P, Q, X, variant="cholqr2", flags=None, k_max=None, **kw):
    import torch

    n, s = X.shape
    k = Q.shape[1]
    Qd, Xd = dev(Q), dev(X)
    U, Pm, Nm = empty(n, s), empty(max(k, 1), s), empty(s, s)
    with P.PQR(n, k_max or k, s, Qd if k else None, k=k, variant=variant, **kw) as h:
        t = h.solve(Xd, U=U, P=Pm, N=Nm, flags=P.PQR_NO_APPEND if flags is None else flags)
        st = h.stats()
    torch.cuda.synchronize()
    return dict(U=host(U)[:, :t], P=host(Pm)[:k], N=host(Nm), t=t, stats=st, Qd=Qd, Ud=U[:, :t])


def check_vs_oracle(out, ref, tol=1e-10):
    assert out["t"] == ref["t"]
    if ref["P"].size:
        assert rel(out["P"], ref["P"]) < tol
    assert rel(out["N"], ref["N"]) < tol
    assert rel(out["U"], ref["U"]) < tol


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("n,k,s", [(10_000, 32, 4), (4097, 13, 3), (20_000, 0, 8), (65_536, 128, 8),
                                   (30_001, 96, 16), (12, 3, 2), (300_007, 64, 8),
                                   (20_011, 144, 16), (50_000, 152, 8),  # these two: k + s = kMMax
                                   (7777, 5, 1), (1000, 0, 1), (2049, 40, 7),
                                   # odd n (odd ld: unaligned Gram path) with s > 8 and a 48 KB
                                   # reduction buffer; leaf remainders that overflow a 512-row block
                                   (20_001, 74, 9), (20_001, 28, 13), (105_253, 92, 14)])
def test_vs_oracle_random(P, orc, variant, n, k, s):
    Q = inputs.orthonormal(7 + n, n, k)
    X = inputs.gaussian(8 + n, n, s)
    out = solve(P, Q, X, variant=variant)
    ref = orc.householder_pqr(Q, X)
    check_vs_oracle(out, ref)
    assert ortho_loss_2(out["Qd"], out["Ud"]) < 1e-12


@pytest.mark.parametrize("variant", VARIANTS)
def test_tiny_config(P, orc, variant):
    """configs[0] at full size: n=10,000, k=32, s=4."""
    Q, X = inputs.tiny_inputs()
    out = solve(P, Q, X, variant=variant)
    check_vs_oracle(out, orc.householder_pqr(Q, X))
    assert ortho_loss_2(out["Qd"], out["Ud"]) < 1e-12


@pytest.mark.parametrize("variant", VARIANTS)
def test_projected(P, orc, variant):
    """configs[1] shape (projection dominates, reading R8) at n = 2^18."""
    Q, X = inputs.projected_inputs(21, 2 ** 18, 64, 8)
    out = solve(P, Q, X, variant=variant)
    check_vs_oracle(out, orc.householder_pqr(Q, X))
    assert ortho_loss_2(out["Qd"], out["Ud"]) < 1e-12


@pytest.mark.parametrize("variant", VARIANTS)
def test_manufactured(P, variant):
    m = inputs.manufactured(31, 2 ** 16, 64, 8)
    out = solve(P, m["Q"], m["X"], variant=variant)
    assert out["t"] == 8
    assert rel(out["P"], m["C"]) < 1e-12 and rel(out["N"], m["D"]) < 1e-11 and rel(out["U"], m["Y"]) < 1e-10


@pytest.mark.parametrize("variant", VARIANTS)
def test_special_cases(P, variant):
    n, k, s = 5000, 16, 4
    m = inputs.manufactured(41, n, k, s)
    # X orthonormal and orthogonal to Q: P = 0, N = I, U = X
    out = solve(P, m["Q"], m["Y"], variant=variant)
    assert np.linalg.norm(out["P"]) < 1e-13 and rel(out["N"], np.eye(s)) < 1e-13 and rel(out["U"], m["Y"]) < 1e-13
    # X inside span(Q): t = 0, P = C
    out = solve(P, m["Q"], np.asfortranarray(m["Q"] @ m["C"]), variant=variant)
    assert out["t"] == 0 and rel(out["P"], m["C"]) < 1e-13 and np.all(out["N"] == 0)
    # X = 0: t = 0, P = 0, N = 0 (every column deflates; no division by a zero norm)
    out = solve(P, m["Q"], np.zeros((n, s), order="F"), variant=variant)
    assert out["t"] == 0 and np.all(out["P"] == 0) and np.all(out["N"] == 0)
    # one zero column among independent ones: it alone deflates
    X = np.array(m["Y"], order="F")
    X[:, 1] = 0.0
    out = solve(P, m["Q"], X, variant=variant)
    assert out["t"] == s - 1 and np.all(out["N"][s - 1:] == 0)


@pytest.mark.parametrize("variant", VARIANTS)
def test_deflation_small(P, orc, variant):
    """configs[3] shape at n = 2^15: two dependent columns -> t = 14, pivots as the oracle."""
    Q, X = inputs.deflation_inputs(51, 2 ** 15, 96, 16)
    ref = orc.householder_pqr(Q, X)
    assert ref["t"] == 14
    out = solve(P, Q, X, variant=variant)
    assert out["t"] == 14
    assert rel(out["P"], ref["P"]) < 1e-10
    # N row-echelon with the oracle's pivot columns; projectors agree
    piv = [int(np.flatnonzero(np.abs(ref["N"][i]) > 0)[0]) for i in range(14)]
    piv_gpu = [int(np.flatnonzero(np.abs(out["N"][i]) > 0)[0]) for i in range(14)]
    assert piv == piv_gpu
    assert np.all(out["N"][14:] == 0)
    Pu = out["U"] @ out["U"].T[:, :64]
    Pr = ref["U"] @ ref["U"].T[:, :64]
    assert rel(Pu, Pr) < 1e-6


def test_deflation_small_tsqr_columnwise(P, orc):
    """configs[3] shape, TSQR (Householder) variant: the grading of X is a column scaling, and
    Householder QR is column-wise backward stable (its Q factor and each column's relative error
    do not depend on the column scales), so every kept column of U and every column of [P; N]
    matches the oracle's Householder QR relative to that column's own norm — not only through
    the 1e-6 projector of test_deflation_small (reading R11 bounds only the Cholesky variant)."""
    Q, X = inputs.deflation_inputs(51, 2 ** 15, 96, 16)
    ref = orc.householder_pqr(Q, X)
    out = solve(P, Q, X, variant="tsqr")
    t = ref["t"]
    assert out["t"] == t == 14
    errs_u = [np.linalg.norm(out["U"][:, j] - ref["U"][:, j]) for j in range(t)]  # unit columns
    assert max(errs_u) < 1e-9, errs_u
    for j in range(16):
        cref = np.concatenate([ref["P"][:, j], ref["N"][:, j]])
        cout = np.concatenate([out["P"][:, j], out["N"][:, j]])
        assert np.linalg.norm(cout - cref) < 1e-10 * np.linalg.norm(cref), j


def test_cholqr2_single_pass_is_bcgs_pip(P, orc):
    """PQR_SINGLE_PASS = Alg. 7 (one BCGS-PIP pass): same result as the oracle's Alg. 7."""
    Q, X = inputs.projected_inputs(61, 20_000, 32, 4, ratio=1e-2)
    out = solve(P, Q, X, flags=P.PQR_NO_APPEND | P.PQR_SINGLE_PASS)
    ref = orc.bcgs_pip(Q, X)
    assert out["t"] == ref["t"]
    assert rel(out["P"], ref["P"]) < 1e-12 and rel(out["N"], ref["N"]) < 1e-10 and rel(out["U"], ref["U"]) < 1e-9


@pytest.mark.parametrize("variant", VARIANTS)
def test_append_and_basis_apply(P, orc, variant):
    """Append semantics (Alg. 1): after two solves k = k0 + 2s; Y = Q C reproduces the basis."""
    import torch

    n, k0, s = 9000, 8, 4
    Q = inputs.orthonormal(71, n, k0)
    X1 = inputs.gaussian(72, n, s)
    X2 = inputs.gaussian(73, n, s)
    with P.PQR(n, k0 + 2 * s, s, dev(Q), variant=variant) as h:
        t1 = h.solve(dev(X1))
        t2 = h.solve(dev(X2))
        assert (t1, t2) == (s, s) and h.k == k0 + 2 * s
        C = np.eye(k0 + 2 * s)
        Y = empty(n, k0 + 2 * s)
        h.apply(dev(C), k0 + 2 * s, Y)
        torch.cuda.synchronize()
        B = host(Y)
    ref1 = orc.householder_pqr(Q, X1)
    Q1 = np.hstack([Q, ref1["U"]])
    ref2 = orc.householder_pqr(Q1, X2)
    assert rel(B[:, :k0], Q) < 1e-13
    assert rel(B[:, k0:k0 + s], ref1["U"]) < 1e-10
    assert rel(B[:, k0 + s:], ref2["U"]) < 1e-10
    # general C: Y = Q C
    C = inputs.gaussian(74, k0 + 2 * s, 5)
    with P.PQR(n, k0, s, dev(Q), variant=variant) as h:
        Y = empty(n, 5)
        h.apply(dev(C[:k0]), 5, Y)
        torch.cuda.synchronize()
        assert rel(host(Y), orc.matmul(Q, C[:k0])) < 1e-13


@pytest.mark.parametrize("variant", VARIANTS)
def test_host_buffers(P, orc, variant):
    """Host (numpy) X/U/P/N go through the library's staging (the e2e path)."""
    n, k, s = 6000, 12, 4
    Q = inputs.orthonormal(81, n, k)
    X = inputs.gaussian(82, n, s)
    U = np.zeros((n, s), order="F")
    Pm = np.zeros((k, s), order="F")
    Nm = np.zeros((s, s), order="F")
    with P.PQR(n, k, s, Q, variant=variant) as h:
        t = h.solve(X, U=U, P=Pm, N=Nm, flags=P.PQR_NO_APPEND)
    ref = orc.householder_pqr(Q, X)
    assert t == s
    assert rel(Pm, ref["P"]) < 1e-10 and rel(Nm, ref["N"]) < 1e-10 and rel(U, ref["U"]) < 1e-10


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("chunks,n", [(None, 300_000), ("3", 6000), ("16", 20_011)])
def test_host_pipeline(P, orc, variant, chunks, n, monkeypatch):
    """Host X and U on one rank: the upload, the first and the last pass run in row chunks on
    two streams (HostPipe; default 8 chunks from 2^18 rows, PQR_HOST_CHUNKS forces it for small,
    ragged n).  Results: the oracle's within the parity tolerance, the device-buffer path's to
    rounding (the chunked Gram sums in chunk order), and the appended basis the same."""
    import torch

    if chunks is not None:
        monkeypatch.setenv("PQR_HOST_CHUNKS", chunks)
    k, s = 24, 8
    Q = inputs.orthonormal(171, n, k)
    X1 = np.asfortranarray(inputs.gaussian(172, n, s) + Q @ inputs.gaussian(173, k, s))
    X2 = inputs.gaussian(174, n, s)
    ref = orc.householder_pqr(Q, X1)
    outs = {}
    for mode in ("host", "device"):
        U = np.zeros((n, s), order="F") if mode == "host" else empty(n, s)
        Pm = np.zeros((k, s), order="F") if mode == "host" else empty(k, s)
        Nm = np.zeros((s, s), order="F") if mode == "host" else empty(s, s)
        with P.PQR(n, k + 2 * s, s, dev(Q), k=k, variant=variant) as h:
            conv = (lambda a: a) if mode == "host" else dev
            t1 = h.solve(conv(X1), U=U, P=Pm, N=Nm)  # appends
            U1, P1, N1 = (np.array(U), np.array(Pm), np.array(Nm)) if mode == "host" else (host(U), host(Pm), host(Nm))
            Pm2 = np.zeros((k + s, s), order="F") if mode == "host" else empty(k + s, s)
            t2 = h.solve(conv(X2), U=U, P=Pm2, N=Nm, flags=P.PQR_NO_APPEND)
            U2 = np.array(U) if mode == "host" else host(U)
            P2 = np.array(Pm2) if mode == "host" else host(Pm2)
        torch.cuda.synchronize()
        outs[mode] = dict(t=(t1, t2), U1=U1, P1=P1, N1=N1, U2=U2, P2=P2)
    hst, dv = outs["host"], outs["device"]
    assert hst["t"] == dv["t"] == (s, s)
    assert rel(hst["P1"], ref["P"]) < 1e-10 and rel(hst["N1"], ref["N"]) < 1e-10 and rel(hst["U1"], ref["U"]) < 1e-10
    for key in ("U1", "P1", "N1", "U2", "P2"):
        assert rel(hst[key], dv[key]) < 1e-12, key


@pytest.mark.parametrize("sms", ["2", "3"])
def test_tsqr_two_groups_many_blocks_per_cta(P, orc, sms, monkeypatch):
    """Grids sized for 2-3 SMs (PQR_SMS) give every CTA several leaf blocks, so both groups of
    the two-group level kernels work, hand ring slots back and forth and run ahead of each
    other; the panel merge (s = 4 after s = 4) runs too.  Parity with the oracle on every call
    and bitwise reproducibility over repeated runs (a race would show up here)."""
    import torch

    monkeypatch.setenv("PQR_SMS", sms)
    n, k = 23 * 1024 + 41, 24
    Q = inputs.orthonormal(191, n, k)
    Xs = [inputs.gaussian(192 + i, n, s) for i, s in enumerate((8, 4, 4))]
    runs = []
    for rep in range(2):
        outs = []
        with P.PQR(n, k + 16, 8, dev(Q), k=k, variant="tsqr") as h:
            Qcur = Q
            for X in Xs:
                s = X.shape[1]
                U = empty(n, s)
                Pm, Nm = empty(Qcur.shape[1], s), empty(s, s)
                t = h.solve(dev(X), U=U, P=Pm, N=Nm, s=s)
                torch.cuda.synchronize()
                ref = orc.householder_pqr(Qcur, X)
                assert t == s
                assert rel(host(Pm), ref["P"]) < 1e-10 and rel(host(U)[:, :t], ref["U"]) < 1e-10
                outs.append(host(U))
                Qcur = np.asfortranarray(np.hstack([Qcur, ref["U"]]))
        runs.append(outs)
    for a, b in zip(runs[0], runs[1]):
        assert np.array_equal(a, b)


def test_two_handles_two_threads(P, orc):
    """Two handles (one per variant, each on its own stream) called concurrently from two host
    threads with host buffers — the bench's e2e leg — give the serial results."""
    import threading

    import torch

    n, k, s = 300_000, 16, 8
    Q = inputs.orthonormal(181, n, k)
    X = inputs.gaussian(182, n, s)
    ref = orc.householder_pqr(Q, X)
    hs = {v: P.PQR(n, k, s, dev(Q), variant=v, stream=torch.cuda.Stream()) for v in VARIANTS}
    res = {}

    def run(v, reps):
        out = []
        for _ in range(reps):
            U = np.zeros((n, s), order="F")
            Pm = np.zeros((k, s), order="F")
            Nm = np.zeros((s, s), order="F")
            t = hs[v].solve(X, U=U, P=Pm, N=Nm, flags=P.PQR_NO_APPEND)
            out.append((t, U, Pm, Nm))
        res[v] = out

    ths = [threading.Thread(target=run, args=(v, 3)) for v in VARIANTS]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for v in VARIANTS:
        hs[v].close()
        assert len(res[v]) == 3
        for t, U, Pm, Nm in res[v]:
            assert t == s
            assert rel(Pm, ref["P"]) < 1e-10 and rel(Nm, ref["N"]) < 1e-10 and rel(U, ref["U"]) < 1e-10
        # repeated concurrent calls are bitwise reproducible
        assert all(np.array_equal(res[v][0][1], r[1]) for r in res[v][1:])


@pytest.mark.parametrize("variant", VARIANTS)
def test_no_deflation_flag_breakdown(P, variant):
    n, k, s = 4000, 8, 4
    Q = inputs.orthonormal(91, n, k)
    X = inputs.gaussian(92, n, s)
    X[:, 2] = X[:, 0]
    with P.PQR(n, k, s, dev(Q), variant=variant) as h:
        with pytest.raises(P.PQRError) as e:
            h.solve(dev(X), flags=P.PQR_NO_DEFLATION)
        assert e.value.code == P.PQR_EBREAKDOWN
        assert h.k == k  # basis unchanged on error


@pytest.mark.parametrize("variant", VARIANTS)
def test_capacity_error(P, variant):
    n = 1000
    with P.PQR(n, 4, 4, None, k=0, variant=variant) as h:
        X = dev(inputs.gaussian(1, n, 4))
        assert h.solve(X) == 4 and h.solve(X) == 0  # second block is in span -> t = 0
        with pytest.raises(P.PQRError) as e:
            h.solve(dev(inputs.gaussian(2, n, 8)))
        assert e.value.code == P.PQR_ECAPACITY


@pytest.mark.parametrize("widths,probe", [([8, 3, 8, 5], 8), ([4, 4, 4, 4, 8, 4, 4], 4)])
@pytest.mark.parametrize("variant", VARIANTS)
def test_mixed_block_widths_and_no_append(P, orc, variant, widths, probe):
    """A sequence with varying s and NO_APPEND probes in between (the Arnoldi pattern when a
    block deflates): every solve matches the oracle on the basis accumulated so far.  Covers
    TSQR panels of different widths in one LOR, stale tree-slot rows after a wider probe, and
    the merge of consecutive 4-wide panels into 8-wide ones (committed and probed)."""
    import torch

    n, k0 = 70_001, 13  # several leaf blocks per CTA, odd n (pad row), odd k0
    Q = inputs.orthonormal(101, n, k0)
    basis = Q.copy(order="F")
    with P.PQR(n, k0 + sum(widths), 8, dev(Q), variant=variant) as h:
        for i, s in enumerate(widths):
            # a probe that must leave no trace (4-wide probes exercise the TSQR panel merge
            # without committing it), then the real (appending) solve
            Xp = inputs.gaussian(200 + i, n, probe)
            Up, Pp, Np = empty(n, probe), empty(basis.shape[1], probe), empty(probe, probe)
            tp = h.solve(dev(Xp), U=Up, P=Pp, N=Np, flags=P.PQR_NO_APPEND, s=probe)
            torch.cuda.synchronize()
            refp = orc.householder_pqr(basis, Xp)
            assert tp == refp["t"] == probe
            assert rel(host(Pp), refp["P"]) < 1e-10 and rel(host(Up)[:, :tp], refp["U"]) < 1e-10
            X = inputs.gaussian(300 + i, n, s)
            U, Pm, Nm = empty(n, s), empty(basis.shape[1], s), empty(s, s)
            t = h.solve(dev(X), U=U, P=Pm, N=Nm, s=s)
            torch.cuda.synchronize()
            ref = orc.householder_pqr(basis, X)
            assert t == ref["t"] == s
            assert rel(host(Pm), ref["P"]) < 1e-10 and rel(host(Nm), ref["N"]) < 1e-10
            assert rel(host(U)[:, :t], ref["U"]) < 1e-10
            basis = np.asfortranarray(np.hstack([basis, ref["U"]]))
        assert h.k == basis.shape[1]


def test_tsqr_invalid_block_plan(P):
    """Leaf blocks larger than the level kernels hold (6 x 256 rows per CTA) are refused with
    PQR_EPLAN (SPEC InvalidPlan), not run."""
    import torch

    n = 100_000
    Q = dev(inputs.orthonormal(5, n, 8))
    with pytest.raises(P.PQRError) as e:
        P.PQR(n, 16, 8, Q, variant="tsqr", block_rows=4096)
    assert e.value.code == P.PQR_EPLAN
    torch.cuda.synchronize()
    # the largest supported leaf (1536 rows) works
    X = dev(inputs.gaussian(6, n, 8))
    with P.PQR(n, 16, 8, Q, variant="tsqr", block_rows=1536) as h:
        assert h.solve(X, U=empty(n, 8), flags=P.PQR_NO_APPEND) == 8
        assert 1024 < h.stats()["block_rows"] <= 1536  # blocks are spread evenly over the rows
