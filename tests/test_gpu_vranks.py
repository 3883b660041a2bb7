"""The library's multi-rank path executed on one GPU with virtual ranks (pqr_vgroup_create):
one global problem row-sharded over P = 2, 4, 8 handles in this process, each driven from its
own host thread and stream; the ranks exchange their (k+s) x s Grams (CholQR2, a2) and their
GPU roots' (C+s) x s blocks (TSQR, a7, the replicated cross-GPU tree) through device copies in
place of ncclAllGather.  This runs every rank >= 1 branch of the library (the per-rank root
offset in the cross-GPU tree, nparts = nranks in the factor, the cross-GPU tree levels).

Pins: the CPU oracle on the global problem (<= 1e-10, BASELINE north_star), the one-rank
result (partition invariance: <= 1e-13), and P, N, t bitwise identical on
every rank (replicated reductions in rank order, R7)."""
import os

import numpy as np
import pytest

from gpu_util import dev, empty, host, rel
from paper_2204_13393_b200 import inputs
import vranks

pytestmark = pytest.mark.gpu
VARIANTS = ["cholqr2", "tsqr"]
os.environ.setdefault("PQR_VGROUP_TIMEOUT", "120")


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_13393_b200 import pqr

    pqr.lib()
    return pqr


def assert_replicated(out, ci=0):
    c0 = out[0]["calls"][ci]
    for o in out[1:]:
        c = o["calls"][ci]
        assert c["t"] == c0["t"]
        assert np.array_equal(c["P"], c0["P"]) and np.array_equal(c["N"], c0["N"])


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("n,k,s", [(200_003, 64, 8), (160_000, 96, 16)])
def test_vranks_vs_oracle_and_one_rank(P, orc, variant, nranks, n, k, s):
    Q = inputs.orthonormal(3 + n + k, n, k)
    X = inputs.gaussian(4 + n + s, n, s)
    ref = orc.householder_pqr(Q, X)
    one = vranks.run(P, Q, X, 1, variant)
    out = vranks.run(P, Q, X, nranks, variant)
    assert_replicated(out)
    c = out[0]["calls"][0]
    U = vranks.gather_u(out)
    assert c["t"] == ref["t"] == s
    for name, got, want in (("P", c["P"], ref["P"]), ("N", c["N"], ref["N"]), ("U", U, ref["U"])):
        assert rel(got, want) < 1e-10, (name, rel(got, want))
    o1 = one[0]["calls"][0]
    for name, got, want in (("P", c["P"], o1["P"]), ("N", c["N"], o1["N"]), ("U", U, o1["U"])):
        assert rel(got, want) < 1e-13, (name, rel(got, want))
    assert np.linalg.norm(np.eye(s) - U.T @ U, 2) < 1e-12 and np.linalg.norm(Q.T @ U, 2) < 1e-12
    st = out[0]["stats"]
    assert st["collectives"] >= (2 if variant == "cholqr2" else 1)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("nranks", [3, 8])
def test_vranks_appending_and_basis_apply(P, orc, variant, nranks):
    """Three appending solves (widths 8, 5, 8) on a growing basis, then the explicit basis via
    pqr_basis_apply on every rank: against the oracle on the same growing basis."""
    n, k = 90_001, 24
    Q = inputs.orthonormal(61, n, k)
    Xs = [inputs.gaussian(62 + i, n, w) for i, w in enumerate((8, 5, 8))]
    out = vranks.run(P, Q, Xs[0], nranks, variant, calls=[(x, 0) for x in Xs], k_max=k + 21, s_max=8,
                     apply_after=True)
    Qg = Q
    for ci, x in enumerate(Xs):
        assert_replicated(out, ci)
        ref = orc.householder_pqr(Qg, x)
        c = out[0]["calls"][ci]
        U = vranks.gather_u(out, ci)
        assert c["t"] == ref["t"]
        assert rel(c["P"], ref["P"]) < 1e-10 and rel(c["N"], ref["N"]) < 1e-10 and rel(U, ref["U"]) < 1e-10
        Qg = np.asfortranarray(np.hstack([Qg, ref["U"]]))
    B = np.vstack([o["basis"] for o in out])
    assert B.shape == Qg.shape and rel(B, Qg) < 1e-10


@pytest.mark.parametrize("variant", VARIANTS)
def test_vranks_deflation_config_shape(P, orc, variant):
    """configs[3] shape (k = 96, s = 16, two dependent columns, reading R9) at 8 ranks: the
    cross-GPU TSQR tree over 8 roots of 112 rows (one node of 896 rows did not fit a 16-wide
    level kernel in round 1: PQR_EPLAN)."""
    Q, X = inputs.deflation_inputs(71, 2 ** 17, 96, 16)
    ref = orc.householder_pqr(Q, X)
    out = vranks.run(P, Q, X, 8, variant)
    assert_replicated(out)
    c = out[0]["calls"][0]
    assert c["t"] == ref["t"] == 14
    assert rel(c["P"], ref["P"]) < 1e-10
    piv = [int(np.flatnonzero(np.abs(ref["N"][i]) > 0)[0]) for i in range(14)]
    assert [int(np.flatnonzero(np.abs(c["N"][i]) > 0)[0]) for i in range(14)] == piv
    U = vranks.gather_u(out)
    assert np.linalg.norm(np.eye(14) - U.T @ U, 2) < 1e-12 and np.linalg.norm(Q.T @ U, 2) < 1e-12


@pytest.mark.parametrize("variant", VARIANTS)
def test_vranks_weak_config_plan_8(P, variant):
    """configs[4] handle shape (k_max = 128, s_max = 8) at 8 ranks creates and solves (the cross
    tree splits 8 roots of 136 rows into two nodes); manufactured truth on 8 x 2^15 rows."""
    n = 8 * 2 ** 15
    m = inputs.manufactured(81, n, 128, 8)
    out = vranks.run(P, m["Q"], m["X"], 8, variant)
    assert_replicated(out)
    c = out[0]["calls"][0]
    assert c["t"] == 8
    assert rel(c["P"], m["C"]) < 1e-11 and rel(c["N"], m["D"]) < 1e-10
    assert rel(vranks.gather_u(out), m["Y"]) < 1e-10
