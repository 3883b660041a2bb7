"""configs[2] at full size: block Arnoldi on the 256^3 7-point Laplacian (n = 2^24), s = 4,
33 PQR calls (k = 0, 4, ..., 128; reading R10), both variants, driven exactly as
`bench.py --workload arnoldi` drives them (same seed, same start block).

Pins: the first three calls against the CPU oracle's own Arnoldi chain at full n (Householder
PQR of [V X], numpy Laplacian; k <= 8 keeps it affordable) to <= 1e-10; for the whole run
properties that hold at any size: ||I - V^T V||_2 <= 1e-12, the Arnoldi relation
A V_m = V_{m+1} H, the Lanczos property (H block tridiagonal up to rounding; the operator is
symmetric), Ritz values inside the closed-form spectrum, and CholQR2-vs-TSQR agreement of H
(unique: P = V^T X, N with positive pivots) <= 1e-9."""
import math

import numpy as np
import pytest

from gpu_util import dev, empty, host, rel
from paper_2204_13393_b200 import inputs
from test_gpu_arnoldi import lap7_numpy

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
G, S, STEPS = 256, 4, 32
SEED = 2204133930 + 2  # bench.py's arnoldi seed (rank 0)


@pytest.fixture(scope="module")
def runs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_13393_b200 import pqr
    from paper_2204_13393_b200.arnoldi import block_arnoldi

    pqr.lib()
    dv = torch.device("cuda", 0)
    R = inputs.device_gaussian(SEED, G ** 3, S, dv)
    out = {}
    for v in ("cholqr2", "tsqr"):
        res = block_arnoldi(G, G, G, R, STEPS, variant=v)
        out[v] = res
    yield R, out
    for res in out.values():
        res["h"].close()


def test_first_calls_vs_oracle(runs, orc):
    R, out = runs
    n = G ** 3
    Rh = host(R)
    o = orc.householder_pqr(None, Rh)
    V = o["U"]
    H0 = o["N"]
    blocks = []
    for i in range(2):
        X = lap7_numpy(V[:, -S:], G, G, G)
        oi = orc.householder_pqr(V, X)
        blocks.append((V.shape[1], oi["P"], oi["N"]))
        V = np.asfortranarray(np.hstack([V, oi["U"]]))
    for v, res in out.items():
        assert res["t_list"] == [S] * (STEPS + 1), v
        assert rel(res["H0"], H0) < 1e-10, v
        H = res["H"]
        for i, (k, Pi, Ni) in enumerate(blocks):
            assert rel(H[:k, i * S:(i + 1) * S], Pi) < 1e-10, (v, i)
            assert rel(H[k:k + S, i * S:(i + 1) * S], Ni) < 1e-10, (v, i)
        # the basis' first 12 columns (three calls) against the oracle's U
        Vd = empty(n, 3 * S)
        res["h"].apply(dev(np.eye(res["k"])[:, :3 * S]), 3 * S, Vd)
        import torch

        torch.cuda.synchronize()
        assert rel(host(Vd), V) < 1e-10, v
        del Vd


def test_whole_run_properties(runs):
    import torch

    from paper_2204_13393_b200 import pqr

    R, out = runs
    n = G ** 3
    m = STEPS * S
    for v, res in out.items():
        k = res["k"]
        assert k == m + S
        h = res["h"]
        V = empty(n, k)
        h.apply(dev(np.eye(k)), k, V)
        torch.cuda.synchronize()
        # orthonormal basis
        Gm = V.t() @ V
        Gm -= torch.eye(k, dtype=Gm.dtype, device=Gm.device)
        assert float(torch.linalg.matrix_norm(Gm, ord=2)) < 1e-12, v
        del Gm
        # Arnoldi relation A V_m = V_{m+1} H, the stencil applied by the library 16 columns at a time
        H = res["H_dev"]
        AV = empty(n, m)
        for c in range(0, m, 16):
            pqr.pqr_laplacian7_apply(G, G, G, 16, V[:, c:c + 16], AV[:, c:c + 16])
        AV -= V @ H
        err = float(torch.linalg.matrix_norm(AV)) / (12.0 * math.sqrt(m))
        assert err < 1e-12, (v, err)
        del AV, V
        torch.cuda.empty_cache()
        Hh = res["H"]
        mask = np.zeros_like(Hh, dtype=bool)
        for bi in range(STEPS):
            mask[max(0, (bi - 1) * S):(bi + 2) * S, bi * S:(bi + 1) * S] = True
        assert np.abs(Hh[~mask]).max() < 1e-10 * np.abs(Hh).max(), v
        ritz = np.linalg.eigvalsh(0.5 * (Hh[:m, :m] + Hh[:m, :m].T))
        lo, hi = 6 - 6 * math.cos(math.pi / (G + 1)), 6 + 6 * math.cos(math.pi / (G + 1))
        assert ritz.min() > lo - 1e-9 and ritz.max() < hi + 1e-9, v
    assert rel(out["cholqr2"]["H"], out["tsqr"]["H"]) < 1e-9
