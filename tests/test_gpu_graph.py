"""CUDA-graph replay of repeated calls (pqr_api.cu, GraphKey): the second call with identical
arguments (device buffers, PQR_NO_APPEND, one rank) is captured and later calls replay it.
Replayed results must be bitwise identical to the uncaptured call's and follow input changes
made in place (same pointers, new values); a changed argument must not replay a stale graph."""
import numpy as np
import pytest

from gpu_util import dev, empty, host, rel
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


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("n,k,s", [(10_000, 32, 4), (70_001, 64, 8), (20_000, 40, 16)])
def test_replay_matches_and_follows_inputs(P, orc, variant, n, k, s):
    import torch

    Q = inputs.orthonormal(90 + n, n, k)
    X1 = inputs.gaussian(91 + n, n, s)
    X2 = inputs.gaussian(92 + n, n, s)
    Xd = dev(X1)
    U, Pm, Nm = empty(n, s), empty(k, s), empty(s, s)
    with P.PQR(n, k + s, s, dev(Q), k=k, variant=variant) as h:
        outs = []
        for _ in range(4):  # call 1 plain, call 2 captured, calls 3-4 replayed
            t = h.solve(Xd, U=U, P=Pm, N=Nm, flags=P.PQR_NO_APPEND)
            torch.cuda.synchronize()
            outs.append((t, host(U).copy(), host(Pm).copy(), host(Nm).copy()))
        for o in outs[1:]:
            assert o[0] == outs[0][0]
            for a, b in zip(o[1:], outs[0][1:]):
                assert np.array_equal(a, b)
        # new values in the same buffer: the replay must compute on them
        Xd.copy_(dev(X2))
        t = h.solve(Xd, U=U, P=Pm, N=Nm, flags=P.PQR_NO_APPEND)
        torch.cuda.synchronize()
        ref = orc.householder_pqr(Q, X2)
        assert t == s and rel(host(Pm), ref["P"]) < 1e-10 and rel(host(Nm), ref["N"]) < 1e-10
        assert rel(host(U), ref["U"]) < 1e-10
        # a different output buffer: no stale replay
        U2 = empty(n, s)
        t = h.solve(Xd, U=U2, P=Pm, N=Nm, flags=P.PQR_NO_APPEND)
        torch.cuda.synchronize()
        assert rel(host(U2), ref["U"]) < 1e-10
        # an appending call after replays, then a replay-eligible call on the grown basis
        h.solve(Xd, U=U, P=Pm, N=Nm)
        assert h.k == k + s
        Pk = empty(k + s, s)
        for _ in range(3):
            t = h.solve(dev(X1), U=U2, P=Pk, N=Nm, flags=P.PQR_NO_APPEND)
        torch.cuda.synchronize()
        ref2 = orc.householder_pqr(np.hstack([Q, ref["U"]]), X1)
        assert rel(host(Pk), ref2["P"]) < 1e-10 and rel(host(U2), ref2["U"]) < 1e-10
