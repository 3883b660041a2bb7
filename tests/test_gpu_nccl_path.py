"""The multi-GPU code path on one GPU: with PQR_FORCE_NCCL=1 a single-rank handle creates its
NCCL communicator and runs the allgather of each CholQR2 pass (a2) and the replicated
cross-GPU TSQR node (a7, reading R12) with one rank; results must still match the oracle."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(exchange, tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, PQR_FORCE_NCCL="1", PQR_TEST_EXCHANGE=exchange, PQR_TEST_DUMP=str(tmp_path / exchange))
    r = subprocess.run([sys.executable, os.path.join(HERE, "nccl_path_worker.py")], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    for variant, d in out.items():
        assert d["t"] == 8, (variant, d)
        assert d["P"] < 1e-10 and d["N"] < 1e-10 and d["U"] < 1e-10, (variant, d)
        assert d["repeat_bitwise"], (variant, d)
    assert out["cholqr2"]["collectives"] == 2 * 3   # one exchange per CholQR pass, three calls
    assert out["tsqr"]["collectives"] >= 3          # the GPU roots' exchange per call (+ LOR build)
    assert out["tsqr_pip2"]["collectives"] >= 2 * 3  # two Gram exchanges per call
    return out


def test_single_rank_nccl_path(tmp_path):
    out = _run("collective", tmp_path)
    assert all(d["exchange"] == 1 for d in out.values())


def test_single_rank_nccl_device_api_path(tmp_path):
    """f4: the exchange through the NCCL device API (symmetric window + LSA barrier, fused into the
    factor kernel for CholQR2).  With one rank its sums see the same single part as the collective
    path: results must be bitwise those of the collective path."""
    import numpy as np

    out = _run("lsa", tmp_path)
    assert all(d["exchange"] == 2 for d in out.values())
    _run("collective", tmp_path)
    for v in out:
        a = np.load(tmp_path / f"lsa_{v}.npz")
        b = np.load(tmp_path / f"collective_{v}.npz")
        for key in ("U", "P", "N"):
            assert np.array_equal(a[key], b[key]), (v, key)
