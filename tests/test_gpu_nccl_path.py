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


def test_single_rank_nccl_path():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, PQR_FORCE_NCCL="1")
    r = subprocess.run([sys.executable, os.path.join(HERE, "nccl_path_worker.py")], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    for variant, d in out.items():
        assert d["t"] == 8, (variant, d)
        assert d["P"] < 1e-10 and d["N"] < 1e-10 and d["U"] < 1e-10, (variant, d)
    assert out["cholqr2"]["collectives"] == 2   # one allgather per CholQR pass
    assert out["tsqr"]["collectives"] >= 1      # the GPU roots' allgather (LOR build + solve)
