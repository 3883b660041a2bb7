"""The NCCL multi-rank path on real GPUs: torchrun over min(#GPUs, 8) >= 2 ranks, one global
problem row-sharded, both variants, against the CPU oracle with P and N bitwise replicated.
Skipped on a box with fewer than 2 GPUs (the virtual-rank tests cover the same library code
with one GPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_torchrun_nccl_ranks():
    import torch

    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(8, torch.cuda.device_count())
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(HERE, "multigpu_worker.py")], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    for v, d in out.items():
        assert d["t"] == [8] * world and d["replicated"], (v, d)
        assert d["P"] < 1e-10 and d["N"] < 1e-10 and d["U"] < 1e-10, (v, d)
