"""World-size-2 tests of the multi-GPU path's HOST logic on CPU (gloo): row sharding, the
NCCL-id broadcast plumbing, the cross-rank Gram reduction (a2) and the TSQR cross-GPU level
(R12).  ORACLE-ONLY: the per-rank arithmetic here is the CPU oracle on each rank's shard; the
library's own multi-rank code (exchanges, cross-GPU tree, nparts = nranks) is executed by
tests/test_gpu_vranks.py (virtual ranks on one GPU) and tests/test_gpu_multigpu.py (torchrun
over >= 2 GPUs, skipped with fewer)."""
import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_shard_unit():
    from paper_2204_13393_b200.dist import row_shard

    for n in (7, 100, 2 ** 20 + 3):
        for world in (1, 2, 3, 8):
            parts = [row_shard(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and sum(p[1] for p in parts) == n
            for a, b in zip(parts, parts[1:]):
                assert a[0] + a[1] == b[0]


def test_sharded_pqr_world2(tmp_path, orc):
    import torch.multiprocessing as mp

    os.environ["PYTHONPATH"] = os.pathsep.join([HERE, ROOT, os.environ.get("PYTHONPATH", "")])
    sys.path.insert(0, HERE)
    import dist_workers

    world = 2
    mp.spawn(dist_workers.sharded_pqr_worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert not (tmp_path / f"rank{r}.err").exists(), (tmp_path / f"rank{r}.err").read_text()
        res = np.load(tmp_path / f"rank{r}.npy", allow_pickle=True).item()
        assert res["shards_ok"] and res["bcast_ok"] and res["max_ok"]
        assert res["gram_rel"] < 1e-13
        assert res["gram_replicated"]
        assert res["pip_N_rel"] < 1e-12 and res["pip_U_rel"] < 1e-10
        assert res["tsqr_P_rel"] < 1e-12 and res["tsqr_N_rel"] < 1e-10
