"""Helpers for the GPU parity tests (marshalling only)."""
import numpy as np


def dev(a, device="cuda"):
    """numpy (Fortran) n x m -> torch CUDA column-major n x m."""
    import torch

    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return torch.from_numpy(np.ascontiguousarray(a.T)).to(device).t()


def host(t):
    """torch column-major -> numpy Fortran."""
    return np.asfortranarray(t.detach().cpu().numpy())


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def empty(n, m, device="cuda"):
    from paper_2204_13393_b200 import inputs

    return inputs.colmajor_empty(n, m, device)


def ortho_loss_2(Q, U):
    """||I - [Q U]^T [Q U]||_2 on the device (torch fp64 GEMM; test-side check only)."""
    import torch

    k, t = Q.shape[1], U.shape[1]
    G = torch.empty((k + t, k + t), dtype=torch.float64, device=U.device)
    if k:
        G[:k, :k] = Q.t() @ Q
        G[:k, k:] = Q.t() @ U
        G[k:, :k] = G[:k, k:].t()
    G[k:, k:] = U.t() @ U
    G -= torch.eye(k + t, dtype=G.dtype, device=G.device)
    return float(torch.linalg.matrix_norm(G, ord=2))
