"""B200-native fp64 project-and-normalize (PQR) library, arXiv 2204.13393.

The compute path lives in the C-ABI shared library ``libpqr.so`` (CUDA, sm_100a;
sources under ``csrc/``, declared in ``include/pqr.h``).  ``pqr`` is the thin
ctypes binding with the same names as the C-ABI; it fails loudly when the
library is missing — there is no CPU fallback.
"""
__all__ = ["pqr", "inputs"]
