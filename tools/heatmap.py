"""fig:heatmap analogue: e_perp and kept rank of block column QR of Stewart
matrices for each (local, reduction) combination over P virtual ranks, at several kappa, with
deflation off in effect and with the library defaults.  JSON lines to stdout."""
import json, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))
sys.path.insert(0, os.path.dirname(HERE))
from paper_2204_13393_b200 import pqr  # noqa: E402
from test_gpu_pip2 import heatmap  # noqa: E402
pqr.lib()
for tol, label in ((1e-300, "deflation off"), (0.0, "library defaults")):
    for kappa in (1e4, 1e6, 1e8, 1e10, 1e12, 1e16):
        print(json.dumps({"kappa": kappa, "tolerances": label, "nranks": 4, "n": 1 << 15, "m": 64, "s": 4,
                          "cells": heatmap(pqr, kappa, tol=tol)}), flush=True)
