"""Build a libpqr.so with the TSQR phase counters compiled in (-DPQR_WY_TRACE) into
build/vtrace/ (the in-tree product library is untouched).  Run with
PQR_LIB=$PWD/build/vtrace/libpqr.so PQR_WY_TRACE=1 python bench.py --variant tsqr ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_13393_b200 import build as b  # noqa: E402

out = os.path.join(b.ROOT, "build", "vtrace", "libpqr.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(b.build(force=True, trace=True, out=out))
