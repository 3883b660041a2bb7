"""Build the current sources into build/<name>/libpqr.so with extra nvcc flags (A/B and trace builds;
the in-tree product library is untouched).  python tools/build_variant.py NAME [-DFOO ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_13393_b200 import build as b  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out = os.path.join(b.ROOT, "build", name, "libpqr.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(b.build(force=True, defines=extra, out=out))
