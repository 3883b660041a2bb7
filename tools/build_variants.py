"""Build several A/B variants of libpqr.so in parallel: python tools/build_variants.py NAME:-DA=1,-DB=0[:trace] ...
Each goes to build/NAME/libpqr.so (the in-tree product library is untouched)."""
import concurrent.futures
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_13393_b200 import build as b  # noqa: E402


def one(spec):
    parts = spec.split(":")
    name = parts[0]
    defs = [d for d in (parts[1].split(",") if len(parts) > 1 else []) if d]
    trace = len(parts) > 2 and parts[2] == "trace"
    out = os.path.join(b.ROOT, "build", name, "libpqr.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    return b.build(force=True, defines=defs, out=out, trace=trace)


with concurrent.futures.ThreadPoolExecutor(max_workers=len(sys.argv) - 1) as ex:
    for r in ex.map(one, sys.argv[1:]):
        print(r)
