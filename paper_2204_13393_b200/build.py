"""Build libpqr.so in-tree with nvcc for sm_100a (no torch JIT, no pip install)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpqr.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl  # torch-bundled NCCL (2.28)

    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return [os.path.join(CSRC, f) for f in ("pqr_api.cu", "stream2_fused.cu", "stream2_gram.cu", "stream2_update.cu")]


def deps():
    return sorted(glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(ROOT, "include", "*.h")))


def build(force: bool = False, verbose: bool = False, trace: bool = False, defines=(), out: str = LIB) -> str:
    """trace=True compiles the TSQR phase counters in (PQR_WY_TRACE=1 then prints them);
    defines: extra -D flags (tuning builds, e.g. -DPQR_WY_WARPS=8); out: library path (A/B builds)."""
    if out == LIB and not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in deps()):
            return LIB
    inc, lib = nccl_dirs()
    tmp = out + f".tmp{os.getpid()}"
    # one object per translation unit, compiled in parallel, then linked
    import concurrent.futures
    import tempfile

    odir = tempfile.mkdtemp(prefix="pqr_build_")
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
             "-I", inc, "-I", os.path.join(ROOT, "include"), *(["-DPQR_WY_TRACE"] if trace else []), *defines]
    objs = [os.path.join(odir, os.path.basename(src) + ".o") for src in sources()]

    def cc(pair):
        src, obj = pair
        subprocess.check_call([NVCC, *flags, "-c", src, "-o", obj])

    with concurrent.futures.ThreadPoolExecutor(max_workers=len(objs)) as ex:
        list(ex.map(cc, zip(sources(), objs)))
    subprocess.check_call([NVCC, *ARCH, "-shared", *objs, "-o", tmp, "-L", lib, "-l:libnccl.so.2",
                           f"-Xlinker=-rpath,{lib}", "-lcudart"])
    for o in objs:
        os.remove(o)
    os.rmdir(odir)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv,
                defines=[a for a in sys.argv[1:] if a.startswith("-D")]))
