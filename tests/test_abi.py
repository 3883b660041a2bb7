"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol
include/*.h declares; the binding's names mirror the C names; argument validation
that needs no GPU.  (No compute calls without a GPU.)"""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?\w[\w\s\*]*?\b(pqr_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return sorted(names)


@pytest.fixture(scope="module")
def libpqr():
    from paper_2204_13393_b200 import build, pqr

    build.build()
    return pqr.lib()


def test_headers_declare_the_four_calls():
    names = declared_functions()
    for f in ("pqr_create", "pqr_project_normalize", "pqr_basis_apply", "pqr_destroy"):
        assert f in names


def test_library_exports_every_declared_symbol(libpqr):
    so = os.path.join(ROOT, "paper_2204_13393_b200", "libpqr.so")
    out = subprocess.check_output(["nm", "-D", "--defined-only", so]).decode()
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    for f in declared_functions():
        assert hasattr(libpqr, f)


def test_binding_mirrors_c_names(libpqr):
    from paper_2204_13393_b200 import pqr

    for f in ("pqr_create", "pqr_project_normalize", "pqr_basis_apply", "pqr_destroy", "pqr_get_stats"):
        assert callable(getattr(pqr, f))


def test_strerror_and_argument_errors(libpqr):
    from paper_2204_13393_b200 import pqr

    assert pqr.strerror(0) == "ok"
    assert "capacity" in pqr.strerror(pqr.PQR_ECAPACITY)
    # invalid configs are rejected before touching the device
    h = ctypes.c_void_p()
    cfg = pqr.pqr_config()
    cfg.n_local = 0
    cfg.s_max = 4
    cfg.nranks = 1
    assert libpqr.pqr_create(ctypes.byref(h), ctypes.byref(cfg), None, 1, 0) == pqr.PQR_EARG
    cfg.n_local = 100
    cfg.s_max = 17  # > 16
    assert libpqr.pqr_create(ctypes.byref(h), ctypes.byref(cfg), None, 1, 0) == pqr.PQR_EARG
    cfg.s_max = 8
    cfg.k_max = 200  # k_max + s_max > 160
    assert libpqr.pqr_create(ctypes.byref(h), ctypes.byref(cfg), None, 1, 0) == pqr.PQR_ECAPACITY
    cfg.k_max = 8
    cfg.nranks = 2  # multi-rank without an NCCL id
    assert libpqr.pqr_create(ctypes.byref(h), ctypes.byref(cfg), None, 1, 0) == pqr.PQR_EARG
    assert libpqr.pqr_project_normalize(None, None, 1, 1, 0, None, 1, None, 1, None, 1, None) == pqr.PQR_EARG
    assert libpqr.pqr_destroy(None) == 0


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_2204_13393_b200 import pqr

    monkeypatch.setattr(pqr, "_lib", None)
    monkeypatch.setattr(pqr, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        pqr.lib()


def test_sm100a_code_in_library(libpqr):
    so = os.path.join(ROOT, "paper_2204_13393_b200", "libpqr.so")
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-lelf", so]).decode()
    assert "sm_100a" in out
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", so]).decode()
    assert "DMMA" in sass  # fp64 tensor-core path of the Gram / update kernels
