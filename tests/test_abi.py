"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
header declares (CPU only: no compute calls)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kaczmarz_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kz_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2501_10689_b200.build import LIB_PATH, build
    if not os.path.exists(LIB_PATH):
        build()
    return LIB_PATH


def test_header_declares_the_boundary():
    fns = declared_functions()
    for name in ("kz_solve", "kz_rzf", "kz_epilogue", "kz_solve_workspace_bytes", "kz_last_error"):
        assert name in fns


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name


def test_python_binding_lists_the_exports(libpath):
    from paper_2501_10689_b200 import _lib
    assert set(_lib.EXPORTS) == set(declared_functions())
    lb = _lib.lib()
    assert lb.kz_abi_version() == _lib.ABI_VERSION == 8


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    """ctypes mirrors of the ABI structs have the header's field order and sizes."""
    from paper_2501_10689_b200 import _lib
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for cname, py in (("kz_problem", _lib.KzProblem), ("kz_stop", _lib.KzStop), ("kz_rng", _lib.KzRng),
                      ("kz_out", _lib.KzOut), ("kz_drop", _lib.KzDrop)):
        body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (cname, cname), src, flags=re.S).group(1)
        names = re.findall(r"\b([a-z_0-9]+)\s*;", body)
        assert names == [f[0] for f in py._fields_], cname


def test_errors_without_gpu_are_reported_not_crashing(libpath):
    from paper_2501_10689_b200 import _lib
    lb = _lib.lib()
    p = _lib.KzProblem()
    p.n_systems, p.n_users, p.n_antennas, p.dtype = 1, 0, 8, 0
    st = _lib.KzStop()
    st.max_iters = 1
    st.check_every = 1
    rc = lb.kz_solve(ctypes.byref(p), 3, ctypes.byref(st), ctypes.byref(_lib.KzRng()), ctypes.byref(_lib.KzOut()),
                     None, 0, 0, None)
    assert rc == _lib.KZ_ERR_INVALID
    assert b"user" in lb.kz_last_error()
    p.n_users = 4
    rc = lb.kz_solve(ctypes.byref(p), 9, ctypes.byref(st), ctypes.byref(_lib.KzRng()), ctypes.byref(_lib.KzOut()),
                     None, 0, 0, None)
    assert rc == _lib.KZ_ERR_INVALID
