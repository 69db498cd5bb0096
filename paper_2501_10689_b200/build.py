"""Build libkaczmarz_b200.so in-tree with nvcc for sm_100a.

The shared library is the product: a C ABI (include/kaczmarz_b200.h) over
hand-written CUDA kernels.  It is built next to this file so it travels with
the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_NAME = "libkaczmarz_b200.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)
# variant "timing": per-phase clock64 accounting in the lockstep kernels (-DKZ_TIMING)
# variant "checked": bounds checks on every on-chip index the kernels compute (-DKZ_CHECKED, kz_common.cuh)
VARIANTS = {"": [], "timing": ["-DKZ_TIMING"], "checked": ["-DKZ_CHECKED"]}


def lib_path(variant: str = "") -> str:
    return LIB_PATH if not variant else os.path.join(HERE, f"libkaczmarz_b200_{variant}.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # numpy-faithful selection arithmetic: no implicit mul+add contraction;
    # every FMA in the kernels is written explicitly.
    "--fmad=false",
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC,-O2",
]

SOURCES = ["kz_api.cu"]


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if os.path.exists(cand) else "nvcc"


def _inputs():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "kaczmarz_b200.h"))
    files.append(os.path.abspath(__file__))
    return files


def up_to_date(variant: str = "") -> bool:
    path = lib_path(variant)
    if not os.path.exists(path):
        return False
    t = os.path.getmtime(path)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def build(force: bool = False, verbose: bool = False, variant: str = "") -> str:
    path = lib_path(variant)
    if not force and up_to_date(variant):
        return path
    tmp = path + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, *VARIANTS[variant], "-I", os.path.join(ROOT, "include"),
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-8000:])
        raise RuntimeError(f"nvcc failed (exit {res.returncode}); see {log}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, path)
    return path


if __name__ == "__main__":
    var = "timing" if "--timing" in sys.argv else ("checked" if "--checked" in sys.argv else "")
    print(build(force="--force" in sys.argv, verbose=True, variant=var))
