"""ctypes binding of libkaczmarz_b200.so (include/kaczmarz_b200.h).

The library is mandatory: there is no CPU fallback.  If it is missing or
fails to load, every product entry point raises `ExtensionMissingError`.
"""

from __future__ import annotations

import ctypes as C
import os

from .build import lib_path

ABI_VERSION = 8  # include/kaczmarz_b200.h KZ_ABI_VERSION: the struct layouts below follow it

KZ_OK = 0
KZ_ERR_INVALID = -1
KZ_ERR_CUDA = -2
KZ_ERR_NOT_PD = -3
KZ_ERR_WORKSPACE = -4

SCHEME_IDS = {"urk": 0, "swor-erk": 1, "gk": 2, "grk": 3, "vr-ogrk": 4, "ahk": 5, "vr-oahk": 6, "vr-oahk-g": 7}
KZ_C128, KZ_C64 = 0, 1
KZ_PROBLEM_CONTIGUOUS, KZ_PROBLEM_GRAM_CACHED = 1, 2  # kz_problem.flags
STOP_LOCKSTEP, STOP_RESIDUAL, STOP_ORACLE = 0, 1, 2
RNG_NONE, RNG_HOST_UNIFORM, RNG_HOST_INDEX, RNG_PHILOX = 0, 1, 2, 3

P = C.c_void_p


class KzProblem(C.Structure):
    _fields_ = [
        ("n_systems", C.c_int32), ("n_users", C.c_int32), ("n_antennas", C.c_int32), ("dtype", C.c_int32),
        ("row_seg_ptr", P), ("seg_start", P), ("seg_len", P), ("row_val_ptr", P), ("heff", P),
        ("row_energy", P), ("reg", P),
        ("coupled_ptr", P), ("coupled_idx", P), ("orth_ptr", P), ("orth_idx", P),
        ("non_ptr", P), ("non_idx", P), ("non_union_size", P),
        ("max_support", C.c_int32), ("flags", C.c_int32),
        ("slice_pairs_128", C.c_int32), ("slice_pairs_256", C.c_int32),
        ("slice_rows_128", C.c_int32), ("slice_rows_256", C.c_int32),
        ("ogrp_sys", P), ("ogrp_ptr", P), ("agg_cap", C.c_int32), ("_pad0", C.c_int32),
        ("val_lo", C.c_int64), ("val_hi", C.c_int64),
    ]


class KzStop(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("max_iters", C.c_int32), ("check_every", C.c_int32), ("_pad", C.c_int32),
        ("epsilon", C.c_double), ("f_ref", P), ("v_ref", P), ("rhs_mask", P),
    ]


class KzRng(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("stream_len", C.c_int32), ("stream_base", C.c_int64),
        ("uniforms", P), ("indices", P), ("seed", C.c_uint64), ("system_base", C.c_int64),
    ]


class KzDrop(C.Structure):
    _fields_ = [
        ("n_systems", C.c_int32), ("n_users", C.c_int32), ("n_antennas", C.c_int32), ("dtype", C.c_int32),
        ("element_spacing", C.c_double), ("wavelength", P), ("r0", P), ("theta", P), ("vr_start", P),
        ("vr_len", P), ("reg", P),
    ]


class KzOut(C.Structure):
    _fields_ = [
        ("v", P), ("iters", P), ("converged", P), ("done", P), ("noop_steps", P), ("flops", P),
        ("n_outer", P), ("sys_converged", P), ("paused", P), ("rows", P),
        ("rows_cap", C.c_int32), ("trace_cap", C.c_int32),
        ("nmse_trace", P), ("resid_trace", P), ("flops_trace", P), ("n_checks", P), ("iterates", P),
    ]


class ExtensionMissingError(RuntimeError):
    """The CUDA extension is not built or cannot be loaded; there is no fallback."""


class KzError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"kz status {code}: {msg}")
        self.code = code


_LIB = None


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    LIB_PATH = lib_path(os.environ.get("KZ_LIB_VARIANT", ""))
    if not os.path.exists(LIB_PATH):
        raise ExtensionMissingError(
            f"{LIB_PATH} not found; build it with `python -m paper_2501_10689_b200.build` "
            "(there is no CPU fallback for the product path)")
    try:
        import torch  # noqa: F401  (initialises the CUDA runtime/driver first)
        lb = C.CDLL(LIB_PATH)
    except OSError as exc:
        raise ExtensionMissingError(f"cannot load {LIB_PATH}: {exc}") from exc
    _declare(lb)
    if lb.kz_abi_version() != ABI_VERSION:
        raise ExtensionMissingError(f"{LIB_PATH} has ABI {lb.kz_abi_version()}, this binding expects {ABI_VERSION}; "
                                    "rebuild it with `python -m paper_2501_10689_b200.build`")
    _LIB = lb
    return lb


EXPORTS = (
    "kz_abi_version", "kz_last_error", "kz_last_launch_count", "kz_last_tma_staging",
    "kz_solve_workspace_bytes", "kz_solve_workspace_bytes_for", "kz_solve_resid_offset", "kz_solve",
    "kz_rzf_workspace_bytes", "kz_rzf", "kz_epilogue_workspace_bytes", "kz_epilogue_uses_gram", "kz_epilogue",
    "kz_channel_synth", "kz_partition_counts", "kz_partition_fill",
    "kz_residual_refresh", "kz_project_rows", "kz_ahk_step",
)


def _declare(lb):
    lb.kz_abi_version.restype = C.c_int32
    lb.kz_last_error.restype = C.c_char_p
    lb.kz_last_launch_count.restype = C.c_int32
    lb.kz_last_tma_staging.restype = C.c_int32
    lb.kz_solve_workspace_bytes.restype = C.c_size_t
    lb.kz_solve_workspace_bytes.argtypes = [C.POINTER(KzProblem), C.POINTER(KzStop)]
    lb.kz_solve_workspace_bytes_for.restype = C.c_size_t
    lb.kz_solve_workspace_bytes_for.argtypes = [C.POINTER(KzProblem), C.c_int32, C.POINTER(KzStop),
                                                C.POINTER(KzRng), C.POINTER(KzOut)]
    lb.kz_solve_resid_offset.restype = C.c_size_t
    lb.kz_solve_resid_offset.argtypes = [C.POINTER(KzProblem)]
    lb.kz_solve.restype = C.c_int
    lb.kz_solve.argtypes = [C.POINTER(KzProblem), C.c_int32, C.POINTER(KzStop), C.POINTER(KzRng),
                            C.POINTER(KzOut), P, C.c_size_t, C.c_int32, P]
    lb.kz_rzf_workspace_bytes.restype = C.c_size_t
    lb.kz_rzf_workspace_bytes.argtypes = [C.POINTER(KzProblem)]
    lb.kz_rzf.restype = C.c_int
    lb.kz_rzf.argtypes = [C.POINTER(KzProblem), P, P, P, P, P, C.c_size_t, P]
    lb.kz_epilogue_workspace_bytes.restype = C.c_size_t
    lb.kz_epilogue_workspace_bytes.argtypes = [C.POINTER(KzProblem)]
    lb.kz_epilogue_uses_gram.restype = C.c_int32
    lb.kz_epilogue_uses_gram.argtypes = [C.POINTER(KzProblem), C.c_int32]
    lb.kz_epilogue.restype = C.c_int
    lb.kz_epilogue.argtypes = [C.POINTER(KzProblem), P, P, P, P, P, P, P, P, P, P, C.c_size_t, P]
    lb.kz_channel_synth.restype = C.c_int
    lb.kz_channel_synth.argtypes = [C.POINTER(KzDrop), P, P, P, P]
    lb.kz_partition_counts.restype = C.c_int
    lb.kz_partition_counts.argtypes = [C.POINTER(KzDrop), P, P, P, P, P]
    lb.kz_partition_fill.restype = C.c_int
    lb.kz_partition_fill.argtypes = [C.POINTER(KzDrop), P, P, P, P, P, P, P]
    i32 = C.c_int32
    lb.kz_residual_refresh.restype = C.c_int
    lb.kz_residual_refresh.argtypes = [C.POINTER(KzProblem), i32, i32, P, P, P, P, i32, i32, P]
    lb.kz_project_rows.restype = C.c_int
    lb.kz_project_rows.argtypes = [C.POINTER(KzProblem), i32, P, P, P, P, i32, P]
    lb.kz_ahk_step.restype = C.c_int
    lb.kz_ahk_step.argtypes = [C.POINTER(KzProblem), i32, P, P, P, P, P, i32, P, i32, P, P]


def check(status: int):
    if status != KZ_OK:
        msg = lib().kz_last_error().decode(errors="replace")
        raise KzError(status, msg)


def ptr(t):
    """Device pointer of a torch tensor (or None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())
