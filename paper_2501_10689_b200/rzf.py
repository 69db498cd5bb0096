"""Batched direct RZF on the GPU (drop-in for pkg/src/kaczprec/rzf.py).

`kz_rzf` forms the Gram H^H H + reg I from the packed VR rows (never the dense
H), factors it by Cholesky, inverts it and assembles F = beta H V with
||F||_F = 1, all in complex128 (rzf.py:38-83).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .batch import DeviceBatch, HostBatch


@dataclass(frozen=True)
class Precoder:
    """rzf.py:19-29."""

    f: np.ndarray
    norm_factor: float
    scheme: str = ""


class _DenseSystem:
    """Minimal AugmentedSystem-like view of a plain (Nt, K) channel for batching."""

    def __init__(self, h, reg, vrs=None):
        from .vrgraph import UserPartition
        h = np.asarray(h)
        self.n_antennas, self.n_users = h.shape
        self.reg = float(reg)
        if vrs is None:
            self.supports = tuple(np.arange(self.n_antennas) for _ in range(self.n_users))
        else:
            self.supports = tuple(np.asarray(vr.antenna_indices) for vr in vrs)
        self.eff_rows = tuple(np.ascontiguousarray(h[s, i]) for i, s in enumerate(self.supports))
        self.row_energies = np.array([np.sum(np.abs(e) ** 2) for e in self.eff_rows]) + self.reg
        k = self.n_users
        self.partition = UserPartition(frozenset(), tuple(range(k)), tuple(frozenset({i}) for i in range(k)))


def _channel_parts(h):
    if hasattr(h, "vrs") and hasattr(h, "h"):
        return np.asarray(h.h), h.vrs
    return np.asarray(h), None


def rzf_batched(dev: DeviceBatch, want_f: bool = False, stream=None) -> dict:
    """V (B,K,K) c128, beta (B,), optional F (B,Nt,K) c128 for every system of `dev`."""
    import torch
    lb = _lib.lib()
    b, k, nt = dev.n_systems, dev.n_users, dev.n_antennas
    d = dev.device
    v = torch.zeros((b, k, k), dtype=torch.complex128, device=d)
    beta = torch.zeros(b, dtype=torch.float64, device=d)
    ok = torch.zeros(b, dtype=torch.uint8, device=d)
    f = torch.zeros((b, nt, k), dtype=torch.complex128, device=d) if want_f else None
    need = lb.kz_rzf_workspace_bytes(C.byref(dev.problem))
    ws = torch.empty(max(need, 1), dtype=torch.uint8, device=d)
    s = stream if stream is not None else torch.cuda.current_stream()
    _lib.check(lb.kz_rzf(C.byref(dev.problem), v.data_ptr(), None if f is None else f.data_ptr(), beta.data_ptr(),
                         ok.data_ptr(), ws.data_ptr(), ws.numel(), C.c_void_p(s.cuda_stream)))
    return {"v": v, "beta": beta, "pd_ok": ok, "f": f, "launches": lb.kz_last_launch_count()}


def _single(h, reg):
    if reg < 0.0:
        raise ValueError("regularisation must be non-negative")
    arr, vrs = _channel_parts(h)
    dev = HostBatch.from_systems([_DenseSystem(arr, reg, vrs)]).to_device("c128")
    out = rzf_batched(dev, want_f=True)
    if not bool(out["pd_ok"][0]):
        raise np.linalg.LinAlgError(
            "Gram matrix is not positive definite; the channel is rank deficient and reg = 0")
    return out


def auxiliary_matrix(h, reg: float) -> np.ndarray:
    """(H^H H + reg I)^{-1} (rzf.py:63-66)."""
    return _single(h, reg)["v"][0].cpu().numpy()


def apply_auxiliary(h, reg: float, s) -> np.ndarray:
    """Solve (H^H H + reg I) v = s for a vector or block of rhs (rzf.py:43-60)."""
    return auxiliary_matrix(h, reg) @ np.asarray(s)


def rzf_precoder(h, reg: float) -> Precoder:
    """beta * H (H^H H + reg I)^{-1}, ||F||_F = 1 (rzf.py:69-83)."""
    out = _single(h, reg)
    beta = float(out["beta"][0])
    if not np.isfinite(beta):
        raise ValueError("degenerate precoder: H (H^H H + reg I)^{-1} vanished")
    return Precoder(f=out["f"][0].cpu().numpy(), norm_factor=beta, scheme="rzf")


def mrc_precoder(h) -> Precoder:
    """Matched filter H/||H||_F (rzf.py:86-93); a normalisation, not on the hot path."""
    import torch
    arr, _ = _channel_parts(h)
    t = torch.as_tensor(arr, device="cuda")
    n = float(torch.linalg.norm(t))
    if n == 0.0:
        raise ValueError("degenerate precoder: zero channel")
    return Precoder(f=(t / n).cpu().numpy(), norm_factor=1.0 / n, scheme="mrc")
