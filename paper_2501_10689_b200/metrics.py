"""NMSE and Eq. (7) sum-rate on the GPU (drop-in for pkg/src/kaczprec/metrics.py:44-78).

Inside the batched path these are fused into `kz_epilogue`; the functions here
serve the reference signatures for precoders the caller already holds.
"""

from __future__ import annotations

import numpy as np

CMUL = 6
CADD = 2


def _t(x):
    import torch
    return torch.as_tensor(np.asarray(x), device="cuda")


def nmse(f, f_ref) -> float:
    """||F_ref - F||_F / ||F_ref||_F (metrics.py:44-51)."""
    import torch
    fr = _t(f_ref)
    den = float(torch.linalg.norm(fr))
    if den == 0.0:
        raise ValueError("reference precoder has zero norm")
    return float(torch.linalg.norm(fr - _t(f).to(fr.dtype))) / den


def spectral_efficiency(h, f, snr_linear: float):
    """Per-user rates and their sum for a unit-power precoder (metrics.py:54-78)."""
    import torch
    h = np.asarray(h)
    f = np.asarray(f)
    if h.shape != f.shape:
        raise ValueError(f"shape mismatch: channel {h.shape} vs precoder {f.shape}")
    if snr_linear <= 0.0:
        raise ValueError("snr_linear must be positive")
    ht, ft = _t(h).to(torch.complex128), _t(f).to(torch.complex128)
    total = float(torch.linalg.norm(ft))
    if total > 1.0 + 1e-9:
        raise ValueError(f"precoder violates the unit power budget: ||F||_F = {total}")
    power = (ht.conj().T @ ft).abs() ** 2
    signal = torch.diagonal(power)
    interference = power.sum(dim=1) - signal
    rates = torch.log2(1.0 + signal / (interference + 1.0 / snr_linear)).cpu().numpy()
    return rates, float(rates.sum())
