"""Precoder assembly / epilogue on the GPU (drop-in for pkg/src/kaczprec/assembly.py).

`kz_epilogue` computes, per system, F = beta H V with beta = 1/||H V||_F over
the rows covering each antenna (assemble_vr's blocked product with one-antenna
blocks, equal to assemble_dense's H V because H is zero off-support), plus the
NMSE against beta_ref H V_ref and the Eq. (7) rates — the per-system scalars
gathered across GPUs.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .batch import DeviceBatch, HostBatch


def epilogue(dev: DeviceBatch, v, *, v_ref=None, beta_ref=None, rates: bool = False, snr_linear=None,
             want_f: bool = False, stream=None, workspace=None, gram_cached: bool = False) -> dict:
    """F / NMSE / sum-rate of the solutions v [B][K][K] (kz_epilogue).  `workspace` (uint8 device tensor, e.g.
    the "workspace" of an earlier result) is reused when large enough; with gram_cached=True it must hold the
    Gram G0 = H^H H of this batch from an earlier Gram-form call on the same workspace (several V of one batch,
    one stream), which is then not recomputed.  The result's "workspace" can be passed back."""
    import torch
    lb = _lib.lib()
    b, k, nt = dev.n_systems, dev.n_users, dev.n_antennas
    d = dev.device
    v = v.to(dev.complex_dtype).contiguous()
    f = torch.zeros((b, nt, k), dtype=dev.complex_dtype, device=d) if want_f else None
    beta = torch.zeros(b, dtype=torch.float64, device=d)
    nm = torch.full((b,), float("nan"), dtype=torch.float64, device=d) if v_ref is not None else None
    keep = []
    if v_ref is not None:
        v_ref = torch.as_tensor(v_ref).to(device=d, dtype=torch.complex128).contiguous()
        beta_ref = torch.as_tensor(beta_ref).to(device=d, dtype=torch.float64).contiguous()
        keep += [v_ref, beta_ref]
    snr = None
    if rates:
        snr = snr_linear if snr_linear is not None else dev.t.get("snr_linear")
        if snr is None:
            raise ValueError("rates need snr_linear (batch built without it)")
        snr = torch.as_tensor(snr).to(device=d, dtype=torch.float64).contiguous()
        keep.append(snr)
    r = torch.zeros((b, k), dtype=torch.float64, device=d) if rates else None
    sr = torch.zeros(b, dtype=torch.float64, device=d) if rates else None
    # the library decides the form (kz_epilogue_uses_gram); the Gram form always needs its G0 / G0 V workspace
    gram_form = bool(lb.kz_epilogue_uses_gram(C.byref(dev.problem), 1 if want_f else 0))
    need = lb.kz_epilogue_workspace_bytes(C.byref(dev.problem)) if (rates or gram_form) else 0
    # a workspace holding G0 is stamped with the batch it was formed for; gram_cached accepts only that batch
    stamp = (dev.problem.heff, dev.problem.row_val_ptr, b, k, nt, id(dev))
    if gram_cached and (workspace is None or getattr(workspace, "_kz_gram_of", None) != stamp):
        raise ValueError("gram_cached needs the workspace of an earlier Gram-form epilogue of this batch")
    if workspace is not None and workspace.numel() >= need:
        ws = workspace
    else:
        ws = torch.empty(max(need, 1), dtype=torch.uint8, device=d)
    prob = dev.problem
    if gram_cached and gram_form:
        prob = type(dev.problem).from_buffer_copy(dev.problem)
        prob.flags |= _lib.KZ_PROBLEM_GRAM_CACHED
    s = stream if stream is not None else torch.cuda.current_stream()
    P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    _lib.check(lb.kz_epilogue(C.byref(prob), v.data_ptr(), P(f), P(v_ref), P(beta_ref), P(snr),
                              beta.data_ptr(), P(nm), P(r), P(sr), ws.data_ptr(), ws.numel(),
                              C.c_void_p(s.cuda_stream)))
    ws._kz_gram_of = stamp if gram_form else None
    return {"f": f, "beta": beta, "nmse": nm, "rates": r, "sum_rate": sr, "launches": lb.kz_last_launch_count(),
            "workspace": ws, "gram_form": gram_form}


@dataclass(frozen=True)
class SubarrayChannel:
    """assembly.py:20-48: the channel as S row blocks with the users active on each block."""

    blocks: tuple
    active_users: tuple
    n_users: int

    @classmethod
    def from_channel(cls, chan) -> "SubarrayChannel":
        h = np.asarray(chan.h)
        s_count, m = chan.cfg.n_subarrays, chan.cfg.subarray_size
        blocks, active = [], []
        for s in range(s_count):
            block = h[s * m:(s + 1) * m, :]
            users = np.asarray(sorted(k for k, vr in enumerate(chan.vrs) if s in vr.visible_subarrays),
                               dtype=np.intp)
            inactive = np.setdiff1d(np.arange(h.shape[1]), users)
            if inactive.size and np.any(block[:, inactive] != 0.0):
                raise ValueError(f"subarray {s}: channel is nonzero for a user outside its visibility region")
            blocks.append(block)
            active.append(users)
        return cls(blocks=tuple(blocks), active_users=tuple(active), n_users=h.shape[1])


class _VrSystem:
    """Batch view of a ChannelMatrix (VR supports) or a SubarrayChannel (block supports) for the epilogue."""

    def __init__(self, chan):
        from .vrgraph import UserPartition
        if hasattr(chan, "blocks"):  # SubarrayChannel: user k is supported on the blocks listing it
            h = np.vstack(chan.blocks)
            starts = np.cumsum([0] + [b.shape[0] for b in chan.blocks])
            sup = [[] for _ in range(chan.n_users)]
            for s, users in enumerate(chan.active_users):
                for k in np.asarray(users).tolist():
                    sup[k].append(np.arange(starts[s], starts[s + 1]))
            supports = tuple(np.concatenate(x) if x else np.zeros(0, np.intp) for x in sup)
        else:
            h = np.asarray(chan.h)
            supports = tuple(np.asarray(vr.antenna_indices) for vr in chan.vrs)
        self.h = h
        self.n_antennas, self.n_users = h.shape
        self.reg = 0.0
        self.supports = supports
        self.eff_rows = tuple(np.ascontiguousarray(h[s, i]) for i, s in enumerate(self.supports))
        self.row_energies = np.array([np.sum(np.abs(e) ** 2) for e in self.eff_rows])
        k = self.n_users
        self.partition = UserPartition(frozenset(), tuple(range(k)), tuple(frozenset({i}) for i in range(k)))


def _assemble(chan, v, counter, scheme, blocked):
    from .rzf import Precoder, _DenseSystem
    vr_view = hasattr(chan, "vrs") or hasattr(chan, "blocks")
    sysv = _VrSystem(chan) if vr_view else None
    h = sysv.h if vr_view else np.asarray(chan.h if hasattr(chan, "h") else chan)
    nt, k = h.shape
    v = np.asarray(v)
    if v.shape != (k, k):
        raise ValueError(f"expected a ({k}, {k}) solution block, got {v.shape}")
    if sysv is None:
        sysv = _DenseSystem(h, 0.0)
    dev = HostBatch.from_systems([sysv]).to_device("c128")
    import torch
    ep = epilogue(dev, torch.as_tensor(v[None], dtype=torch.complex128, device="cuda"), want_f=True)
    beta = float(ep["beta"][0])
    if not np.isfinite(beta):
        raise ValueError("degenerate precoder: H V vanished")
    if counter is not None:
        if blocked and hasattr(chan, "blocks"):
            for block, users in zip(chan.blocks, chan.active_users):
                m, q = block.shape[0], int(np.asarray(users).size)
                if q:
                    counter.total += 6 * m * q * k + 2 * m * (q - 1) * k
        elif blocked:
            m = chan.cfg.subarray_size
            for s in range(chan.cfg.n_subarrays):
                q = sum(1 for vr in chan.vrs if s in vr.visible_subarrays)
                if q:
                    counter.total += 6 * m * q * k + 2 * m * (q - 1) * k
        else:
            counter.total += 6 * nt * k * k + 2 * nt * k * (k - 1)
    return Precoder(f=ep["f"][0].cpu().numpy(), norm_factor=beta, scheme=scheme)


def assemble_dense(chan, v, counter=None, scheme: str = ""):
    """F = H V then unit-power normalisation (assembly.py:59-71)."""
    return _assemble(chan, v, counter, scheme, blocked=False)


def assemble_vr(sub, v, counter=None, scheme: str = ""):
    """Subarray-blocked F = H V (assembly.py:74-92).  Takes the reference's SubarrayChannel (or this
    package's), or the ChannelMatrix itself (its VR supports give the same blocking)."""
    return _assemble(sub, v, counter, scheme, blocked=True)
