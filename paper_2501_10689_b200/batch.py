"""Packing B independent systems into the flat device layout of kz_problem.

Host side (numpy) builds the CSR-style arrays once; `to_device` uploads them
as torch tensors and fills the ctypes `KzProblem` with their device pointers.
Layout in HBM:

  heff         complex[n_val]   rows packed back to back, row r = b*K + i
  row_val_ptr  int64[B*K+1]     offset of row r in heff
  row_seg_ptr  int32[B*K+1]     row r's support segments (one per contiguous run)
  seg_start    int32[n_seg]     first antenna of each segment
  seg_len      int32[n_seg]
  row_energy   float64[B*K]     ||h_r||^2 + reg_b
  reg          float64[B]
  coupled/orth/non CSR          the VR partition (vrgraph.py:84-114)
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C

import os

import numpy as np

from . import _lib
from .vrgraph import greedy_mis, grouped_mis, overlap_from_intervals, overlap_from_segments


def _union_size_intervals(start, length):
    if len(start) == 0:
        return 0
    order = np.argsort(start, kind="stable")
    s = np.asarray(start)[order].astype(np.int64)
    e = s + np.asarray(length)[order].astype(np.int64)
    tot, cur_s, cur_e = 0, int(s[0]), int(e[0])
    for a, b in zip(s[1:], e[1:]):
        if a <= cur_e:
            cur_e = max(cur_e, int(b))
        else:
            tot += cur_e - cur_s
            cur_s, cur_e = int(a), int(b)
    return tot + cur_e - cur_s


def cluster_blocks(warps: int) -> int:
    """Chunk blocks per CTA of the cluster kernel's interleaved layout (must match kz_solve_cluster.cuh:
    KZ_CLUSTER_NBLK, default 2)."""
    n = int(os.environ.get("KZ_CLUSTER_NBLK", "2"))
    return n if n > 0 and warps % n == 0 else 2


@dataclass
class HostBatch:
    n_systems: int
    n_users: int
    n_antennas: int
    row_seg_ptr: np.ndarray
    seg_start: np.ndarray
    seg_len: np.ndarray
    row_val_ptr: np.ndarray
    heff: np.ndarray
    row_energy: np.ndarray
    reg: np.ndarray
    coupled_ptr: np.ndarray
    coupled_idx: np.ndarray
    orth_ptr: np.ndarray
    orth_idx: np.ndarray
    non_ptr: np.ndarray
    non_idx: np.ndarray
    non_union_size: np.ndarray
    contiguous: bool
    snr_linear: np.ndarray | None = None
    # orthogonal groups (grouped VR-OAHK, kz_problem.ogrp_*): system b's groups are [ogrp_ptr[j], ogrp_ptr[j+1])
    # for j in [ogrp_sys[b], ogrp_sys[b+1]) (absolute offsets into orth_idx); None = one group per system
    ogrp_sys: np.ndarray | None = None
    ogrp_ptr: np.ndarray | None = None
    orth_groups: int = 1      # groups built per system (1: the reference's single orthogonal set)
    agg_cap: int = 0          # hyperplanes per aggregated step of vr-oahk-g (0: all non-orthogonal rows)

    def __post_init__(self):
        if self.ogrp_sys is None:  # one group per system: the reference's orthogonal set
            self.ogrp_sys = np.arange(self.n_systems + 1, dtype=np.int32)
            self.ogrp_ptr = np.asarray(self.orth_ptr, dtype=np.int32).copy()

    # ------------------------------------------------------------ builders
    @classmethod
    def from_contiguous(cls, ch, partition: bool = True, orth_groups: int = 1, agg_cap: int = 0) -> "HostBatch":
        """From `channel.ContiguousChannels` (one segment per user).  orth_groups > 1 builds the orthogonal row
        groups of the grouped VR-OAHK variant (vrgraph.grouped_mis; the orthogonal set then holds every group and
        is NOT one mutually orthogonal set, so plain vr-oahk refuses such a batch); agg_cap = hyperplanes per
        aggregated step of vr-oahk-g (0 = all non-orthogonal rows at once)."""
        b, k = ch.start.shape
        rows = b * k
        lens = ch.length.reshape(-1).astype(np.int64)
        if np.all(lens == lens[0]):
            e = np.sum(np.abs(ch.heff.reshape(rows, int(lens[0]))) ** 2, axis=1)
        else:
            e = np.array([np.sum(np.abs(ch.heff[ch.row_val_ptr[r]:ch.row_val_ptr[r + 1]]) ** 2)
                          for r in range(rows)])
        energy = e + np.repeat(ch.reg, k)
        cp, ci, op, oi, np_, ni, nu = [0], [], [0], [], [0], [], []
        gs, gp = [0], [0]
        if partition:
            for s in range(b):
                adj = overlap_from_intervals(ch.start[s], ch.length[s])
                groups = grouped_mis(adj, orth_groups) if orth_groups > 1 else [greedy_mis(adj)]
                orth = np.concatenate(groups)
                for g in groups:
                    gp.append(gp[-1] + len(g))
                gs.append(len(gp) - 1)
                in_o = np.zeros(k, dtype=bool)
                in_o[orth] = True
                non = np.flatnonzero(~in_o)
                for i in range(k):
                    x = np.flatnonzero(adj[i] | (np.arange(k) == i))
                    ci.extend(x.tolist())
                    cp.append(len(ci))
                oi.extend(orth.tolist())
                op.append(len(oi))
                ni.extend(non.tolist())
                np_.append(len(ni))
                nu.append(_union_size_intervals(ch.start[s][non], ch.length[s][non]))
        else:
            cp = [0] * (rows + 1)
            op = [0] * (b + 1)
            np_ = [0] * (b + 1)
            nu = [0] * b
            gs, gp = list(range(b + 1)), [0] * (b + 1)
        i32 = lambda a: np.asarray(a, dtype=np.int32)  # noqa: E731
        return cls(b, k, ch.n_antennas, np.arange(rows + 1, dtype=np.int32), i32(ch.start.reshape(-1)),
                   i32(ch.length.reshape(-1)), ch.row_val_ptr.astype(np.int64), ch.heff.astype(np.complex128),
                   energy, np.asarray(ch.reg, dtype=np.float64), i32(cp), i32(ci), i32(op), i32(oi), i32(np_),
                   i32(ni), i32(nu), True, np.asarray(ch.snr_linear, dtype=np.float64), i32(gs), i32(gp),
                   max(1, orth_groups), int(agg_cap))

    @classmethod
    def from_systems(cls, systems, snr_linear=None) -> "HostBatch":
        """From AugmentedSystem-like objects (reference or this package): uses their
        supports, eff_rows, row_energies, reg and partition as-is."""
        b = len(systems)
        k, nt = systems[0].n_users, systems[0].n_antennas
        seg_ptr, seg_s, seg_l, val_ptr, vals = [0], [], [], [0], []
        energy, reg = [], []
        cp, ci, op, oi, np_, ni, nu = [0], [], [0], [], [0], [], []
        contiguous = True
        for s in systems:
            if s.n_users != k or s.n_antennas != nt:
                raise ValueError("all systems of a batch must share (K, Nt)")
            for i in range(k):
                idx = np.asarray(s.supports[i], dtype=np.int64)
                brk = np.flatnonzero(np.diff(idx) != 1) + 1
                starts = np.concatenate([[0], brk])
                ends = np.concatenate([brk, [idx.size]])
                for a, e in zip(starts, ends):
                    seg_s.append(int(idx[a]))
                    seg_l.append(int(e - a))
                if len(starts) != 1:
                    contiguous = False
                seg_ptr.append(len(seg_s))
                vals.append(np.asarray(s.eff_rows[i], dtype=np.complex128))
                val_ptr.append(val_ptr[-1] + idx.size)
            energy.extend(np.asarray(s.row_energies, dtype=np.float64).tolist())
            reg.append(float(s.reg))
            part = s.partition
            for i in range(k):
                ci.extend(sorted(part.coupled[i]))
                cp.append(len(ci))
            orth = sorted(part.orthogonal)
            non = list(part.non_orthogonal)
            oi.extend(orth)
            op.append(len(oi))
            ni.extend(non)
            np_.append(len(ni))
            if non:
                nu.append(int(np.unique(np.concatenate([np.asarray(s.supports[i]) for i in non])).size))
            else:
                nu.append(0)
        i32 = lambda a: np.asarray(a, dtype=np.int32)  # noqa: E731
        return cls(b, k, nt, i32(seg_ptr), i32(seg_s), i32(seg_l), np.asarray(val_ptr, dtype=np.int64),
                   np.concatenate(vals), np.asarray(energy), np.asarray(reg), i32(cp), i32(ci), i32(op), i32(oi),
                   i32(np_), i32(ni), i32(nu), contiguous,
                   None if snr_linear is None else np.asarray(snr_linear, dtype=np.float64))

    @classmethod
    def concat(cls, parts) -> "HostBatch":
        """Stack batches sharing (K, Nt) (offsets rebased)."""
        k, nt = parts[0].n_users, parts[0].n_antennas

        def cat_ptr(name, base_name=None):
            out, off = [np.zeros(1, dtype=getattr(parts[0], name).dtype)], 0
            for p in parts:
                a = getattr(p, name)
                out.append(a[1:] + off)
                off += a[-1]
            return np.concatenate(out)

        if any(p.orth_groups != parts[0].orth_groups or p.agg_cap != parts[0].agg_cap for p in parts):
            raise ValueError("batches to concatenate must share orth_groups and agg_cap")
        gsys, gptr, goff, ooff = [np.zeros(1, dtype=np.int32)], [np.zeros(1, dtype=np.int32)], 0, 0
        for p in parts:
            gsys.append(p.ogrp_sys[1:] + goff)
            gptr.append(p.ogrp_ptr[1:] - p.ogrp_ptr[0] + ooff)
            goff += int(p.ogrp_sys[-1])
            ooff += int(p.orth_ptr[-1])
        return cls(sum(p.n_systems for p in parts), k, nt, cat_ptr("row_seg_ptr"),
                   np.concatenate([p.seg_start for p in parts]), np.concatenate([p.seg_len for p in parts]),
                   cat_ptr("row_val_ptr"), np.concatenate([p.heff for p in parts]),
                   np.concatenate([p.row_energy for p in parts]), np.concatenate([p.reg for p in parts]),
                   cat_ptr("coupled_ptr"), np.concatenate([p.coupled_idx for p in parts]),
                   cat_ptr("orth_ptr"), np.concatenate([p.orth_idx for p in parts]),
                   cat_ptr("non_ptr"), np.concatenate([p.non_idx for p in parts]),
                   np.concatenate([p.non_union_size for p in parts]), all(p.contiguous for p in parts),
                   None if any(p.snr_linear is None for p in parts) else np.concatenate([p.snr_linear for p in parts]),
                   np.concatenate(gsys).astype(np.int32), np.concatenate(gptr).astype(np.int32),
                   parts[0].orth_groups, parts[0].agg_cap)

    # ------------------------------------------------------------ accessors
    def val_range(self) -> tuple:
        """heff element range [lo, hi) of this batch's rows (kz_problem.val_lo / val_hi)."""
        if self.row_val_ptr.size == 0:
            return 0, 0
        return int(self.row_val_ptr[0]), int(self.row_val_ptr[-1])

    def support_sizes(self) -> np.ndarray:
        return np.diff(self.row_val_ptr).reshape(self.n_systems, self.n_users)

    def layout_hints(self) -> dict:
        """kz_problem shape hints of this batch (computed once: host packing work, not per upload)."""
        h = self.__dict__.get("_hints")
        if h is None:
            sup = np.diff(self.row_val_ptr)
            h = {"max_support": int(sup.max()) if sup.size else 0,
                 "slice_pairs_128": self.slice_pairs(128) if self.contiguous else 0,
                 "slice_pairs_256": self.slice_pairs(256) if self.contiguous else 0,
                 "slice_rows_128": self.slice_pairs(128, rows=True) if self.contiguous else 0,
                 "slice_rows_256": self.slice_pairs(256, rows=True) if self.contiguous else 0}
            self.__dict__["_hints"] = h
        return h

    def slice_pairs(self, width: int, chunk: int = 32, block: int = 1024, rows: bool = False) -> int:  # noqa: C901
        """Max over systems and CTAs of the (row, `chunk`-antenna chunk) pairs a CTA of the cluster kernel
        holds, for CTAs of `width` antennas in the block-interleaved layout of csrc/kz_solve_cluster.cuh
        (CL = ceil(Nt / width) CTAs; with CL > 1 each CTA owns two blocks of width/2 antennas, block j of
        CTA c at chunk (j CL + c) * (width/2) / chunk).  Contiguous supports only; this is the shared-memory
        layout bound kz_problem.slice_pairs_* (the kernel traps if it is exceeded).  rows=True: the number of
        rows with at least one piece in the CTA instead (kz_problem.slice_rows_*)."""
        if not self.contiguous or self.n_systems == 0:
            return 0
        w = width // chunk
        nch = self.n_antennas // chunk
        ncl = -(-nch // w)
        nblk = cluster_blocks(w) if ncl > 1 else 1
        bc = w // nblk
        # chunk ranges [lo, hi) of block j of CTA c
        lo = np.array([[(j * ncl + c) * bc for j in range(nblk)] for c in range(ncl)], dtype=np.int64)
        hi = np.minimum(lo + bc, nch)
        seg = self.row_seg_ptr[:-1]
        c0 = (self.seg_start[seg] // chunk).astype(np.int64).reshape(self.n_systems, self.n_users)
        c1 = ((self.seg_start[seg] + self.seg_len[seg] - 1) // chunk).astype(np.int64).reshape(self.n_systems,
                                                                                                 self.n_users)
        best = 0
        for s in range(0, self.n_systems, block):
            a, b = c0[s:s + block, :, None, None], c1[s:s + block, :, None, None]
            n = np.clip(np.minimum(b + 1, hi[None, None]) - np.maximum(a, lo[None, None]), 0, None)
            if rows:
                best = max(best, int((n.sum(axis=3) > 0).sum(axis=1).max()))
            else:
                best = max(best, int(n.sum(axis=(1, 3)).max()))
        return best

    def to_device(self, dtype: str = "c128", device=None) -> "DeviceBatch":
        return DeviceBatch(self, dtype, device)

    @property
    def nbytes(self) -> int:
        return sum(getattr(self, f).nbytes for f in (
            "row_seg_ptr", "seg_start", "seg_len", "row_val_ptr", "heff", "row_energy", "reg", "coupled_ptr",
            "coupled_idx", "orth_ptr", "orth_idx", "non_ptr", "non_idx", "non_union_size"))


class _HostView:
    """Shape / hint stand-in for the HostBatch of a DeviceBatch.view (the packed host arrays stay the parent's)."""

    def __init__(self, parent, n_systems: int, row0: int):
        while isinstance(parent, _HostView):  # a view of a view: rows relative to the root batch
            parent = parent.parent
        self.parent = parent
        self.n_systems = n_systems
        self.row0 = row0  # first row of the view in the root batch
        self.n_users, self.n_antennas, self.contiguous = parent.n_users, parent.n_antennas, parent.contiguous
        self.orth_groups, self.agg_cap = parent.orth_groups, parent.agg_cap

    def layout_hints(self) -> dict:
        return self.parent.layout_hints()

    def val_range(self) -> tuple:
        k, lo = self.n_users, self.row0 // self.n_users
        return int(self.parent.row_val_ptr[self.row0]), int(self.parent.row_val_ptr[(lo + self.n_systems) * k])


def pin_host(host: HostBatch, dtype: str = "c128", pin: bool = True) -> dict:
    """Host tensors of a batch (page-locked when `pin`), heff already in the compute dtype."""
    import torch
    cdt = torch.complex128 if dtype == "c128" else torch.complex64
    out = {}
    for name in DeviceBatch.FIELDS + (("snr_linear",) if host.snr_linear is not None else ()):
        t = torch.from_numpy(np.ascontiguousarray(getattr(host, name)))
        if name == "heff":
            t = t.to(cdt)
        out[name] = t.pin_memory() if pin else t
    return out


class DeviceBatch:
    """Device-resident copy of a HostBatch plus the KzProblem that points at it."""

    FIELDS = ("row_seg_ptr", "seg_start", "seg_len", "row_val_ptr", "heff", "row_energy", "reg", "coupled_ptr",
              "coupled_idx", "orth_ptr", "orth_idx", "non_ptr", "non_idx", "non_union_size", "ogrp_sys", "ogrp_ptr")

    def __init__(self, host: HostBatch, dtype: str = "c128", device=None, pinned=None):
        """Upload `host`.  `pinned` may be the dict returned by `pin_host(host, dtype)`:
        the copies then come from page-locked memory and are asynchronous on the
        current stream (the end-to-end path)."""
        import torch
        if dtype not in ("c128", "c64"):
            raise ValueError(f"dtype must be 'c128' or 'c64', got {dtype!r}")
        self.host = host
        self.dtype = dtype
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.type != "cuda":
            raise ValueError("the Kaczmarz path runs on CUDA devices only (no CPU fallback)")
        src = pinned if pinned is not None else pin_host(host, dtype, pin=False)
        self.t = {k: v.to(self.device, non_blocking=pinned is not None) for k, v in src.items()}
        self.problem = self._make_problem(self.t)

    def _make_problem(self, t):
        p = _lib.KzProblem()
        p.n_systems = self.host.n_systems
        p.n_users = self.host.n_users
        p.n_antennas = self.host.n_antennas
        p.dtype = _lib.KZ_C128 if self.dtype == "c128" else _lib.KZ_C64
        for name in self.FIELDS:
            ten = t[name]
            setattr(p, name, ten.data_ptr() if ten.numel() else None)
        hints = self.host.layout_hints()
        p.max_support = hints["max_support"]
        p.flags = 1 if self.host.contiguous else 0
        p.slice_pairs_128 = hints["slice_pairs_128"]
        p.slice_pairs_256 = hints["slice_pairs_256"]
        p.slice_rows_128 = hints["slice_rows_128"]
        p.slice_rows_256 = hints["slice_rows_256"]
        p.agg_cap = self.host.agg_cap if self.host.agg_cap > 0 else self.host.n_users
        p.val_lo, p.val_hi = self.host.val_range()  # heff element range of the rows (TMA staging bounds)
        return p

    @classmethod
    def from_drops(cls, drops, dtype: str = "c64", device=None, stream=None) -> "DeviceBatch":
        """Build the batch on the device from user drops: channel entries by
        kz_channel_synth and the VR partition by kz_partition_counts / kz_partition_fill; only the drop
        parameters (a few numbers per user) cross PCIe.  Equal to
        `HostBatch.from_contiguous(channel.generate(...)).to_device(dtype)` for the same drops."""
        import torch
        if dtype not in ("c128", "c64"):
            raise ValueError(f"dtype must be 'c128' or 'c64', got {dtype!r}")
        dev = torch.device(device if device is not None else "cuda")
        if dev.type != "cuda":
            raise ValueError("the Kaczmarz path runs on CUDA devices only (no CPU fallback)")
        # everything (uploads, kernels, the one size read-back) on `stream`: a caller can build the next batch on
        # an upload stream while the compute stream works
        s = stream if stream is not None else torch.cuda.current_stream()
        sp = C.c_void_p(s.cuda_stream)
        with torch.cuda.stream(s):
            lb = _lib.lib()
            b, k, nt = drops.n_systems, drops.n_users, drops.n_antennas
            rows = b * k
            lens = drops.length.reshape(-1).astype(np.int64)
            val_ptr = np.zeros(rows + 1, dtype=np.int64)
            np.cumsum(lens, out=val_ptr[1:])
            # the small host-side arrays (layout hints and CSR of the supports)
            host = HostBatch(b, k, nt, np.arange(rows + 1, dtype=np.int32), drops.start.reshape(-1).astype(np.int32),
                             drops.length.reshape(-1).astype(np.int32), val_ptr, np.zeros(0, dtype=np.complex128),
                             np.zeros(0), np.asarray(drops.reg, dtype=np.float64), np.zeros(0, np.int32),
                             np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32),
                             np.zeros(0, np.int32), np.zeros(0, np.int32), True,
                             np.asarray(drops.snr_linear, dtype=np.float64))
            up = lambda a, dt=None: torch.from_numpy(np.ascontiguousarray(a if dt is None else a.astype(dt))).to(dev)  # noqa: E731
            t = {"row_seg_ptr": up(host.row_seg_ptr), "seg_start": up(host.seg_start), "seg_len": up(host.seg_len),
                 "row_val_ptr": up(val_ptr), "reg": up(host.reg), "snr_linear": up(host.snr_linear)}
            wl, r0, th = up(drops.wavelength, np.float64), up(drops.r0, np.float64), up(drops.theta, np.float64)
            kd = _lib.KzDrop()
            kd.n_systems, kd.n_users, kd.n_antennas = b, k, nt
            kd.dtype = _lib.KZ_C128 if dtype == "c128" else _lib.KZ_C64
            kd.element_spacing = float(drops.element_spacing)
            kd.wavelength, kd.r0, kd.theta = wl.data_ptr(), r0.data_ptr(), th.data_ptr()
            kd.vr_start, kd.vr_len, kd.reg = t["seg_start"].data_ptr(), t["seg_len"].data_ptr(), t["reg"].data_ptr()
            cdt = torch.complex128 if dtype == "c128" else torch.complex64
            t["heff"] = torch.empty(int(val_ptr[-1]), dtype=cdt, device=dev)
            t["row_energy"] = torch.empty(rows, dtype=torch.float64, device=dev)
            _lib.check(lb.kz_channel_synth(C.byref(kd), t["row_val_ptr"].data_ptr(), t["heff"].data_ptr(),
                                           t["row_energy"].data_ptr(), sp))
            ccnt = torch.empty(rows, dtype=torch.int32, device=dev)
            ocnt = torch.empty(b, dtype=torch.int32, device=dev)
            t["non_union_size"] = torch.empty(b, dtype=torch.int32, device=dev)
            inset = torch.empty(rows, dtype=torch.uint8, device=dev)
            _lib.check(lb.kz_partition_counts(C.byref(kd), ccnt.data_ptr(), ocnt.data_ptr(),
                                              t["non_union_size"].data_ptr(), inset.data_ptr(), sp))
            z = torch.zeros(1, dtype=torch.int32, device=dev)
            t["coupled_ptr"] = torch.cat([z, torch.cumsum(ccnt, 0, dtype=torch.int32)])
            t["orth_ptr"] = torch.cat([z, torch.cumsum(ocnt, 0, dtype=torch.int32)])
            t["ogrp_sys"] = torch.arange(b + 1, dtype=torch.int32, device=dev)  # one orthogonal group per system
            t["ogrp_ptr"] = t["orth_ptr"]
            t["non_ptr"] = torch.cat([z, torch.cumsum(k - ocnt, 0, dtype=torch.int32)])
            n_c, n_o = int(t["coupled_ptr"][-1]), int(t["orth_ptr"][-1])  # sizes: one small device->host read
            t["coupled_idx"] = torch.empty(max(n_c, 1), dtype=torch.int32, device=dev)
            t["orth_idx"] = torch.empty(max(n_o, 1), dtype=torch.int32, device=dev)
            t["non_idx"] = torch.empty(max(rows - n_o, 1), dtype=torch.int32, device=dev)
            _lib.check(lb.kz_partition_fill(C.byref(kd), t["coupled_ptr"].data_ptr(), t["orth_ptr"].data_ptr(),
                                            t["non_ptr"].data_ptr(), t["coupled_idx"].data_ptr(),
                                            t["orth_idx"].data_ptr(), t["non_idx"].data_ptr(), sp))
        obj = cls.__new__(cls)
        obj.host, obj.dtype, obj.device, obj.t = host, dtype, dev, t
        obj._drop_keep = (wl, r0, th, ccnt, ocnt, inset)
        obj.problem = obj._make_problem(t)
        return obj

    # CSR pointer fields indexed by row (b*K + i) / by system; their VALUES are absolute offsets into the value
    # arrays, so a contiguous range of systems is the same value arrays behind offset pointer arrays
    _PER_ROW = ("row_seg_ptr", "row_val_ptr", "row_energy", "coupled_ptr")
    _PER_SYSTEM = ("reg", "orth_ptr", "non_ptr", "non_union_size", "snr_linear", "ogrp_sys")

    def view(self, lo: int, hi: int) -> "DeviceBatch":
        """Systems [lo, hi) of this batch without copying: the kz_problem's per-row / per-system arrays start at
        row lo*K / system lo, the packed values are shared (layout hints are the whole batch's upper bounds)."""
        if not 0 <= lo <= hi <= self.n_systems:
            raise ValueError(f"system range [{lo}, {hi}) outside [0, {self.n_systems})")
        k = self.n_users
        t = dict(self.t)
        for name in self._PER_ROW:
            t[name] = self.t[name][lo * k:]
        for name in self._PER_SYSTEM:
            if name in self.t:
                t[name] = self.t[name][lo:hi] if name == "snr_linear" else self.t[name][lo:]
        obj = DeviceBatch.__new__(DeviceBatch)
        obj.host = _HostView(self.host, hi - lo, getattr(self.host, "row0", 0) + lo * k)
        obj.dtype, obj.device, obj.t = self.dtype, self.device, t
        obj.parent = self
        obj.problem = obj._make_problem(t)
        return obj

    @property
    def n_systems(self):
        return self.host.n_systems

    @property
    def n_users(self):
        return self.host.n_users

    @property
    def n_antennas(self):
        return self.host.n_antennas

    @property
    def complex_dtype(self):
        import torch
        return torch.complex128 if self.dtype == "c128" else torch.complex64
