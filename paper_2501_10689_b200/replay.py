"""Channel replay formats.

* The reference's text format (pkg/src/kaczprec/channel.py:316-392): a magic line, a header
  ``nt= k= s= f= seed= p=``, one ``vr k: subarrays`` line per user, then ``re im`` per entry
  (row-major over antennas x users) with repr() doubles — bit-faithful but one line per complex
  entry, zeros included.  `save_channel` / `load_channel` read and write it byte-compatibly so
  channels saved by the reference can be replayed here (and vice versa).
* A binary batch format for many realizations: the packed kz_problem layout (only the VR entries,
  no zeros) in one uncompressed ``.npz`` — `save_batch` / `load_batch`, exact round trip of a
  HostBatch.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TEXT_MAGIC = "kaczprec-channel 1"
BATCH_MAGIC = "kz-b200-batch 1"


@dataclass(frozen=True)
class SubarrayRegion:
    """Visibility region as a set of visible subarrays of equal size (channel.py:59-91)."""

    visible_subarrays: frozenset
    n_subarrays: int
    subarray_size: int

    @property
    def antenna_indices(self) -> np.ndarray:
        m = self.subarray_size
        return np.asarray([s * m + j for s in sorted(self.visible_subarrays) for j in range(m)], dtype=np.int64)


@dataclass(frozen=True)
class Channel:
    """Channel matrix + visibility regions, the fields AugmentedSystem.from_channel reads."""

    h: np.ndarray
    vrs: tuple
    n_subarrays: int
    carrier_freq: float

    @property
    def n_users(self) -> int:
        return self.h.shape[1]

    @property
    def n_antennas(self) -> int:
        return self.h.shape[0]


def save_channel(path, h, vrs, n_subarrays: int, carrier_freq: float, seed=None, p_visible=None) -> None:
    """Write one realization in the reference's text format (channel.py:324-346)."""
    h = np.asarray(h)
    nt, k = h.shape
    lines = [TEXT_MAGIC,
             "nt=%d k=%d s=%d f=%s seed=%s p=%s" % (nt, k, n_subarrays, repr(float(carrier_freq)),
                                                   "none" if seed is None else int(seed),
                                                   "none" if p_visible is None else repr(float(p_visible)))]
    for i, vr in enumerate(vrs):
        subs = vr.visible_subarrays if hasattr(vr, "visible_subarrays") else vr
        lines.append(f"vr {i}: " + " ".join(str(s) for s in sorted(subs)))
    for n in range(nt):
        for i in range(k):
            z = complex(h[n, i])
            lines.append(f"{z.real!r} {z.imag!r}")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def load_channel(path):
    """Read a text channel (channel.py:349-392): returns (Channel, meta)."""
    with open(path) as fh:
        lines = [ln.rstrip("\n") for ln in fh]
    if not lines or lines[0] != TEXT_MAGIC:
        raise ValueError(f"{path}: not a channel file (bad magic)")
    header = dict(item.split("=", 1) for item in lines[1].split())
    nt, k, s = int(header["nt"]), int(header["k"]), int(header["s"])
    freq = float(header["f"])
    if nt % s != 0:
        raise ValueError(f"{path}: {nt} antennas do not split into {s} subarrays")
    vrs = []
    for i in range(k):
        tag, subs = lines[2 + i].split(":")
        if tag.strip() != f"vr {i}":
            raise ValueError(f"{path}: malformed visibility line {i}")
        vrs.append(SubarrayRegion(frozenset(int(x) for x in subs.split()), s, nt // s))
    body = lines[2 + k:]
    if len(body) != nt * k:
        raise ValueError(f"{path}: expected {nt * k} entries, found {len(body)}")
    vals = np.array([[float(x) for x in ln.split()] for ln in body], dtype=np.float64)
    h = np.empty(nt * k, dtype=np.complex128)
    h.real, h.imag = vals[:, 0], vals[:, 1]  # keeps signed zeros (bit-faithful round trip)
    h = h.reshape(nt, k)
    meta = {"seed": None if header["seed"] == "none" else int(header["seed"]),
            "p_visible": None if header["p"] == "none" else float(header["p"])}
    return Channel(h=h, vrs=tuple(vrs), n_subarrays=s, carrier_freq=freq), meta


_FIELDS = ("row_seg_ptr", "seg_start", "seg_len", "row_val_ptr", "heff", "row_energy", "reg", "coupled_ptr",
           "coupled_idx", "orth_ptr", "orth_idx", "non_ptr", "non_idx", "non_union_size")


def save_batch(path, host) -> None:
    """Packed binary batch (exact): the kz_problem arrays of a HostBatch in one .npz."""
    arrays = {name: np.asarray(getattr(host, name)) for name in _FIELDS}
    if host.snr_linear is not None:
        arrays["snr_linear"] = np.asarray(host.snr_linear)
    np.savez(path, magic=np.asarray(BATCH_MAGIC),
             shape=np.asarray([host.n_systems, host.n_users, host.n_antennas, int(host.contiguous)], dtype=np.int64),
             **arrays)


def load_batch(path):
    """Inverse of save_batch: a HostBatch."""
    from .batch import HostBatch
    with np.load(path, allow_pickle=False) as z:
        if str(z["magic"]) != BATCH_MAGIC:
            raise ValueError(f"{path}: not a kz-b200 batch file")
        b, k, nt, contiguous = (int(x) for x in z["shape"])
        f = {name: z[name] for name in _FIELDS}
        snr = z["snr_linear"] if "snr_linear" in z.files else None
    return HostBatch(b, k, nt, f["row_seg_ptr"], f["seg_start"], f["seg_len"], f["row_val_ptr"], f["heff"],
                     f["row_energy"], f["reg"], f["coupled_ptr"], f["coupled_idx"], f["orth_ptr"], f["orth_idx"],
                     f["non_ptr"], f["non_idx"], f["non_union_size"], bool(contiguous), snr)
