"""Builders shared by the tests (inputs for the oracle and for the GPU path)."""

import os

import numpy as np

import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def oracle_channel_from_mask(h, vr_mask, n_subarrays, carrier_freq=100e9):
    """Rebuild an oracle ChannelMatrix from a stored (h, per-user subarray mask)."""
    nt, k = h.shape
    cfg = O.ArrayConfig(nt, carrier_freq, int(n_subarrays))
    vrs = tuple(O.VisibilityRegion(frozenset(np.flatnonzero(vr_mask[i]).tolist()), int(n_subarrays),
                                   nt // int(n_subarrays)) for i in range(k))
    return O.ChannelMatrix(h=np.asarray(h), vrs=vrs, cfg=cfg)


def oracle_channel_contiguous(ch, b):
    """Oracle ChannelMatrix of system b of a ContiguousChannels batch (1-antenna subarray grid)."""
    nt, k = ch.n_antennas, ch.n_users
    cfg = O.ArrayConfig(nt, 30e9, nt)
    vrs = tuple(O.contiguous_region(int(ch.start[b, i]), int(ch.length[b, i]), nt) for i in range(k))
    return O.ChannelMatrix(h=ch.dense(b), vrs=vrs, cfg=cfg)


def contiguous_from_fixture(z):
    from paper_2501_10689_b200.channel import ContiguousChannels
    return ContiguousChannels(int(z["n_antennas"]), int(z["start"].shape[1]), z["start"], z["length"], z["heff"],
                              z["row_val_ptr"], z["reg"], z["snr_linear"])
