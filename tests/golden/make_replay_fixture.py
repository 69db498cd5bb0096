"""Writes tests/golden/channel_ref.txt with the REFERENCE's save_channel (run here, where
/root/reference is importable) plus the same channel as arrays in channel_ref.npz."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from kaczprec import ArrayConfig, power_control, random_channel, save_channel  # noqa: E402

here = os.path.dirname(os.path.abspath(__file__))
cfg = ArrayConfig(n_antennas=32, carrier_freq=100e9, n_subarrays=4)
chan, reg = power_control(random_channel(cfg, 4, 5, 0.6, np.random.default_rng(3)), 10.0)
save_channel(os.path.join(here, "channel_ref.txt"), chan, seed=3, p_visible=0.6)
np.savez(os.path.join(here, "channel_ref.npz"), h=chan.h, reg=reg,
         vr=np.array([[s in vr.visible_subarrays for s in range(4)] for vr in chan.vrs]))
print("wrote channel_ref.txt / .npz")
