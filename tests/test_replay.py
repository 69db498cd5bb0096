"""Channel replay formats: the reference's text format read and written
byte-compatibly (fixture written by the reference's own save_channel, tests/golden/make_replay_fixture.py),
and the exact binary batch round trip."""

import os

import numpy as np

import paper_2501_10689_b200 as kz
from paper_2501_10689_b200 import replay

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_reads_reference_text_channel():
    chan, meta = replay.load_channel(os.path.join(GOLDEN, "channel_ref.txt"))
    z = np.load(os.path.join(GOLDEN, "channel_ref.npz"))
    np.testing.assert_array_equal(chan.h, z["h"])  # repr() doubles: bit-faithful
    assert meta == {"seed": 3, "p_visible": 0.6}
    for i, vr in enumerate(chan.vrs):
        assert vr.visible_subarrays == frozenset(np.flatnonzero(z["vr"][i]).tolist())
    # the reference-format channel feeds the solver API directly
    sys_ = kz.AugmentedSystem.from_channel(chan, float(z["reg"]))
    assert sys_.n_users == 4 and sys_.n_antennas == 32


def test_writes_reference_text_channel_byte_identical(tmp_path):
    chan, meta = replay.load_channel(os.path.join(GOLDEN, "channel_ref.txt"))
    out = tmp_path / "c.txt"
    replay.save_channel(out, chan.h, chan.vrs, chan.n_subarrays, chan.carrier_freq, seed=meta["seed"],
                        p_visible=meta["p_visible"])
    assert out.read_bytes() == open(os.path.join(GOLDEN, "channel_ref.txt"), "rb").read()


def test_binary_batch_round_trip(tmp_path):
    host = kz.HostBatch.from_contiguous(kz.generate("cfg1", range(5)))
    p = tmp_path / "b.npz"
    replay.save_batch(p, host)
    back = replay.load_batch(p)
    for name in ("row_seg_ptr", "seg_start", "seg_len", "row_val_ptr", "heff", "row_energy", "reg", "coupled_ptr",
                 "coupled_idx", "orth_ptr", "orth_idx", "non_ptr", "non_idx", "non_union_size", "snr_linear"):
        np.testing.assert_array_equal(getattr(back, name), getattr(host, name), err_msg=name)
    assert (back.n_systems, back.n_users, back.n_antennas, back.contiguous) == (5, 16, 256, True)
    # binary is far smaller than one text line per dense entry
    assert os.path.getsize(p) < 0.2 * 40 * host.n_systems * host.n_users * host.n_antennas
