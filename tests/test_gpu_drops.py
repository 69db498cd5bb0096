"""On-device input preparation: DeviceBatch.from_drops (kz_channel_synth +
kz_partition_counts/fill) against the host path HostBatch.from_contiguous(generate(...)) on the same
drops: packed rows within fp64 rounding (complex128), energies, the VR partition exactly, and identical
solver output."""

import numpy as np
import pytest

from helpers import c64_nmse_ok
import torch

pytestmark = pytest.mark.gpu


def _kz():
    import paper_2501_10689_b200 as kz
    return kz


def _both(cfg, seeds, dtype):
    kz = _kz()
    host = kz.HostBatch.from_contiguous(kz.generate(cfg, seeds))
    ref = host.to_device(dtype)
    dev = kz.DeviceBatch.from_drops(kz.generate_drops(cfg, seeds), dtype)
    return host, ref, dev


@pytest.mark.parametrize("cfg,seeds", [("cfg2", range(6)), ("cfg3", range(3)), ("cfg4", [0]),
                                        ("cfg5", [0, [0, 511, 1023]])])
def test_device_batch_equals_host_batch(cfg, seeds):
    host, ref, dev = _both(cfg, seeds, "c128")
    for name in ("row_seg_ptr", "seg_start", "seg_len", "row_val_ptr", "coupled_ptr", "coupled_idx", "orth_ptr",
                 "orth_idx", "non_ptr", "non_idx", "non_union_size"):
        np.testing.assert_array_equal(dev.t[name].cpu().numpy()[:len(getattr(host, name))], getattr(host, name),
                                      err_msg=name)
    h_dev, h_ref = dev.t["heff"].cpu().numpy(), ref.t["heff"].cpu().numpy()
    # phases 2 pi r / lambda reach ~3e4 rad: one ulp of r moves an entry by ~1e-12 relative
    assert np.max(np.abs(h_dev - h_ref)) <= 1e-10 * np.max(np.abs(h_ref))
    np.testing.assert_allclose(dev.t["row_energy"].cpu().numpy(), host.row_energy, rtol=1e-12)
    assert dev.problem.max_support == ref.problem.max_support
    assert dev.problem.slice_pairs_256 == ref.problem.slice_pairs_256


def test_device_batch_solves_like_host_batch():
    kz = _kz()
    _, ref, dev = _both("cfg2", range(8), "c128")
    for sc in ("vr-oahk", "grk"):
        rng = ("philox", 4) if sc == "grk" else None
        a = kz.solve_batch(ref, sc, mode="lockstep", max_iters=40, rng=rng).v.cpu().numpy()
        b = kz.solve_batch(dev, sc, mode="lockstep", max_iters=40, rng=rng).v.cpu().numpy()
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(a), sc
    # complex64 path: same rows to fp32 rounding, same precoders to the c64 criterion
    _, ref64, dev64 = _both("cfg3", range(2), "c64")
    np.testing.assert_allclose(dev64.t["heff"].cpu().numpy(), ref64.t["heff"].cpu().numpy(), rtol=0, atol=1e-7)
    rz = kz.rzf_batched(ref64)
    o1 = kz.run_precoding_batched("vr-oahk", ref64, max_iters=20, v_ref=rz["v"], beta_ref=rz["beta"])
    o2 = kz.run_precoding_batched("vr-oahk", dev64, max_iters=20, v_ref=rz["v"], beta_ref=rz["beta"])
    a, b = o2["nmse"].cpu().numpy(), o1["nmse"].cpu().numpy()
    assert np.all(c64_nmse_ok(a, b)), (a, b)
    torch.cuda.synchronize()
