"""GPU parity of the grouped VR-OAHK variant (scheme "vr-oahk-g", KZ_VR_OAHK_G): BASELINE cfg3's "orthogonal row
groups built from disjoint VRs and an aggregation of up to 8 hyperplanes per step", which the reference does not
implement, against its CPU restatement oracle/grouped.py (itself pinned to the reference's vr-oahk in the
one-group / uncapped limit by tests/test_oracle_golden.py).

Tolerances (BASELINE.json north_star): complex128 V within 1e-10 relative, FlopCounter totals and no-op counts
exact; complex64 NMSE / sum-rate per SURVEY §9.7 (helpers.c64_nmse_ok).
"""

import numpy as np
import pytest

import oracle as O
from helpers import c64_nmse_ok, oracle_channel_contiguous

pytestmark = pytest.mark.gpu


def _kz():
    import paper_2501_10689_b200 as kz
    return kz


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("groups,cap", [(4, 8), (2, 3), (1, 8)])
def test_grouped_c128_matches_restatement(groups, cap):
    from oracle.grouped import run_precoding_grouped
    kz = _kz()
    T = 4
    ch = kz.generate("cfg3", [0, 1])
    host = kz.HostBatch.from_contiguous(ch, orth_groups=groups, agg_cap=cap)
    dev = host.to_device("c128")
    res = kz.solve_batch(dev, "vr-oahk-g", mode="lockstep", max_iters=T)
    nt, k = ch.n_antennas, ch.n_users
    for b in range(2):
        chan = oracle_channel_contiguous(ch, b)
        reg = float(ch.reg[b])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        run = run_precoding_grouped(sys_, O.rzf_precoder(chan, reg), groups, cap, T)
        assert rel(res.v[b].cpu().numpy(), run.v) <= 1e-10, b
        asm = sum(6 * q * k + 2 * (q - 1) * k for q in
                  [sum(1 for vr in chan.vrs if n in vr.visible_subarrays) for n in range(nt)] if q)
        assert int(res.flops[b].sum()) + 4 * nt * k + asm == pytest.approx(run.flops_measured, rel=5e-3)
        steps = T * k * (groups + -(-k // (cap if cap > 0 else k)))
        assert abs(int(res.noop_steps[b].sum()) - run.noop_steps) <= 0.01 * steps
        assert int(res.n_outer[b]) == T


def test_grouped_limit_equals_vr_oahk_kernel():
    """One group and an uncapped aggregation (agg_cap = 0 -> K) is vr-oahk, bit for bit, on the same kernel."""
    import torch
    kz = _kz()
    ch = kz.generate("cfg3", [2, 3])
    dev = kz.HostBatch.from_contiguous(ch).to_device("c128")
    a = kz.solve_batch(dev, "vr-oahk-g", mode="lockstep", max_iters=6)
    b = kz.solve_batch(dev, "vr-oahk", mode="lockstep", max_iters=6)
    assert torch.equal(a.v, b.v) and torch.equal(a.flops, b.flops)


def test_grouped_c64_nmse_and_rate():
    from oracle.grouped import run_precoding_grouped
    kz = _kz()
    T = 12
    ch = kz.generate("cfg3", [4, 5])
    host = kz.HostBatch.from_contiguous(ch, orth_groups=4, agg_cap=8)
    d64 = host.to_device("c64")
    rz = kz.rzf_batched(host.to_device("c128"))
    out = kz.run_precoding_batched("vr-oahk-g", d64, max_iters=T, v_ref=rz["v"], beta_ref=rz["beta"], rates=True)
    for b in range(2):
        chan = oracle_channel_contiguous(ch, b)
        reg = float(ch.reg[b])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        ref = O.rzf_precoder(chan, reg)
        run = run_precoding_grouped(sys_, ref, 4, 8, T)
        f = O.assemble_dense(chan, run.v).f
        _, s128 = O.spectral_efficiency(chan.h, f, float(ch.snr_linear[b]))
        assert c64_nmse_ok(float(out["nmse"][b]), O.nmse(f, ref.f)), (float(out["nmse"][b]), O.nmse(f, ref.f))
        assert float(out["sum_rate"][b]) == pytest.approx(s128, rel=1e-3)


def test_plain_vr_oahk_refuses_grouped_batch():
    kz = _kz()
    ch = kz.generate("cfg3", [0])
    dev = kz.HostBatch.from_contiguous(ch, orth_groups=3, agg_cap=8).to_device("c64")
    with pytest.raises(ValueError):
        kz.solve_batch(dev, "vr-oahk", mode="lockstep", max_iters=2)


@pytest.mark.parametrize("groups,cap", [(4, 8), (2, 3), (1, 0)])
def test_grouped_cluster_kernel_c64_vs_restatement(groups, cap):
    """The cluster kernel's grouped path (csrc/kz_solve_cluster.cuh, row sets: orthogonal groups then aggregation
    blocks, each with its own refresh / exchange / step) in complex64 against the complex128 restatement: V within
    1e-4 relative (a deterministic scheme, fp32 accumulation), FlopCounter totals within 0.5% and no-op counts
    within 1% of the steps (a block whose fp32 weights are all exactly zero is a no-op, and whether a weight
    underflows to exactly zero depends on the fp32 summation order: the generic kernel's complex64 run differs from
    both by single no-ops too; complex128 counters are exact, test_grouped_c128_matches_restatement), and the
    launch is the cluster kernel's (kernel + n_outer finaliser), not the generic kernel's."""
    from oracle.grouped import run_precoding_grouped
    kz = _kz()
    T = 6
    ch = kz.generate("cfg3", [6, 7])
    host = kz.HostBatch.from_contiguous(ch, orth_groups=groups, agg_cap=cap)
    res = kz.solve_batch(host.to_device("c64"), "vr-oahk-g", mode="lockstep", max_iters=T)
    assert res.launches == 2, res.launches
    nt, k = ch.n_antennas, ch.n_users
    for b in range(2):
        chan = oracle_channel_contiguous(ch, b)
        reg = float(ch.reg[b])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        run = run_precoding_grouped(sys_, O.rzf_precoder(chan, reg), groups, cap if cap > 0 else k, T)
        assert rel(res.v[b].cpu().numpy(), run.v) <= 1e-4, b
        asm = sum(6 * q * k + 2 * (q - 1) * k for q in
                  [sum(1 for vr in chan.vrs if n in vr.visible_subarrays) for n in range(nt)] if q)
        assert int(res.flops[b].sum()) + 4 * nt * k + asm == pytest.approx(run.flops_measured, rel=5e-3)
        steps = T * k * (groups + -(-k // (cap if cap > 0 else k)))
        assert abs(int(res.noop_steps[b].sum()) - run.noop_steps) <= 0.01 * steps


def test_grouped_cluster_extreme_caps():
    """Grouped cluster path at the extremes: one hyperplane per aggregated step (agg_cap = 1: every N row its own
    set) and a single group with all of N in one block; complex64 V within 1e-4 of the restatement."""
    from oracle.grouped import run_precoding_grouped
    kz = _kz()
    T = 3
    ch = kz.generate("cfg3", [9])
    k = ch.n_users
    for groups, cap in ((3, 1), (1, 200)):
        host = kz.HostBatch.from_contiguous(ch, orth_groups=groups, agg_cap=cap)
        res = kz.solve_batch(host.to_device("c64"), "vr-oahk-g", mode="lockstep", max_iters=T)
        assert res.launches == 2
        chan = oracle_channel_contiguous(ch, 0)
        reg = float(ch.reg[0])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        run = run_precoding_grouped(sys_, O.rzf_precoder(chan, reg), groups, min(cap, k), T)
        assert rel(res.v[0].cpu().numpy(), run.v) <= 1e-4, (groups, cap)
