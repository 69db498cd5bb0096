"""GPU parity: libkaczmarz_b200.so against the CPU oracle and the committed
reference fixtures.

Tolerances (BASELINE.json north_star):
  complex128 oracle mode  - selected row sequences identical; iterates within
                            1e-10 relative (Frobenius) of the reference.
  complex64 throughput    - final NMSE against RZF and sum-rate within 1e-3
                            relative, NMSE compared only above the fp32 floor
                            (NMSE_128 >= 1e-5; below it NMSE_64 <= 1e-6), per
                            SURVEY.md §9.7, with the same host streams.
"""

import numpy as np
import pytest

import oracle as O
from helpers import c64_nmse_ok, contiguous_from_fixture, load, oracle_channel_contiguous, oracle_channel_from_mask

pytestmark = pytest.mark.gpu

REL_C128 = 1e-10
REL_C64 = 1e-3


def _kz():
    import paper_2501_10689_b200 as kz
    return kz


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (n if n > 0 else 1.0)


def run_rows(sys_list, scheme, T, rngs, dtype="c128", epsilon=0.0, f_ref=None, spawn=True):
    """Lockstep run of a list of systems; returns (BatchResult, DeviceBatch)."""
    kz = _kz()
    host = kz.HostBatch.from_systems(sys_list)
    dev = host.to_device(dtype)
    k = host.n_users
    streams = None
    if scheme in kz.STOCHASTIC_SCHEMES:
        gens = [r.spawn(k) if spawn else r for r in rngs]
        streams = kz.HostStreams(scheme, gens, host.row_energy.reshape(host.n_systems, k))
    res = kz.solve_batch(dev, scheme, mode="lockstep", max_iters=T, epsilon=epsilon, f_ref=f_ref,
                         rng=streams, rows_cap=T)
    return res, dev


def assert_rows(res_rows, want_rows, b):
    got = res_rows[b].cpu().numpy()
    for c in range(got.shape[0]):
        g = got[c][got[c] >= 0]
        w = np.asarray(want_rows[c])
        w = w[w >= 0]
        np.testing.assert_array_equal(g, w, err_msg=f"rhs {c}")


# --------------------------------------------------------------------------- c128 parity

@pytest.mark.parametrize("scheme", O.SCHEMES)
def test_lockstep_nmse_stop_matches_reference(scheme):
    """run_precoding(eps=1e-6, rng=42) on the reference test drop: iteration count, V,
    flops, noop steps, traces and row sequences (tests/test_solvers.py:505-523)."""
    kz = _kz()
    z = load("ref_lockstep.npz")
    chan = oracle_channel_from_mask(z["h"], z["vr_mask"], z["n_subarrays"])
    reg = float(z["reg"])
    sys_ = O.AugmentedSystem.from_channel(chan, reg)
    ref = O.rzf_precoder(chan, reg)
    run = kz.run_precoding(scheme, sys_, ref, epsilon=1e-6, rng=np.random.default_rng(42))
    assert run.n_iters == int(z[f"{scheme}/n_iters"])
    assert run.converged
    assert rel(run.v, z[f"{scheme}/v"]) <= REL_C128
    assert run.flops_measured == int(z[f"{scheme}/flops_measured"])
    assert run.noop_steps == int(z[f"{scheme}/noop_steps"])
    np.testing.assert_array_equal(run.flops_trace, z[f"{scheme}/flops_trace"])
    np.testing.assert_allclose(run.nmse_trace, z[f"{scheme}/nmse_trace"], rtol=1e-7, atol=1e-14)
    np.testing.assert_allclose(run.resid_trace, z[f"{scheme}/resid_trace"], rtol=1e-7, atol=1e-13)
    assert rel(run.precoder.f, z[f"{scheme}/f"]) <= REL_C128
    res, _ = run_rows([sys_], scheme, int(z[f"{scheme}/n_iters"]), [np.random.default_rng(42)])
    assert_rows(res.rows, z[f"{scheme}/rows"], 0)


def test_fixed_t_batch_matches_reference():
    """Four conftest-scale drops batched in one launch per scheme, T = 15."""
    kz = _kz()
    z = load("ref_fixed_t.npz")
    systems, chans = [], []
    for seed in range(4):
        chan = oracle_channel_from_mask(z[f"{seed}/h"], z[f"{seed}/vr_mask"], 4)
        chans.append(chan)
        systems.append(O.AugmentedSystem.from_channel(chan, float(z[f"{seed}/reg"])))
    for sc in O.SCHEMES:
        rngs = [np.random.default_rng(100 + s) for s in range(4)]
        res, dev = run_rows(systems, sc, 15, rngs)
        ep = kz.epilogue(dev, res.v, want_f=True, rates=True,
                         snr_linear=np.array([1.0 / float(z[f"{s}/reg"]) for s in range(4)]))
        for s in range(4):
            assert rel(res.v[s].cpu().numpy(), z[f"{s}/{sc}/v"]) <= REL_C128, (sc, s)
            assert_rows(res.rows, z[f"{s}/{sc}/rows"], s)
            assert rel(ep["f"][s].cpu().numpy(), z[f"{s}/{sc}/f"]) <= REL_C128
            assert float(ep["sum_rate"][s]) == pytest.approx(float(z[f"{s}/{sc}/sum_rate"]), rel=1e-10)


@pytest.mark.parametrize("mode,eps", [("residual", 1e-8), ("oracle", 1e-6)])
def test_solve_all_modes_match_reference(mode, eps):
    kz = _kz()
    z = load("ref_solve.npz")
    chan = oracle_channel_from_mask(z["h"], z["vr_mask"], 8)
    sys_ = O.AugmentedSystem.from_channel(chan, float(z["reg"]))
    vref = z["v_ref"]
    for sc in O.SCHEMES:
        key = f"{mode}/{sc}"
        stop = kz.StoppingRule(mode=mode, epsilon=eps, reference=vref if mode == "oracle" else None,
                               check_every=2)
        v = kz.solve_all(sc, sys_, stop, rng=np.random.default_rng(7))
        assert rel(v, z[f"{key}/v"]) <= REL_C128, sc
        host = kz.HostBatch.from_systems([sys_])
        dev = host.to_device("c128")
        streams = None
        if sc in kz.STOCHASTIC_SCHEMES:
            streams = kz.HostStreams(sc, [np.random.default_rng(7).spawn(8)], host.row_energy.reshape(1, 8))
        res = kz.solve_batch(dev, sc, mode=mode, max_iters=80_000, epsilon=eps, check_every=2,
                             v_ref=vref[None] if mode == "oracle" else None, rng=streams, rows_cap=4096,
                             trace_cap=4096, chunk=64)
        np.testing.assert_array_equal(res.iters[0].cpu().numpy(), z[f"{key}/iters"])
        np.testing.assert_array_equal(res.converged[0].cpu().numpy().astype(bool), z[f"{key}/converged"])
        np.testing.assert_array_equal(res.n_checks[0].cpu().numpy(), z[f"{key}/n_checks"])
        assert_rows(res.rows, z[f"{key}/rows"], 0)


def test_single_rhs_solve_frozen_counts():
    """tests/test_solvers.py:435-446 through the GPU `solve`: gk 32, urk 93."""
    kz = _kz()
    cfg = O.ArrayConfig(64, 100e9, 8)
    chan, reg = O.power_control(O.random_channel(cfg, 8, 5, 0.5, np.random.default_rng(0)), 0.0)
    sys_ = O.AugmentedSystem.from_channel(chan, reg)
    vref = O.auxiliary_matrix(chan, reg)
    st, tr = kz.solve("gk", sys_, 0, kz.StoppingRule(epsilon=1e-6, reference=vref[:, 0]))
    assert tr.n_iters == 32 and tr.converged
    st, tr = kz.solve("urk", sys_, 0, kz.StoppingRule(epsilon=1e-6, reference=vref[:, 0]),
                      rng=np.random.default_rng(7))
    assert tr.n_iters == 93
    ost, otr = O.solve("urk", sys_, 0, O.StoppingRule(epsilon=1e-6, reference=vref[:, 0]),
                       rng=np.random.default_rng(7))
    assert rel(st.coef, ost.coef) <= REL_C128
    assert rel(st.col, ost.col) <= REL_C128
    assert st.counter.total == ost.counter.total
    np.testing.assert_allclose(tr.resid, otr.resid, rtol=1e-7, atol=1e-14)


@pytest.mark.parametrize("name", ["ref_cfg1.npz", "ref_cfg2.npz"])
def test_config_parity_c128(name):
    """BASELINE cfg1 (GRK, T=50) and cfg2 (5 schemes, T=200) shapes in complex128."""
    kz = _kz()
    z = load(name)
    ch = contiguous_from_fixture(z)
    T = int(z["n_iters"])
    host = kz.HostBatch.from_contiguous(ch)
    dev = host.to_device("c128")
    b, k = host.n_systems, host.n_users
    schemes = sorted({key.split("/")[1] for key in z.files if key.count("/") == 2})
    for b_i in range(b):
        assert np.array_equal(host.orth_idx[host.orth_ptr[b_i]:host.orth_ptr[b_i + 1]], z[f"{b_i}/orthogonal"])
    v_ref = np.stack([z[f"{i}/v_ref"] for i in range(b)])
    beta_ref = np.array([float(z[f"{i}/beta_ref"]) for i in range(b)])
    rz = kz.rzf_batched(dev)
    assert rel(rz["v"].cpu().numpy(), v_ref) <= REL_C128
    np.testing.assert_allclose(rz["beta"].cpu().numpy(), beta_ref, rtol=1e-12)
    for sc in schemes:
        streams = None
        if sc in kz.STOCHASTIC_SCHEMES:
            gens = [np.random.default_rng(kz.solver_seed_sequence(int(s))).spawn(k) for s in z["seeds"]]
            streams = kz.HostStreams(sc, gens, host.row_energy.reshape(b, k))
        res = kz.solve_batch(dev, sc, mode="lockstep", max_iters=T, rng=streams, rows_cap=T)
        ep = kz.epilogue(dev, res.v, v_ref=v_ref, beta_ref=beta_ref, rates=True)
        for b_i in range(b):
            assert rel(res.v[b_i].cpu().numpy(), z[f"{b_i}/{sc}/v"]) <= REL_C128, (sc, b_i)
            assert_rows(res.rows, z[f"{b_i}/{sc}/rows"], b_i)
            assert float(ep["nmse"][b_i]) == pytest.approx(float(z[f"{b_i}/{sc}/nmse"]), rel=1e-6, abs=1e-13)
            assert float(ep["sum_rate"][b_i]) == pytest.approx(float(z[f"{b_i}/{sc}/sum_rate"]), rel=1e-10)


# --------------------------------------------------------------------------- c64 throughput mode

def _c64_ok(n64, n128, s64, s128):
    assert s64 == pytest.approx(s128, rel=REL_C64)
    assert c64_nmse_ok(n64, n128), (n64, n128)


@pytest.mark.parametrize("name", ["ref_cfg1.npz", "ref_cfg2.npz"])
def test_config_parity_c64(name):
    kz = _kz()
    z = load(name)
    ch = contiguous_from_fixture(z)
    T = int(z["n_iters"])
    host = kz.HostBatch.from_contiguous(ch)
    dev = host.to_device("c64")
    b, k = host.n_systems, host.n_users
    v_ref = np.stack([z[f"{i}/v_ref"] for i in range(b)])
    beta_ref = np.array([float(z[f"{i}/beta_ref"]) for i in range(b)])
    schemes = sorted({key.split("/")[1] for key in z.files if key.count("/") == 2})
    for sc in schemes:
        streams = None
        if sc in kz.STOCHASTIC_SCHEMES:
            gens = [np.random.default_rng(kz.solver_seed_sequence(int(s))).spawn(k) for s in z["seeds"]]
            streams = kz.HostStreams(sc, gens, host.row_energy.reshape(b, k))
        out = kz.run_precoding_batched(sc, dev, max_iters=T, rng=streams, v_ref=v_ref, beta_ref=beta_ref)
        for b_i in range(b):
            _c64_ok(float(out["nmse"][b_i]), float(z[f"{b_i}/{sc}/nmse"]),
                    float(out["sum_rate"][b_i]), float(z[f"{b_i}/{sc}/sum_rate"]))


# --------------------------------------------------------------------------- RZF / epilogue

def test_rzf_frozen_entries_gpu():
    kz = _kz()
    rng = np.random.default_rng(1234)
    h = (rng.standard_normal((8, 3)) + 1j * rng.standard_normal((8, 3))) / np.sqrt(2)
    v = kz.auxiliary_matrix(h, 0.4)
    assert v[0, 0] == pytest.approx(0.08743823337750342 + 0j, abs=1e-10)
    assert v[1, 2] == pytest.approx(-0.00047276679288917284 - 0.0117275702144454j, abs=1e-10)
    prec = kz.rzf_precoder(h, 0.4)
    assert prec.norm_factor == pytest.approx(1.8189422748831143, rel=1e-10)
    assert prec.f[0, 0] == pytest.approx(-0.16744310691337447 + 0.09294283936181302j, abs=1e-10)
    assert np.linalg.norm(prec.f) == pytest.approx(1.0, abs=1e-12)
    np.testing.assert_allclose(v, O.auxiliary_matrix(h, 0.4), rtol=0, atol=1e-13)


def test_rzf_not_pd_raises():
    kz = _kz()
    with pytest.raises(Exception):
        kz.rzf_precoder(np.zeros((6, 2), dtype=complex), 0.0)


def test_rzf_on_vr_drops_matches_oracle():
    kz = _kz()
    for seed in range(5):
        chan, reg = O.power_control(O.random_channel(O.ArrayConfig(32, 100e9, 4), 4, 3, 0.6,
                                                     np.random.default_rng(seed)), 0.0)
        p = kz.rzf_precoder(chan, reg)
        q = O.rzf_precoder(chan, reg)
        assert rel(p.f, q.f) <= 1e-12
        assert p.norm_factor == pytest.approx(q.norm_factor, rel=1e-12)


def test_assembly_and_metrics_match_oracle():
    kz = _kz()
    z = load("ref_lockstep.npz")
    chan = oracle_channel_from_mask(z["h"], z["vr_mask"], z["n_subarrays"])
    v = z["gk/v"]
    a = kz.assemble_vr(chan, v, scheme="GK")
    b = O.assemble_vr(chan, v)
    c = kz.assemble_dense(chan, v)
    assert rel(a.f, b.f) <= 1e-13 and rel(c.f, b.f) <= 1e-13
    assert a.norm_factor == pytest.approx(b.norm_factor, rel=1e-13)
    assert kz.nmse(a.f, z["f_ref"]) == pytest.approx(O.nmse(b.f, z["f_ref"]), rel=1e-9)
    r1, s1 = kz.spectral_efficiency(chan.h, a.f, 1.0)
    r2, s2 = O.spectral_efficiency(chan.h, b.f, 1.0)
    np.testing.assert_allclose(r1, r2, rtol=1e-12)
    # the reference's calling form: assemble_vr(SubarrayChannel.from_channel(chan), v, counter)
    ca, cb = kz.FlopCounter(), O.FlopCounter()
    d = kz.assemble_vr(kz.SubarrayChannel.from_channel(chan), v, counter=ca)
    e = O.assemble_vr(chan, v, counter=cb)
    assert rel(d.f, e.f) <= 1e-13 and ca.total == cb.total


# --------------------------------------------------------------------------- edge cases

def test_single_user_one_iteration_all_schemes():
    """tests/test_solvers.py:396-406: K = 1 converges in one iteration for every scheme."""
    kz = _kz()
    cfg = O.ArrayConfig(8, 1e9, 2)
    chan, reg = O.power_control(O.random_channel(cfg, 1, 2, 1.0, np.random.default_rng(0)), 0.0)
    sys_ = O.AugmentedSystem.from_channel(chan, reg)
    expect = 1.0 / (np.linalg.norm(chan.h[:, 0]) ** 2 + reg)
    for sc in O.SCHEMES:
        st, tr = kz.solve(sc, sys_, 0, kz.StoppingRule(epsilon=1e-9, reference=np.array([expect])),
                          rng=np.random.default_rng(5))
        assert tr.n_iters == 1, sc
        assert st.coef[0] == pytest.approx(expect, rel=1e-12)


def test_disjoint_vrs_vr_oahk_one_iteration():
    """tests/test_solvers.py:449-469: all users orthogonal -> the block step solves outright (N empty)."""
    kz = _kz()
    nt, k = 16, 4
    rng = np.random.default_rng(4)
    h = np.zeros((nt, k), dtype=complex)
    for i in range(k):
        h[4 * i:4 * i + 4, i] = rng.standard_normal(4) + 1j * rng.standard_normal(4)
    h /= np.linalg.norm(h, axis=0)
    cfg = O.ArrayConfig(nt, 1e9, 4)
    vrs = tuple(O.VisibilityRegion(frozenset({i}), 4, 4) for i in range(k))
    chan = O.ChannelMatrix(h=h, vrs=vrs, cfg=cfg)
    sys_ = O.AugmentedSystem.from_channel(chan, 1.0)
    vref = O.auxiliary_matrix(chan, 1.0)
    _, tr = kz.solve("vr-oahk", sys_, 0, kz.StoppingRule(epsilon=1e-9, reference=vref[:, 0]))
    assert tr.n_iters == 1
    run = kz.run_precoding("vr-oahk", sys_, O.rzf_precoder(chan, 1.0), epsilon=1e-9)
    assert run.n_iters == 1 and run.converged


def test_ragged_vr_lengths_cfg3_shape():
    """cfg3-style ragged VR lengths (U[128,512]) at reduced B: VR-OAHK c128 vs oracle."""
    kz = _kz()
    ch = kz.generate("cfg3", [0, 1])
    host = kz.HostBatch.from_contiguous(ch)
    dev = host.to_device("c128")
    res = kz.solve_batch(dev, "vr-oahk", mode="lockstep", max_iters=20)
    for b in range(2):
        chan = oracle_channel_contiguous(ch, b)
        sys_ = O.AugmentedSystem.from_channel(chan, float(ch.reg[b]))
        run = O.run_precoding("vr-oahk", sys_, O.rzf_precoder(chan, float(ch.reg[b])), epsilon=0.0,
                              max_iters=20, traces=False)
        assert rel(res.v[b].cpu().numpy(), run.v) <= REL_C128
        assert int(res.noop_steps[b].sum()) == run.noop_steps


def test_rhs_mask_leaves_other_columns_untouched():
    kz = _kz()
    z = load("ref_lockstep.npz")
    chan = oracle_channel_from_mask(z["h"], z["vr_mask"], z["n_subarrays"])
    sys_ = O.AugmentedSystem.from_channel(chan, float(z["reg"]))
    dev = kz.HostBatch.from_systems([sys_]).to_device("c128")
    mask = np.zeros(8, dtype=np.uint8)
    mask[3] = 1
    res = kz.solve_batch(dev, "gk", mode="residual", max_iters=1000, epsilon=1e-8, rhs_mask=mask)
    v = res.v[0].cpu().numpy()
    assert np.all(v[:, [0, 1, 2, 4, 5, 6, 7]] == 0)
    assert int(res.iters[0, 3]) > 0 and bool(res.converged[0, 3])


def test_invalid_arguments_raise():
    kz = _kz()
    z = load("ref_lockstep.npz")
    chan = oracle_channel_from_mask(z["h"], z["vr_mask"], z["n_subarrays"])
    sys_ = O.AugmentedSystem.from_channel(chan, float(z["reg"]))
    ref = O.rzf_precoder(chan, float(z["reg"]))
    with pytest.raises(ValueError):
        kz.run_precoding("bogus", sys_, ref)
    with pytest.raises(ValueError):
        kz.run_precoding("grk", sys_, ref, rng=None)
    with pytest.raises(ValueError):
        kz.solve("gk", sys_, 0, kz.StoppingRule(mode="oracle", reference=None))
    dev = kz.HostBatch.from_systems([sys_]).to_device("c128")
    from paper_2501_10689_b200._lib import KzError
    with pytest.raises(KzError):
        kz.solve_batch(dev, "gk", mode="residual", max_iters=10, epsilon=0.0)


# --------------------------------------------------------------------------- throughput-mode properties

@pytest.mark.parametrize("scheme", ["urk", "grk", "vr-ogrk", "ahk", "vr-oahk", "gk", "swor-erk"])
def test_philox_full_cfg2_properties(scheme):
    """Full cfg2 shape (Nt=512, K=64) at B=148 in c64 with on-device draws:
    col = H coef invariant, power-normalised F, finite rates, error contraction."""
    import torch
    kz = _kz()
    ch = kz.generate("cfg2", range(148))
    host = kz.HostBatch.from_contiguous(ch)
    dev = host.to_device("c64")
    rz = kz.rzf_batched(dev)
    errs = []
    for T in (25, 200):
        res = kz.solve_batch(dev, scheme, mode="lockstep", max_iters=T, rng=("philox", 1234), want_iterates=True)
        ep = kz.epilogue(dev, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True, want_f=True)
        errs.append(ep["nmse"].cpu().numpy())
        assert torch.isfinite(ep["sum_rate"]).all()
        fn = torch.linalg.norm(ep["f"].reshape(dev.n_systems, -1), dim=1)
        np.testing.assert_allclose(fn.cpu().numpy(), 1.0, rtol=1e-5)
        # col = H coef: the workspace iterate equals H v
        m = res.iterates()[:4].to(torch.complex128)
        hv = kz.epilogue(dev, res.v, want_f=True)  # beta H V for every system
        hv_f = hv["f"][:4].to(torch.complex128) / hv["beta"][:4, None, None]
        assert rel(m.transpose(1, 2).cpu().numpy(), hv_f.cpu().numpy()) <= 1e-4
    # contraction, or both already at the fp32 floor (c64 NMSE floors near 5e-8)
    assert np.median(errs[1]) < np.median(errs[0]) or np.median(errs[1]) < 1e-6


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("scheme", O.SCHEMES)
def test_register_resident_path_all_schemes(scheme, dtype):
    """Every scheme through the lockstep fast path (contiguous VRs, Nt <= 512) on
    cfg1-shaped drops vs the oracle: V, row sequences and the per-rhs flop counters."""
    kz = _kz()
    T = 30
    ch = kz.generate("cfg1", range(4))
    host = kz.HostBatch.from_contiguous(ch)
    dev = host.to_device(dtype)
    k = host.n_users
    streams = None
    if scheme in kz.STOCHASTIC_SCHEMES:
        gens = [np.random.default_rng(kz.solver_seed_sequence(s)).spawn(k) for s in range(4)]
        streams = kz.HostStreams(scheme, gens, host.row_energy.reshape(4, k))
    res = kz.solve_batch(dev, scheme, mode="lockstep", max_iters=T, rng=streams, rows_cap=T)
    assert res.launches == 2  # the fused lockstep kernel + its n_outer finaliser
    for b in range(4):
        chan = oracle_channel_contiguous(ch, b)
        sys_ = O.AugmentedSystem.from_channel(chan, float(ch.reg[b]))
        ref = O.rzf_precoder(chan, float(ch.reg[b]))
        run = O.run_precoding(scheme, sys_, ref, epsilon=0.0, max_iters=T, traces=False,
                              rng=np.random.default_rng(kz.solver_seed_sequence(b)))
        v = res.v[b].cpu().numpy()
        if dtype == "c128":
            assert rel(v, run.v) <= REL_C128, b
            assert_rows(res.rows, run.rows, b)
            setup = 4 * ch.n_antennas * k
            asm = sum(6 * q * k + 2 * (q - 1) * k for q in
                      [sum(1 for vr in chan.vrs if n in vr.visible_subarrays) for n in range(ch.n_antennas)] if q)
            if scheme not in kz.VR_SCHEMES:
                asm = 6 * ch.n_antennas * k * k + 2 * ch.n_antennas * k * (k - 1)
            assert int(res.flops[b].sum()) + setup + asm == run.flops_measured
            assert int(res.noop_steps[b].sum()) == run.noop_steps
            np.testing.assert_array_equal(res.iters[b].cpu().numpy(), run.iters)
        else:
            if scheme in ("grk", "vr-ogrk", "gk"):
                # greedy picks may break fp32 near-ties differently, so V is judged through the north_star's
                # complex64 criterion: NMSE vs RZF and sum-rate against the complex128 oracle
                ep = kz.epilogue(dev.view(b, b + 1), res.v[b:b + 1], v_ref=O.auxiliary_matrix(chan, sys_.reg)[None],
                                 beta_ref=[ref.norm_factor], rates=True)
                f_run = O.assemble_dense(chan, run.v).f
                _, s128 = O.spectral_efficiency(chan.h, f_run, float(ch.snr_linear[b]))
                _c64_ok(float(ep["nmse"][0]), O.nmse(f_run, ref.f), float(ep["sum_rate"][0]), s128)
            else:
                assert rel(v, run.v) <= 1e-3
            if scheme in ("urk", "swor-erk"):  # host index streams: rows and flop counters exact in c64 too
                assert_rows(res.rows, run.rows, b)
                setup = 4 * ch.n_antennas * k
                asm = 6 * ch.n_antennas * k * k + 2 * ch.n_antennas * k * (k - 1)
                assert int(res.flops[b].sum()) + setup + asm == run.flops_measured
                np.testing.assert_array_equal(res.iters[b].cpu().numpy(), run.iters)
        assert int(res.n_outer[b]) == T


def test_register_resident_iterates_are_h_coef():
    """The M block written back by the fast kernel equals H V (col = H coef)."""
    import torch
    kz = _kz()
    ch = kz.generate("cfg2", range(8))
    dev = kz.HostBatch.from_contiguous(ch).to_device("c128")
    res = kz.solve_batch(dev, "vr-oahk", mode="lockstep", max_iters=20, want_iterates=True)
    hv = kz.epilogue(dev, res.v, want_f=True)
    f = (hv["f"] / hv["beta"][:, None, None]).transpose(1, 2).cpu().numpy()
    assert rel(res.iterates().cpu().numpy(), f) <= 1e-12


# --------------------------------------------------------------------------- BASELINE cfg3/4/5 shapes (reduced B)

def test_cfg4_residual_tolerance_solve_all():
    """cfg4 semantics (Nt=4096, K=256, VR=512): per-rhs residual tolerance 1e-4 (solve_all,
    solvers.py:510-537) for GRK and VR-OAHK on one realization, complex128, vs the oracle."""
    kz = _kz()
    ch = kz.generate("cfg4", [0])
    chan = oracle_channel_contiguous(ch, 0)
    reg = float(ch.reg[0])
    sys_ = O.AugmentedSystem.from_channel(chan, reg)
    for sc in ("vr-oahk", "grk"):
        # a fresh SeedSequence per generator: Generator.spawn advances the shared sequence
        stop = kz.StoppingRule(mode="residual", epsilon=1e-4)
        v_gpu = kz.solve_all(sc, sys_, stop, rng=np.random.default_rng(kz.solver_seed_sequence(0)))
        traces = []
        v_ref = O.solve_all(sc, sys_, O.StoppingRule(mode="residual", epsilon=1e-4),
                            rng=np.random.default_rng(kz.solver_seed_sequence(0)), traces=traces)
        assert rel(v_gpu, v_ref) <= REL_C128, sc
        assert all(t.converged for t in traces)


def test_cfg5_wideband_subcarriers_c128():
    """cfg5 shape: Nt=2048, K=128, frequency-dependent channels on shared VRs, AHK and
    VR-OAHK at T=10 on two subcarriers, complex128 vs the oracle."""
    kz = _kz()
    ch = kz.generate("cfg5", [0, [0, 1023]])
    dev = kz.HostBatch.from_contiguous(ch).to_device("c128")
    for sc in ("ahk", "vr-oahk"):
        res = kz.solve_batch(dev, sc, mode="lockstep", max_iters=10)
        for b in range(2):
            chan = oracle_channel_contiguous(ch, b)
            sys_ = O.AugmentedSystem.from_channel(chan, float(ch.reg[b]))
            run = O.run_precoding(sc, sys_, O.rzf_precoder(chan, float(ch.reg[b])), epsilon=0.0,
                                  max_iters=10, traces=False)
            assert rel(res.v[b].cpu().numpy(), run.v) <= REL_C128, (sc, b)


def test_cfg3_c64_vr_oahk_nmse_and_rate():
    """cfg3 shape (Nt=1024, K=128, VR ~ U[128,512]) in complex64: VR-OAHK T=30 NMSE and
    sum-rate within the c64 criterion of the complex128 oracle."""
    kz = _kz()
    ch = kz.generate("cfg3", [5, 6])
    dev64 = kz.HostBatch.from_contiguous(ch).to_device("c64")
    dev128 = kz.HostBatch.from_contiguous(ch).to_device("c128")
    rz = kz.rzf_batched(dev128)
    out = kz.run_precoding_batched("vr-oahk", dev64, max_iters=30, v_ref=rz["v"], beta_ref=rz["beta"])
    for b in range(2):
        chan = oracle_channel_contiguous(ch, b)
        reg = float(ch.reg[b])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        ref = O.rzf_precoder(chan, reg)
        run = O.run_precoding("vr-oahk", sys_, ref, epsilon=0.0, max_iters=30, traces=False)
        n128 = O.nmse(run.precoder.f, ref.f)
        s128 = O.spectral_efficiency(chan.h, run.precoder.f, float(ch.snr_linear[b]))[1]
        _c64_ok(float(out["nmse"][b]), n128, float(out["sum_rate"][b]), s128)


def test_c_abi_direct_call_as_in_integration_md():
    """The ctypes binding shown in INTEGRATION.md §3 drives kz_solve directly."""
    import ctypes as C
    import torch
    from paper_2501_10689_b200._lib import KzOut, KzRng, KzStop, SCHEME_IDS, check, lib
    kz = _kz()
    ch = kz.generate("cfg2", range(4))
    dev = kz.HostBatch.from_contiguous(ch).to_device("c64")
    lb = lib()
    stop = KzStop(mode=0, max_iters=50, check_every=1, epsilon=0.0)
    rng = KzRng(kind=3, seed=1)
    b, k = dev.n_systems, dev.n_users
    v = torch.zeros((b, k, k), dtype=torch.complex64, device="cuda")
    out = KzOut(v=v.data_ptr())
    ws = torch.empty(lb.kz_solve_workspace_bytes(C.byref(dev.problem), C.byref(stop)), dtype=torch.uint8,
                     device="cuda")
    check(lb.kz_solve(C.byref(dev.problem), SCHEME_IDS["grk"], C.byref(stop), C.byref(rng), C.byref(out),
                      ws.data_ptr(), ws.numel(), 0, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    res = kz.solve_batch(dev, "grk", mode="lockstep", max_iters=50, rng=("philox", 1))
    torch.testing.assert_close(v, res.v, rtol=0, atol=0)  # deterministic: identical bits


def test_gpu_traces_match_kaczplot_golden_csv():
    """The reference's cross-machine golden traces (pkg/kaczplot/tests/data/convergence.csv, kept as
    tests/golden/kaczplot_convergence.npz) through the GPU run_precoding in complex128: iteration
    counts and FlopCounter traces exact, NMSE within 1e-9 relative above 1e-9, true residual traces."""
    kz = _kz()
    z = load("kaczplot_convergence.npz")
    cfg = O.ArrayConfig(32, 100e9, 4)
    for seed in (0, 1):
        chan, reg = O.power_control(O.random_channel(cfg, 4, 5, 0.6, np.random.default_rng(seed)), 0.0)
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        ref = O.rzf_precoder(chan, reg)
        for sc in O.SCHEMES:
            rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(1,)))
            run = kz.run_precoding(sc, sys_, ref, epsilon=1e-6, max_iters=20_000, rng=rng)
            want_n = z[f"{sc}/{seed}/nmse"]
            assert run.n_iters == want_n.size, (sc, seed)
            np.testing.assert_array_equal(run.flops_trace, z[f"{sc}/{seed}/flops"])
            big = want_n > 1e-9
            np.testing.assert_allclose(np.asarray(run.nmse_trace)[big], want_n[big], rtol=1e-9)
            np.testing.assert_allclose(run.resid_trace, z[f"{sc}/{seed}/resid"], rtol=1e-8, atol=1e-14)


@pytest.mark.parametrize("scheme", ["urk", "grk", "vr-ogrk", "ahk", "vr-oahk"])
def test_bench_workload_c64_vs_c128_same_draws(scheme):
    """The benchmark workload (cfg2, T=200, on-device Philox draws) on 48 realizations: the complex64
    throughput kernels against the complex128 oracle-mode kernels fed the same Philox draws — NMSE vs RZF
    and sum-rate per system within the c64 criterion."""
    kz = _kz()
    ch = kz.generate("cfg2", range(48))
    host = kz.HostBatch.from_contiguous(ch)
    d64, d128 = host.to_device("c64"), host.to_device("c128")
    rz = kz.rzf_batched(d128)
    rng = ("philox", 2024) if scheme in kz.STOCHASTIC_SCHEMES else None
    o64 = kz.run_precoding_batched(scheme, d64, max_iters=200, rng=rng, v_ref=rz["v"], beta_ref=rz["beta"],
                                   rates=True)
    o128 = kz.run_precoding_batched(scheme, d128, max_iters=200, rng=rng, v_ref=rz["v"], beta_ref=rz["beta"],
                                    rates=True)
    n64, n128 = o64["nmse"].cpu().numpy(), o128["nmse"].cpu().numpy()
    assert np.all(c64_nmse_ok(n64, n128)), (n64, n128)
    np.testing.assert_allclose(o64["sum_rate"].cpu().numpy(), o128["sum_rate"].cpu().numpy(), rtol=1e-3)


def test_epilogue_gram_cache_is_exact():
    """kz_epilogue with KZ_PROBLEM_GRAM_CACHED (G0 from an earlier call on the same workspace) returns bitwise
    the same beta / NMSE / rates as recomputing G0 (the bench's five epilogues of one step share it)."""
    import torch
    kz = _kz()
    ch = kz.generate(kz.CONFIGS["cfg2"], range(8))
    dev = kz.HostBatch.from_contiguous(ch).to_device("c64")
    rz = kz.rzf_batched(dev)
    r1 = kz.solve_batch(dev, "ahk", mode="lockstep", max_iters=20)
    r2 = kz.solve_batch(dev, "grk", mode="lockstep", max_iters=20, rng=("philox", 3))
    e1 = kz.epilogue(dev, r1.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True)
    assert e1["gram_form"]
    fresh = kz.epilogue(dev, r2.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True)
    cached = kz.epilogue(dev, r2.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True, workspace=e1["workspace"],
                         gram_cached=True)
    for key in ("beta", "nmse", "rates", "sum_rate"):
        assert torch.equal(fresh[key], cached[key]), key
    with pytest.raises(ValueError):
        kz.epilogue(dev, r2.v, rates=True, gram_cached=True)


def test_cfg3_cfg5_c64_vs_oracle_at_stated_iterations():
    """The large-array configs at their stated iteration counts in complex64 against the complex128 oracle (not the
    GPU's own complex128 path): cfg3 VR-OAHK at T=200 on 8 realizations, cfg5 AHK and VR-OAHK at T=100 (the top of
    its sweep) on 4 subcarriers of one drop -- NMSE vs RZF per SURVEY §9.7 and the Eq. (7) sum-rate within 1e-3
    (north_star's complex64 criterion); the oracle runs on a spawn pool of host cores."""
    from helpers import oracle_precoding_task, spawn_pool_map
    kz = _kz()
    cases = [("cfg3", [s], "vr-oahk", 200) for s in range(20, 28)]
    cases += [("cfg5", [0, [m]], sc, 100) for m in (5, 300, 611, 1000) for sc in ("ahk", "vr-oahk")]
    want = spawn_pool_map(oracle_precoding_task, cases)
    for name, T in (("cfg3", 200), ("cfg5", 100)):
        mine = [(i, c) for i, c in enumerate(cases) if c[0] == name]
        seeds = [c[1][0] for _, c in mine] if name == "cfg3" else [0, [m for m in (5, 300, 611, 1000)]]
        ch = kz.generate(name, seeds)
        host = kz.HostBatch.from_contiguous(ch)
        d64 = host.to_device("c64")
        rz = kz.rzf_batched(host.to_device("c128"))
        for sc in sorted({c[2] for _, c in mine}):
            out = kz.run_precoding_batched(sc, d64, max_iters=T, v_ref=rz["v"], beta_ref=rz["beta"], rates=True)
            idx = [i for i, c in mine if c[2] == sc]
            for b, i in enumerate(idx):
                n128, s128 = want[i]
                n64, s64 = float(out["nmse"][b]), float(out["sum_rate"][b])
                assert c64_nmse_ok(n64, n128), (name, sc, b, n64, n128)
                assert s64 == pytest.approx(s128, rel=1e-3), (name, sc, b, s64, s128)


def _custom_contiguous(nt, starts, lengths, seed, snr_db=10.0):
    """One system with the given contiguous VRs (unit-norm random rows), as a ContiguousChannels batch."""
    from paper_2501_10689_b200.channel import ContiguousChannels
    rng = np.random.default_rng(seed)
    k = len(starts)
    vals, ptr = [], [0]
    for ln in lengths:
        v = rng.standard_normal(ln) + 1j * rng.standard_normal(ln)
        vals.append(v / np.linalg.norm(v))
        ptr.append(ptr[-1] + ln)
    snr = 10.0 ** (snr_db / 10.0)
    return ContiguousChannels(nt, k, np.asarray([starts], dtype=np.int32), np.asarray([lengths], dtype=np.int32),
                              np.concatenate(vals), np.asarray(ptr, dtype=np.int64), np.asarray([k / snr]),
                              np.asarray([snr]))


@pytest.mark.parametrize("case", ["all_orthogonal", "many_orthogonal_plus_overlap"])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_wide_vr_oahk_many_orthogonal_rows(case, dtype):
    """VR-OAHK on the register-resident kernels with more orthogonal rows than warps (the block step hands one O row
    to each warp in turn) and, in the first case, no non-orthogonal rows at all (no aggregated step, nothing
    pending for the coefficient update); the second case has short VRs inside single chunks, half pieces and an
    aggregated step whose q += gamma phi is applied by the next weights pass / flushed at the end.  Against the
    complex128 oracle (solvers.py:312-332, 407-421)."""
    kz = _kz()
    nt = 512
    if case == "all_orthogonal":
        starts, lengths = [16 * i for i in range(32)], [16] * 32          # 32 disjoint VRs: N is empty
    else:
        starts = [12 * i for i in range(24)] + [300 + 5 * i for i in range(16)]  # 24 disjoint + 16 overlapping
        lengths = [12] * 24 + [128] * 16
    ch = _custom_contiguous(nt, starts, lengths, seed=11)
    dev = kz.HostBatch.from_contiguous(ch).to_device(dtype)
    T = 6
    res = kz.solve_batch(dev, "vr-oahk", mode="lockstep", max_iters=T)
    chan = oracle_channel_contiguous(ch, 0)
    sys_ = O.AugmentedSystem.from_channel(chan, float(ch.reg[0]))
    if case == "all_orthogonal":
        assert len(sys_.partition.non_orthogonal) == 0
    else:
        assert len(sys_.partition.orthogonal) > 16 and len(sys_.partition.non_orthogonal) > 0
    run = O.run_precoding("vr-oahk", sys_, O.rzf_precoder(chan, float(ch.reg[0])), epsilon=0.0, max_iters=T,
                          traces=False)
    v = res.v[0].cpu().numpy()
    assert rel(v, run.v) <= (REL_C128 if dtype == "c128" else 1e-4)
    assert int(res.noop_steps[0].sum()) == run.noop_steps
    if dtype == "c128":
        np.testing.assert_array_equal(res.iters[0].cpu().numpy(), run.iters)
