"""Pin the CPU oracle to the reference: committed fixtures from the real
reference (tests/golden/make_golden.py) plus the reference tests' own frozen
known answers.  CPU only."""

import math

import numpy as np
import pytest

import oracle as O
from helpers import contiguous_from_fixture, load, oracle_channel_contiguous, oracle_channel_from_mask

SCHEMES = O.SCHEMES


def test_frozen_lockstep_iteration_counts():
    """tests/test_solvers.py:505-523 of the reference: urk 127 ... vr-oahk 8."""
    cfg = O.ArrayConfig(64, 100e9, 8)
    chan, reg = O.power_control(O.random_channel(cfg, 8, 5, 0.5, np.random.default_rng(0)), 0.0)
    sys_ = O.AugmentedSystem.from_channel(chan, reg)
    ref = O.rzf_precoder(chan, reg)
    expected = {"urk": 127, "swor-erk": 56, "gk": 33, "grk": 37, "vr-ogrk": 37, "ahk": 10, "vr-oahk": 8}
    flops = {}
    for sc, t in expected.items():
        run = O.run_precoding(sc, sys_, ref, epsilon=1e-6, rng=np.random.default_rng(42))
        assert run.converged and run.n_iters == t, sc
        flops[sc] = run.flops_measured
    assert flops["vr-ogrk"] < 0.5 * flops["grk"]


def test_frozen_single_rhs_counts():
    """tests/test_solvers.py:435-446: gk 32, urk 93 (rng 7)."""
    cfg = O.ArrayConfig(64, 100e9, 8)
    chan, reg = O.power_control(O.random_channel(cfg, 8, 5, 0.5, np.random.default_rng(0)), 0.0)
    sys_ = O.AugmentedSystem.from_channel(chan, reg)
    vref = O.auxiliary_matrix(chan, reg)
    _, tr = O.solve("gk", sys_, 0, O.StoppingRule(epsilon=1e-6, reference=vref[:, 0]))
    assert tr.n_iters == 32
    _, tr = O.solve("urk", sys_, 0, O.StoppingRule(epsilon=1e-6, reference=vref[:, 0]),
                    rng=np.random.default_rng(7))
    assert tr.n_iters == 93


def test_rzf_frozen_entries():
    """tests/test_rzf.py:33-51: seed-1234 8x3, xi = 0.4."""
    rng = np.random.default_rng(1234)
    h = (rng.standard_normal((8, 3)) + 1j * rng.standard_normal((8, 3))) / math.sqrt(2)
    v = O.auxiliary_matrix(h, 0.4)
    assert v[0, 0] == pytest.approx(0.08743823337750342 + 0j, abs=1e-10)
    assert v[1, 2] == pytest.approx(-0.00047276679288917284 - 0.0117275702144454j, abs=1e-10)
    prec = O.rzf_precoder(h, 0.4)
    assert prec.norm_factor == pytest.approx(1.8189422748831143, rel=1e-10)
    assert prec.f[0, 0] == pytest.approx(-0.16744310691337447 + 0.09294283936181302j, abs=1e-10)


def test_sum_rate_hand_case():
    """tests/test_metrics.py:63-70: every rate exactly 1."""
    h = np.zeros((4, 2), dtype=complex)
    h[0, 0] = h[1, 1] = 1.0
    rates, total = O.spectral_efficiency(h, h / math.sqrt(2), 2.0)
    np.testing.assert_allclose(rates, [1.0, 1.0], rtol=1e-14)
    assert total == pytest.approx(2.0)


def test_lockstep_fixture_bitwise():
    z = load("ref_lockstep.npz")
    chan = oracle_channel_from_mask(z["h"], z["vr_mask"], z["n_subarrays"])
    reg = float(z["reg"])
    sys_ = O.AugmentedSystem.from_channel(chan, reg)
    ref = O.rzf_precoder(chan, reg)
    np.testing.assert_allclose(ref.f, z["f_ref"], rtol=0, atol=1e-14)
    for sc in SCHEMES:
        run = O.run_precoding(sc, sys_, ref, epsilon=1e-6, rng=np.random.default_rng(42))
        assert run.n_iters == int(z[f"{sc}/n_iters"]), sc
        assert run.flops_measured == int(z[f"{sc}/flops_measured"]), sc
        assert run.noop_steps == int(z[f"{sc}/noop_steps"]), sc
        np.testing.assert_array_equal(run.v, z[f"{sc}/v"])
        np.testing.assert_array_equal(np.asarray(run.flops_trace), z[f"{sc}/flops_trace"])
        np.testing.assert_allclose(run.nmse_trace, z[f"{sc}/nmse_trace"], rtol=1e-12, atol=0)
        rows = z[f"{sc}/rows"]
        for c in range(8):
            got = run.rows[c]
            np.testing.assert_array_equal(got, rows[c, :len(got)])
            assert np.all(rows[c, len(got):] == -1)


def test_fixed_t_fixture():
    z = load("ref_fixed_t.npz")
    for seed in range(4):
        chan = oracle_channel_from_mask(z[f"{seed}/h"], z[f"{seed}/vr_mask"], 4)
        reg = float(z[f"{seed}/reg"])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        ref = O.rzf_precoder(chan, reg)
        for sc in SCHEMES:
            run = O.run_precoding(sc, sys_, ref, epsilon=0.0, max_iters=15,
                                  rng=np.random.default_rng(100 + seed))
            np.testing.assert_array_equal(run.v, z[f"{seed}/{sc}/v"])
            assert run.flops_measured == int(z[f"{seed}/{sc}/flops_measured"])
            _, sr = O.spectral_efficiency(chan.h, run.precoder.f, 1.0 / reg)
            assert sr == pytest.approx(float(z[f"{seed}/{sc}/sum_rate"]), rel=1e-13)


def test_solve_fixture():
    z = load("ref_solve.npz")
    chan = oracle_channel_from_mask(z["h"], z["vr_mask"], 8)
    reg = float(z["reg"])
    sys_ = O.AugmentedSystem.from_channel(chan, reg)
    vref = z["v_ref"]
    for mode, eps in (("residual", 1e-8), ("oracle", 1e-6)):
        for sc in SCHEMES:
            traces = []
            v = O.solve_all(sc, sys_, O.StoppingRule(mode=mode, epsilon=eps,
                                                     reference=vref if mode == "oracle" else None,
                                                     check_every=2),
                            rng=np.random.default_rng(7), traces=traces)
            key = f"{mode}/{sc}"
            np.testing.assert_array_equal(v, z[f"{key}/v"])
            np.testing.assert_array_equal([t.n_iters for t in traces], z[f"{key}/iters"])
            np.testing.assert_array_equal([t.converged for t in traces], z[f"{key}/converged"])
            np.testing.assert_array_equal([len(t.resid) for t in traces], z[f"{key}/n_checks"])


@pytest.mark.parametrize("name", ["ref_cfg1.npz", "ref_cfg2.npz"])
def test_config_fixtures(name):
    z = load(name)
    ch = contiguous_from_fixture(z)
    iters = int(z["n_iters"])
    schemes = sorted({k.split("/")[1] for k in z.files if k.count("/") == 2})
    for b, seed in enumerate(z["seeds"]):
        chan = oracle_channel_contiguous(ch, b)
        reg = float(ch.reg[b])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        assert np.array_equal(np.asarray(sys_.partition.orthogonal_sorted), z[f"{b}/orthogonal"])
        ref = O.rzf_precoder(chan, reg)
        np.testing.assert_allclose(O.auxiliary_matrix(chan, reg), z[f"{b}/v_ref"], rtol=0, atol=1e-13)
        for sc in schemes:
            rng = np.random.default_rng(np.random.SeedSequence(entropy=int(seed), spawn_key=(1,)))
            run = O.run_precoding(sc, sys_, ref, epsilon=0.0, max_iters=iters, rng=rng, traces=False)
            np.testing.assert_array_equal(run.v, z[f"{b}/{sc}/v"])
            rows = z[f"{b}/{sc}/rows"]
            for c in range(ch.n_users):
                np.testing.assert_array_equal(run.rows[c], rows[c, :len(run.rows[c])])


def test_kaczplot_golden_csv():
    """The reference's own cross-machine golden (pkg/kaczplot/tests/data/convergence.csv)."""
    z = load("kaczplot_convergence.npz")
    cfg = O.ArrayConfig(32, 100e9, 4)
    for seed in (0, 1):
        chan, reg = O.power_control(O.random_channel(cfg, 4, 5, 0.6, np.random.default_rng(seed)), 0.0)
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        ref = O.rzf_precoder(chan, reg)
        for sc in SCHEMES:
            rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(1,)))
            run = O.run_precoding(sc, sys_, ref, epsilon=1e-6, max_iters=20_000, rng=rng)
            want_n = z[f"{sc}/{seed}/nmse"]
            assert run.n_iters == want_n.size, (sc, seed)
            np.testing.assert_array_equal(run.flops_trace, z[f"{sc}/{seed}/flops"])
            big = want_n > 1e-9
            np.testing.assert_allclose(np.asarray(run.nmse_trace)[big], want_n[big], rtol=1e-9)
            np.testing.assert_allclose(run.resid_trace, z[f"{sc}/{seed}/resid"], rtol=1e-8, atol=1e-14)


# --------------------------------------------------------------------------- throughput-mode draws (oracle/philox.py)

def test_philox_known_answers():
    """Philox4x32-10 known-answer vectors of its publication (Salmon et al., SC'11: zero, all-ones and pi-digit
    counter/key pairs) for the numpy restatement of the device's draw generator."""
    from oracle.philox import philox4x32_10
    cases = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
             ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
             ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
              (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in cases:
        got = philox4x32_10(np.array([ctr], dtype=np.uint32), key[0], key[1])[0]
        assert [int(x) for x in got] == list(want)


def test_philox_uniform_keying_and_range():
    from oracle.philox import philox_uniform
    u = philox_uniform(2024, np.arange(64)[:, None], 3, np.arange(200)[None, :])
    assert u.shape == (64, 200) and np.all((u >= 0) & (u < 1))
    assert abs(u.mean() - 0.5) < 0.01
    # one (system, rhs, draw) evaluated alone equals its entry in the broadcast evaluation
    assert philox_uniform(2024, 17, 3, 123) == u[17, 123]
    assert philox_uniform(2025, 17, 3, 123) != u[17, 123]


def test_philox_choice_is_numpy_generator_choice():
    """The shim's choice(n, p) is numpy Generator.choice's own algorithm on the stream's next uniform
    (cumsum, normalise by the last entry, searchsorted right): checked against numpy itself with twin PCG64
    generators over random weight vectors."""
    from oracle.philox import PhiloxStream
    rs = np.random.default_rng(5)
    for trial in range(300):
        k = int(rs.integers(1, 200))
        w = rs.random(k) ** 4
        if trial % 7 == 0:
            w[rs.integers(k)] = 0.0
        p = w / w.sum()
        g1, g2 = np.random.default_rng(trial), np.random.default_rng(trial)
        want = int(g1.choice(k, p=p))
        s = PhiloxStream(0, 0, 0)
        s._next = lambda g=g2: float(g.random())  # feed the twin generator's uniform
        assert s.choice(k, p=p) == want


def test_philox_fixture_reference_bitwise():
    """The oracle port fed the device's Philox draws (PhiloxGenerator) reproduces the REAL reference run with the
    same draws (tests/golden/ref_cfg2_philox.npz, cfg2 realizations 0-1, urk / grk / vr-ogrk, T = 200): row
    sequences and V bitwise."""
    from oracle.philox import PhiloxGenerator
    z = load("ref_cfg2_philox.npz")
    from paper_2501_10689_b200.channel import generate
    seeds = [int(s) for s in z["seeds"]]
    ch = generate("cfg2", seeds)
    T = int(z["n_iters"])
    for b, seed in enumerate(seeds):
        chan = oracle_channel_contiguous(ch, b)
        reg = float(ch.reg[b])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        ref = O.rzf_precoder(chan, reg)
        for sc in ("urk", "grk", "vr-ogrk"):
            run = O.run_precoding(sc, sys_, ref, epsilon=0.0, max_iters=T,
                                  rng=PhiloxGenerator(int(z["philox_seed"]), seed), traces=False)
            np.testing.assert_array_equal(run.v, z[f"{b}/{sc}/v"])
            rows = z[f"{b}/{sc}/rows"]
            for c in range(ch.n_users):
                np.testing.assert_array_equal(run.rows[c], rows[c, :len(run.rows[c])])


# --------------------------------------------------------------------------- grouped VR-OAHK (oracle/grouped.py)

def test_grouped_restatement_limit_is_reference_vr_oahk():
    """One orthogonal group and an aggregation cap >= |N| is the reference's vr-oahk: bitwise equal to the REAL
    reference's fixed-T runs (tests/golden/ref_fixed_t.npz, Bernoulli-subarray drops, T = 15) -- V and flop
    counts -- so the restatement is anchored to the reference path it extends."""
    from oracle.grouped import run_precoding_grouped
    z = load("ref_fixed_t.npz")
    for seed in range(4):
        chan = oracle_channel_from_mask(z[f"{seed}/h"], z[f"{seed}/vr_mask"], 4)
        reg = float(z[f"{seed}/reg"])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        run = run_precoding_grouped(sys_, O.rzf_precoder(chan, reg), 1, sys_.n_users, 15)
        np.testing.assert_array_equal(run.v, z[f"{seed}/vr-oahk/v"])
        assert run.flops_measured == int(z[f"{seed}/vr-oahk/flops_measured"])


def test_grouped_partition_properties():
    """Groups are pairwise VR-disjoint (mutually orthogonal rows), disjoint from each other and from N, cover
    every row; group 1 is the reference's maximal independent set; each group's block step solves its rows
    exactly (Theorem 4: their residuals vanish right after the step)."""
    from oracle.grouped import GroupedRun, grouped_partition
    from paper_2501_10689_b200.channel import generate
    ch = generate("cfg3", [3])
    chan = oracle_channel_contiguous(ch, 0)
    sys_ = O.AugmentedSystem.from_channel(chan, float(ch.reg[0]))
    groups, non = grouped_partition(chan.vrs, 4)
    assert tuple(groups[0]) == sys_.partition.orthogonal_sorted
    seen = set()
    for g in groups:
        for a in g:
            for b in g:
                if a < b:
                    assert not (chan.vrs[a].visible_subarrays & chan.vrs[b].visible_subarrays)
        assert not (seen & set(g))
        seen |= set(g)
    assert seen | set(non) == set(range(sys_.n_users)) and not (seen & set(non))
    assert list(non) == sorted(non)
    run = GroupedRun(sys_, 5, groups, non, 8)
    st = run.state
    for g in groups:
        O.residual_refresh(st, sys_, rows=np.asarray(g), use_vr=True)
        O.orthogonal_block_step(st, sys_, np.asarray(g), use_vr=True)
        O.residual_refresh(st, sys_, rows=np.asarray(g), use_vr=True)
        assert np.max(np.abs(st.resid[list(g)])) <= 1e-13


def test_grouped_aggregation_cap_blocks():
    """agg_cap splits N into consecutive ascending blocks; every setting contracts the error towards RZF."""
    from oracle.grouped import run_precoding_grouped
    from paper_2501_10689_b200.channel import generate
    ch = generate("cfg3", [1])
    chan = oracle_channel_contiguous(ch, 0)
    reg = float(ch.reg[0])
    sys_ = O.AugmentedSystem.from_channel(chan, reg)
    ref = O.rzf_precoder(chan, reg)
    for ng, cap in ((1, 8), (4, 8), (2, 3)):
        e1 = run_precoding_grouped(sys_, ref, ng, cap, 1).nmse_trace[-1]
        e3 = run_precoding_grouped(sys_, ref, ng, cap, 3).nmse_trace[-1]
        assert e3 < e1 < 1.0, (ng, cap, e1, e3)
