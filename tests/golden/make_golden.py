"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the build container, where the read-only reference checkout exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed as
small .npz fixtures.  Row sequences are captured by wrapping
kaczprec.solvers.select_row (InstanceRun.step calls it by module-global name,
solvers.py:388,393,401), keyed by the state's rhs.

Fixtures
  ref_lockstep.npz   reference test drop (Nt=64,K=8,S=8,L=5,p=0.5,0 dB, seed 0), all 7
                     schemes, run_precoding(eps=1e-6, rng=default_rng(42))
                     (= tests/test_solvers.py:505-523 frozen counts)
  ref_fixed_t.npz    conftest-scale drops (Nt=32,K=4,S=4,L=3,p=0.6) seeds 0-3, all
                     schemes, fixed T=15 (eps=0), rng=default_rng(100+seed)
  ref_solve.npz      per-column solve() at Nt=64,K=8 seed 1: residual and oracle modes
  ref_cfg1.npz       BASELINE cfg1-shaped inputs (contiguous VRs, lambda/(4 pi r) LoS,
                     unit columns, xi=K/SNR), 3 realizations, GRK T=50 + RZF + rates
  ref_cfg2.npz       BASELINE cfg2-shaped, 1 realization, the 5 cfg2 schemes, T=200
  ref_cfg2_philox.npz  BASELINE cfg2-shaped, realizations 0-1, urk / grk / vr-ogrk at T=200 with the row draws
                     of the throughput mode: the reference's rng is oracle.philox.PhiloxGenerator(seed, b),
                     whose spawned children serve the device's Philox4x32-10 draws (pins the draw shim and the
                     device keying against the real reference)
  kaczplot_convergence.npz   per-iteration nmse/resid/flops of the reference's own
                     golden CSV pkg/kaczplot/tests/data/convergence.csv
"""

from __future__ import annotations

import csv
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import kaczprec  # noqa: E402
import kaczprec.solvers as ks  # noqa: E402
from kaczprec.channel import (ArrayConfig, ChannelMatrix, VisibilityRegion, power_control,  # noqa: E402
                              random_channel)

from paper_2501_10689_b200.channel import CONFIGS, generate, solver_seed_sequence  # noqa: E402

_real_select = ks.select_row
_LOG = None


def _recording_select(strategy, state, sys_, rng=None):
    i = _real_select(strategy, state, sys_, rng)
    if _LOG is not None and i is not None:
        _LOG[state.rhs].append(i)
    return i


ks.select_row = _recording_select


def run_logged(scheme, sys_, ref, eps, rng, max_iters=None):
    global _LOG
    _LOG = [[] for _ in range(sys_.n_users)]
    run = ks.run_precoding(scheme, sys_, ref, epsilon=eps, max_iters=max_iters, rng=rng)
    rows = _LOG
    _LOG = None
    return run, rows


def pad_rows(rows, width):
    out = np.full((len(rows), max(width, 1)), -1, dtype=np.int16)
    for c, r in enumerate(rows):
        out[c, :len(r)] = r
    return out


def vr_mask(chan):
    m = np.zeros((chan.n_users, chan.cfg.n_subarrays), dtype=bool)
    for k, vr in enumerate(chan.vrs):
        m[k, sorted(vr.visible_subarrays)] = True
    return m


def ref_drop(seed, nt, k, s, paths, p, snr=0.0, f=100e9):
    cfg = ArrayConfig(n_antennas=nt, carrier_freq=f, n_subarrays=s)
    chan = random_channel(cfg, k, paths, p, np.random.default_rng(seed))
    return power_control(chan, snr)


def lockstep_fixture():
    chan, reg = ref_drop(0, 64, 8, 8, 5, 0.5)
    sys_ = kaczprec.AugmentedSystem.from_channel(chan, reg)
    ref = kaczprec.rzf_precoder(chan, reg)
    out = {"h": chan.h, "reg": reg, "vr_mask": vr_mask(chan), "n_subarrays": 8, "f_ref": ref.f,
           "beta_ref": ref.norm_factor, "v_ref": kaczprec.auxiliary_matrix(chan, reg)}
    for sc in ks.SCHEMES:
        run, rows = run_logged(sc, sys_, ref, 1e-6, np.random.default_rng(42))
        out[f"{sc}/n_iters"] = run.n_iters
        out[f"{sc}/converged"] = run.converged
        out[f"{sc}/v"] = run.v
        out[f"{sc}/f"] = run.precoder.f
        out[f"{sc}/nmse_trace"] = np.asarray(run.nmse_trace)
        out[f"{sc}/resid_trace"] = np.asarray(run.resid_trace)
        out[f"{sc}/flops_trace"] = np.asarray(run.flops_trace, dtype=np.int64)
        out[f"{sc}/flops_measured"] = run.flops_measured
        out[f"{sc}/noop_steps"] = run.noop_steps
        out[f"{sc}/rows"] = pad_rows(rows, run.n_iters)
    np.savez_compressed(os.path.join(HERE, "ref_lockstep.npz"), **out)


def fixed_t_fixture():
    out = {}
    for seed in range(4):
        chan, reg = ref_drop(seed, 32, 4, 4, 3, 0.6)
        sys_ = kaczprec.AugmentedSystem.from_channel(chan, reg)
        ref = kaczprec.rzf_precoder(chan, reg)
        out[f"{seed}/h"] = chan.h
        out[f"{seed}/reg"] = reg
        out[f"{seed}/vr_mask"] = vr_mask(chan)
        out[f"{seed}/f_ref"] = ref.f
        _, out[f"{seed}/rzf_sum_rate"] = kaczprec.spectral_efficiency(chan.h, ref.f, 1.0 / reg)
        for sc in ks.SCHEMES:
            run, rows = run_logged(sc, sys_, ref, 0.0, np.random.default_rng(100 + seed), max_iters=15)
            out[f"{seed}/{sc}/v"] = run.v
            out[f"{seed}/{sc}/f"] = run.precoder.f
            out[f"{seed}/{sc}/rows"] = pad_rows(rows, 15)
            out[f"{seed}/{sc}/nmse"] = run.nmse_trace[-1]
            out[f"{seed}/{sc}/flops_measured"] = run.flops_measured
            out[f"{seed}/{sc}/noop_steps"] = run.noop_steps
            _, out[f"{seed}/{sc}/sum_rate"] = kaczprec.spectral_efficiency(chan.h, run.precoder.f, 1.0 / reg)
    np.savez_compressed(os.path.join(HERE, "ref_fixed_t.npz"), **out)


def solve_fixture():
    global _LOG
    chan, reg = ref_drop(1, 64, 8, 8, 5, 0.5)
    sys_ = kaczprec.AugmentedSystem.from_channel(chan, reg)
    vref = kaczprec.auxiliary_matrix(chan, reg)
    out = {"h": chan.h, "reg": reg, "vr_mask": vr_mask(chan), "v_ref": vref}
    for mode, eps in (("residual", 1e-8), ("oracle", 1e-6)):
        for sc in ks.SCHEMES:
            kids = np.random.default_rng(7).spawn(8)
            v = np.zeros((8, 8), dtype=complex)
            iters, conv, rows = [], [], []
            last_resid, n_checks = [], []
            for c in range(8):
                _LOG = [[] for _ in range(8)]
                stop = ks.StoppingRule(mode=mode, epsilon=eps,
                                       reference=vref[:, c] if mode == "oracle" else None, check_every=2)
                st, tr = ks.solve(sc, sys_, c, stop, rng=kids[c])
                rows.append(_LOG[c])
                _LOG = None
                v[:, c] = st.coef
                iters.append(tr.n_iters)
                conv.append(tr.converged)
                last_resid.append(tr.resid[-1])
                n_checks.append(len(tr.resid))
            # solve_all with the same rng must agree (solvers.py:510-537)
            va = ks.solve_all(sc, sys_, ks.StoppingRule(mode=mode, epsilon=eps,
                                                        reference=vref if mode == "oracle" else None,
                                                        check_every=2),
                              rng=np.random.default_rng(7))
            assert np.array_equal(va, v)
            key = f"{mode}/{sc}"
            out[f"{key}/v"] = v
            out[f"{key}/iters"] = np.asarray(iters)
            out[f"{key}/converged"] = np.asarray(conv)
            out[f"{key}/rows"] = pad_rows(rows, max(len(r) for r in rows))
            out[f"{key}/last_resid"] = np.asarray(last_resid)
            out[f"{key}/n_checks"] = np.asarray(n_checks)
    np.savez_compressed(os.path.join(HERE, "ref_solve.npz"), **out)


def contiguous_reference(ch, b):
    """Reference ChannelMatrix for system b of a ContiguousChannels batch (1-antenna subarrays)."""
    nt, k = ch.n_antennas, ch.n_users
    cfg = ArrayConfig(n_antennas=nt, carrier_freq=30e9, n_subarrays=nt)
    vrs = tuple(VisibilityRegion(frozenset(range(int(ch.start[b, i]), int(ch.start[b, i] + ch.length[b, i]))), nt, 1)
                for i in range(k))
    return ChannelMatrix(h=ch.dense(b), vrs=vrs, cfg=cfg)


def config_fixture(name, seeds, schemes, iters, fname):
    cfgd = CONFIGS[name]
    ch = generate(cfgd, seeds)
    out = {"start": ch.start, "length": ch.length, "heff": ch.heff, "row_val_ptr": ch.row_val_ptr,
           "reg": ch.reg, "snr_linear": ch.snr_linear, "seeds": np.asarray(seeds), "n_antennas": ch.n_antennas,
           "n_iters": iters}
    for b, seed in enumerate(seeds):
        chan = contiguous_reference(ch, b)
        reg = float(ch.reg[b])
        sys_ = kaczprec.AugmentedSystem.from_channel(chan, reg)
        ref = kaczprec.rzf_precoder(chan, reg)
        out[f"{b}/v_ref"] = kaczprec.auxiliary_matrix(chan, reg)
        out[f"{b}/beta_ref"] = ref.norm_factor
        out[f"{b}/orthogonal"] = np.asarray(sys_.partition.orthogonal_sorted)
        _, out[f"{b}/rzf_sum_rate"] = kaczprec.spectral_efficiency(chan.h, ref.f, float(ch.snr_linear[b]))
        for sc in schemes:
            rng = np.random.default_rng(solver_seed_sequence(int(seed)))
            run, rows = run_logged(sc, sys_, ref, 0.0, rng, max_iters=iters)
            out[f"{b}/{sc}/v"] = run.v
            out[f"{b}/{sc}/rows"] = pad_rows(rows, iters)
            out[f"{b}/{sc}/nmse"] = run.nmse_trace[-1]
            out[f"{b}/{sc}/flops_measured"] = run.flops_measured
            _, out[f"{b}/{sc}/sum_rate"] = kaczprec.spectral_efficiency(chan.h, run.precoder.f,
                                                                        float(ch.snr_linear[b]))
    np.savez_compressed(os.path.join(HERE, fname), **out)


PHILOX_SEED = 2024


def philox_fixture(seeds, schemes, iters, fname):
    from oracle.philox import PhiloxGenerator
    cfgd = CONFIGS["cfg2"]
    ch = generate(cfgd, seeds)
    out = {"seeds": np.asarray(seeds), "n_iters": iters, "philox_seed": PHILOX_SEED}
    for b, seed in enumerate(seeds):
        chan = contiguous_reference(ch, b)
        reg = float(ch.reg[b])
        sys_ = kaczprec.AugmentedSystem.from_channel(chan, reg)
        ref = kaczprec.rzf_precoder(chan, reg)
        for sc in schemes:
            run, rows = run_logged(sc, sys_, ref, 0.0, PhiloxGenerator(PHILOX_SEED, int(seed)), max_iters=iters)
            out[f"{b}/{sc}/v"] = run.v
            out[f"{b}/{sc}/rows"] = pad_rows(rows, iters)
            out[f"{b}/{sc}/nmse"] = run.nmse_trace[-1]
            _, out[f"{b}/{sc}/sum_rate"] = kaczprec.spectral_efficiency(chan.h, run.precoder.f,
                                                                        float(ch.snr_linear[b]))
    np.savez_compressed(os.path.join(HERE, fname), **out)


def kaczplot_fixture():
    path = "/root/reference/pkg/kaczplot/tests/data/convergence.csv"
    with open(path) as fh:
        rows = [r for r in csv.reader(line for line in fh if not line.startswith("#"))]
    head, body = rows[0], rows[1:]
    col = {n: i for i, n in enumerate(head)}
    out = {}
    for sc in ks.SCHEMES:
        for seed in (0, 1):
            sel = [r for r in body if r[col["scheme"]] == sc and int(r[col["seed"]]) == seed]
            sel.sort(key=lambda r: int(r[col["iter"]]))
            out[f"{sc}/{seed}/nmse"] = np.array([float(r[col["nmse"]]) for r in sel])
            out[f"{sc}/{seed}/resid"] = np.array([float(r[col["resid"]]) for r in sel])
            out[f"{sc}/{seed}/flops"] = np.array([int(r[col["flops_measured"]]) for r in sel], dtype=np.int64)
    out["config"] = np.array("N_t=32 K=4 S=4 f_Hz=100e9 p=0.6 L=5 snr_db=0 epsilon=1e-6 max_iters=20000")
    np.savez_compressed(os.path.join(HERE, "kaczplot_convergence.npz"), **out)


if __name__ == "__main__":
    only = set(sys.argv[1:])
    if not only or "lockstep" in only:
        lockstep_fixture()
    if not only or "fixed_t" in only:
        fixed_t_fixture()
    if not only or "solve" in only:
        solve_fixture()
    if not only or "cfg1" in only:  # BASELINE cfg1: all 100 seeded realizations
        config_fixture("cfg1", list(range(100)), ["grk"], 50, "ref_cfg1.npz")
    if not only or "cfg2" in only:
        config_fixture("cfg2", [0], ["urk", "grk", "vr-ogrk", "ahk", "vr-oahk"], 200, "ref_cfg2.npz")
    if not only or "philox" in only:
        philox_fixture([0, 1], ["urk", "grk", "vr-ogrk"], 200, "ref_cfg2_philox.npz")
    if not only or "kaczplot" in only:
        kaczplot_fixture()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
