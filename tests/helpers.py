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


def oracle_cfg2_philox_task(args):
    """One cfg2 realization through the oracle port fed the device's Philox draws (worker of a spawn pool:
    regenerates its own channel).  Returns rows (K, T) int16 (-1 padded), V, NMSE vs RZF and the Eq. (7)
    sum-rate, for the scheme."""
    system, scheme, seed, iters = args
    from threadpoolctl import threadpool_limits
    from oracle.philox import PhiloxGenerator
    from paper_2501_10689_b200.channel import generate
    with threadpool_limits(1):
        ch = generate("cfg2", [system])
        chan = oracle_channel_contiguous(ch, 0)
        reg = float(ch.reg[0])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        ref = O.rzf_precoder(chan, reg)
        rng = PhiloxGenerator(seed, system) if scheme in ("urk", "swor-erk", "grk", "vr-ogrk") else None
        run = O.run_precoding(scheme, sys_, ref, epsilon=0.0, max_iters=iters, rng=rng, traces=False)
        rows = np.full((ch.n_users, iters), -1, dtype=np.int16)
        for c, r in enumerate(run.rows):
            rows[c, :len(r)] = r
        f = O.assemble_dense(chan, run.v).f
        _, sr = O.spectral_efficiency(chan.h, f, float(ch.snr_linear[0]))
        return {"system": system, "scheme": scheme, "rows": rows, "v": run.v, "nmse": O.nmse(f, ref.f),
                "sum_rate": sr}


def spawn_pool_map(fn, tasks, max_workers=None):
    """Map fn over tasks on a spawn-context process pool (safe after CUDA initialisation: the workers never
    touch the GPU), one task at a time per worker, order preserved."""
    import multiprocessing as mp
    n = max_workers or min(len(tasks), len(os.sched_getaffinity(0)))
    with mp.get_context("spawn").Pool(processes=max(1, n)) as pool:
        return pool.map(fn, tasks, chunksize=1)


def oracle_solve_columns_task(args):
    """Per-rhs `solve` (residual mode) of columns `cols` of realization `system` of a named config, the
    stochastic schemes fed the device's Philox draws (spawn-pool worker).  Returns (cols, V columns, iters)."""
    cfg_name, system, scheme, cols, seed, eps = args
    from threadpoolctl import threadpool_limits
    from oracle.philox import PhiloxGenerator
    from paper_2501_10689_b200.channel import generate
    with threadpool_limits(1):
        ch = generate(cfg_name, [system])
        chan = oracle_channel_contiguous(ch, 0)
        sys_ = O.AugmentedSystem.from_channel(chan, float(ch.reg[0]))
        kids = PhiloxGenerator(seed, system).spawn(ch.n_users)
        vcols, iters = [], []
        for c in cols:
            st, tr = O.solve(scheme, sys_, c, O.StoppingRule(mode="residual", epsilon=eps), rng=kids[c])
            vcols.append(st.coef)
            iters.append(tr.n_iters)
        return cols, np.stack(vcols, axis=1), iters


C64_REL = 1e-3      # north_star: complex64 NMSE / sum-rate within 1e-3 relative
C64_FLOOR = 1e-6    # the complex64 NMSE floor (~5e-8 measured on cfg2) sits below this


def c64_nmse_ok(n64, n128):
    """SURVEY.md §9.7 complex64 NMSE criterion, elementwise: within 1e-3 relative of the complex128 NMSE where
    that is above 1e-5; below it (within a few decades of the fp32 floor, where fp32 rounding of F alone moves
    the NMSE by ~1e-8) the two agree to 1e-6 absolute (for a c128 NMSE at 1e-15 this is NMSE_64 <= 1e-6)."""
    n64, n128 = np.asarray(n64, dtype=np.float64), np.asarray(n128, dtype=np.float64)
    return np.where(n128 >= 1e-5, np.abs(n64 - n128) <= C64_REL * n128, np.abs(n64 - n128) <= C64_FLOOR)


def oracle_precoding_task(args):
    """run_precoding (fixed T, deterministic scheme) of one system of a named config through the oracle port
    (spawn-pool worker: regenerates its channel from the seeds spec given to channel.generate).  Returns the
    complex128 NMSE vs RZF and the Eq. (7) sum-rate."""
    cfg_name, seeds, scheme, iters = args
    from threadpoolctl import threadpool_limits
    from paper_2501_10689_b200.channel import generate
    with threadpool_limits(1):
        ch = generate(cfg_name, seeds)
        chan = oracle_channel_contiguous(ch, 0)
        reg = float(ch.reg[0])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        ref = O.rzf_precoder(chan, reg)
        run = O.run_precoding(scheme, sys_, ref, epsilon=0.0, max_iters=iters, traces=False)
        f = O.assemble_dense(chan, run.v).f
        _, sr = O.spectral_efficiency(chan.h, f, float(ch.snr_linear[0]))
        return O.nmse(f, ref.f), sr


def oracle_cfg2_nmse_stop_task(args):
    """run_precoding with the NMSE stop (solvers.py:556-603) on cfg2 realization `system`, the greedy schemes fed
    the device's Philox draws (spawn-pool worker).  Returns the stop iteration, converged flag and NMSE trace."""
    system, scheme, seed, eps = args[:4]
    cap = args[4] if len(args) > 4 else 2000
    from threadpoolctl import threadpool_limits
    from oracle.philox import PhiloxGenerator
    from paper_2501_10689_b200.channel import generate
    with threadpool_limits(1):
        ch = generate("cfg2", [system])
        chan = oracle_channel_contiguous(ch, 0)
        reg = float(ch.reg[0])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)
        ref = O.rzf_precoder(chan, reg)
        rng = PhiloxGenerator(seed, system) if scheme in ("urk", "swor-erk", "grk", "vr-ogrk") else None
        run = O.run_precoding(scheme, sys_, ref, epsilon=eps, max_iters=cap, rng=rng)
        return {"system": system, "scheme": scheme, "n": run.n_iters, "conv": run.converged,
                "trace": np.asarray(run.nmse_trace), "flops": np.asarray(run.flops_trace), "v": run.v,
                "rows": [np.asarray(r, dtype=np.int32) for r in run.rows]}
