"""Per-config kernel timings (cfg1..cfg5 of BASELINE.json) on one GPU.

    python tools/bench_configs.py [--configs cfg3,cfg4] [--batch N] [--json out.jsonl]

For each config: RZF, every scheme's solve (lockstep fixed T, or residual
tolerance for cfg4) and the epilogue, timed with CUDA events after a warm-up,
plus rhs-iterations/s, elements streamed per rhs-iteration and the FP32 FMA
fraction (8 flops per complex MAC of the algorithmic work).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402

DEFAULT_B = {"cfg1": 1024, "cfg2": 1024, "cfg3": 1024, "cfg4": 256, "cfg5": 512}
FFMA_PEAK = 68.34e12  # profiles/r01_microbench.json


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best, out


def elements_per_iter(scheme, host, b, k):
    """Mean algorithmic elements streamed per rhs-iteration."""
    lens = np.diff(host.row_val_ptr).reshape(b, k).astype(np.float64)
    tot = lens.sum(axis=1).mean()
    mean_l = lens.mean()
    if scheme in ("grk", "gk"):
        return tot + mean_l
    if scheme in ("urk", "swor-erk"):
        return 2 * mean_l
    if scheme in ("ahk", "vr-oahk"):
        return 2 * tot
    if scheme == "vr-ogrk":
        cp = np.diff(host.coupled_ptr).astype(np.float64)
        return cp.mean() * mean_l + mean_l
    raise ValueError(scheme)


def run(cfg_name, batch, dtype, out):
    cfg = kz.CONFIGS[cfg_name]
    seeds = [0, range(batch)] if cfg.n_subcarriers > 1 else range(batch)
    ch = kz.generate(cfg, seeds)
    host = kz.HostBatch.from_contiguous(ch)
    dev = host.to_device(dtype)
    b, k = dev.n_systems, dev.n_users
    t_rzf, rz = timed(lambda: kz.rzf_batched(dev))
    print(f"{cfg_name} B={b} K={k} Nt={dev.n_antennas} {dtype}: rzf {t_rzf:.2f} ms", flush=True)
    tol = cfg.extra.get("residual_tol")
    for scheme in cfg.schemes:
        rng = ("philox", 7) if scheme in kz.STOCHASTIC_SCHEMES else None
        if tol:
            fn = lambda: kz.solve_batch(dev, scheme, mode="residual", epsilon=tol,  # noqa: E731
                                        max_iters=10000 * k, check_every=1, rng=rng)
        else:
            fn = lambda: kz.solve_batch(dev, scheme, mode="lockstep", max_iters=cfg.n_iters, rng=rng)  # noqa: E731
        t_solve, res = timed(fn)
        iters = res.iters.double().sum().item()
        t_epi, ep = timed(lambda: kz.epilogue(dev, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True))
        e_it = elements_per_iter(scheme, host, b, k)
        rate = iters / (t_solve * 1e-3)
        frac = rate * e_it * 8 / FFMA_PEAK
        rec = {"config": cfg_name, "scheme": scheme, "dtype": dtype, "B": b, "K": k, "Nt": dev.n_antennas,
               "rzf_ms": round(t_rzf, 3), "solve_ms": round(t_solve, 3), "epilogue_ms": round(t_epi, 3),
               "mean_iters": round(iters / (b * k), 2), "launches": res.launches,
               "rhs_iter_per_s": rate, "elements_per_rhs_iter": round(e_it, 1),
               "fp32_fma_frac": round(frac, 4),
               "precoders_per_s": b / ((t_rzf + t_solve + t_epi) * 1e-3),
               "nmse_median": float(ep["nmse"].median().item())}
        print(json.dumps(rec), flush=True)
        if out:
            out.write(json.dumps(rec) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg2,cfg3,cfg4,cfg5")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    out = open(a.json, "a") if a.json else None
    for c in a.configs.split(","):
        run(c, a.batch or DEFAULT_B[c], a.dtype, out)


if __name__ == "__main__":
    main()
