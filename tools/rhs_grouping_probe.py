"""How much of a residual-mode cluster launch is lockstep waste (rhs already converged while the cluster's slowest
rhs runs on), and how much an rhs-to-cluster grouping by a per-rhs feature would recover.

    python tools/rhs_grouping_probe.py [--config cfg4] [--batch 16]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--scheme", default="grk")
a = ap.parse_args()
cfg = kz.CONFIGS[a.config]
ch = kz.generate(cfg, range(a.batch))
host = kz.HostBatch.from_contiguous(ch)
dev = host.to_device("c64")
k = ch.n_users
res = kz.solve_batch(dev, a.scheme, mode="residual", epsilon=cfg.extra["residual_tol"], max_iters=10000 * k,
                     check_every=1, rng=("philox", 5) if a.scheme in kz.STOCHASTIC_SCHEMES else None)
its = res.iters.cpu().numpy().astype(float)  # (B, K)
G = 32
cp = host.coupled_ptr
ncoup = np.diff(cp).reshape(a.batch, k).astype(float)
energy = host.row_energy.reshape(a.batch, k)
start = ch.start.astype(float)


def waste(order):
    tot = used = 0.0
    for b in range(a.batch):
        o = order(b)
        for g in range(0, k, G):
            grp = its[b, o[g:g + G]]
            used += grp.sum()
            tot += grp.max() * len(grp)
    return used / tot


print(f"{a.config} {a.scheme} B={a.batch}: mean iters {its.mean():.2f}, max {its.max():.0f}")
print(f"  useful lane fraction, rhs in index order (the kernel's):  {waste(lambda b: np.arange(k)):.3f}")
print(f"  sorted by the iteration count itself (upper bound):     {waste(lambda b: np.argsort(its[b])):.3f}")
# overlap mass: sum over the coupled rows of the shared support length (contiguous VRs)
L = ch.length.astype(float)
ov = np.zeros((a.batch, k))
for b in range(a.batch):
    s_, e_ = start[b], start[b] + L[b]
    ov[b] = np.clip(np.minimum(e_[:, None], e_[None, :]) - np.maximum(s_[:, None], s_[None, :]), 0, None).sum(axis=1)
# |<h_c, h_j>|^2 summed over j (the Gram row energy)
gram = np.zeros((a.batch, k))
for b in range(a.batch):
    h = ch.dense(b)
    g = np.abs(h.conj().T @ h) ** 2
    gram[b] = g.sum(axis=1) - np.diag(g)
for name, feat in (("coupled-set size", ncoup), ("row energy", energy), ("VR start", start),
                   ("overlap mass", ov), ("Gram row energy", gram), ("|X| + overlap/L", ncoup + ov / L)):
    r = np.corrcoef(feat.ravel(), its.ravel())[0, 1]
    print(f"  sorted by {name:17s} (corr {r:+.2f}):                {waste(lambda b: np.argsort(feat[b])):.3f}")
