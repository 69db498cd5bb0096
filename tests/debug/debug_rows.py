"""Find the first row-sequence divergence between the GPU (c128) and the oracle for
solve_all residual mode on one realization of a config; print the CDF margin."""
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # test-side debugging aid
sys.path[:0] = [_ROOT, os.path.join(_ROOT, "tests")]
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2501_10689_b200 as kz  # noqa: E402
from helpers import oracle_channel_contiguous  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
scheme = sys.argv[2] if len(sys.argv) > 2 else "grk"
ch = kz.generate(cfg, [0])
chan = oracle_channel_contiguous(ch, 0)
reg = float(ch.reg[0])
sys_ = O.AugmentedSystem.from_channel(chan, reg)
k = sys_.n_users
host = kz.HostBatch.from_systems([sys_])
dev = host.to_device("c128")
ss = kz.solver_seed_sequence(0)
streams = kz.HostStreams(scheme, [np.random.default_rng(ss).spawn(k)], host.row_energy.reshape(1, k))
res = kz.solve_batch(dev, scheme, mode="residual", max_iters=100000, epsilon=1e-4, rng=streams, rows_cap=4096)
traces = []
O.solve_all(scheme, sys_, O.StoppingRule(mode="residual", epsilon=1e-4), rng=np.random.default_rng(ss), traces=traces)
rows = res.rows[0].cpu().numpy()
iters = res.iters[0].cpu().numpy()
bad = 0
for c in range(k):
    g = rows[c][rows[c] >= 0]
    w = np.asarray(traces[c].rows)
    if len(g) != len(w) or np.any(g != w):
        bad += 1
        n = min(len(g), len(w))
        d = int(np.argmax(g[:n] != w[:n])) if np.any(g[:n] != w[:n]) else n
        if bad <= 5:
            print(f"rhs {c}: gpu iters {iters[c]} oracle {traces[c].n_iters}; first diff at step {d}: "
                  f"gpu {g[d] if d < len(g) else None} oracle {w[d] if d < len(w) else None}")
            # replay the oracle to step d and report the CDF margin of the uniform
            kids = np.random.default_rng(ss).spawn(k)
            run = O.InstanceRun(scheme, sys_, c, kids[c])
            for _ in range(d):
                run.step()
            st = run.state
            O.residual_refresh(st, sys_, use_vr=False)
            wts = np.abs(st.resid) ** 2
            p = wts / wts.sum()
            cdf = np.cumsum(p)
            cdf /= cdf[-1]
            u = np.random.default_rng(ss).spawn(k)[c].random(d + 1)[d]
            j = int(np.searchsorted(cdf, u, "right"))
            print(f"    u={u:.17g} cdf[j-1]={cdf[j-1] if j else 0:.17g} cdf[j]={cdf[j]:.17g} "
                  f"margin={min(abs(u - cdf[j]), abs(u - (cdf[j-1] if j else 0))):.3e} total={wts.sum():.3e}")
print("rhs with divergent rows:", bad, "of", k)
