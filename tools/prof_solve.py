"""Run one lockstep solve of a cfg workload (for ncu / timing).

    python tools/prof_solve.py --scheme grk --dtype c64 --batch 1024 --iters 200 [--reps 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--scheme", default="grk")
ap.add_argument("--dtype", default="c64")
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--residual", type=float, default=0.0, help="residual tolerance (solve_all semantics); 0: fixed T")
ap.add_argument("--groups", type=int, default=1, help="orthogonal groups per system (vr-oahk-g)")
ap.add_argument("--cap", type=int, default=0, help="hyperplanes per aggregated step (vr-oahk-g; 0: all)")
ap.add_argument("--dump", default="", help="save V, iters, flops of the last run to this .npz (bitwise A/B of builds)")
a = ap.parse_args()
cfg = kz.CONFIGS[a.config]
ch = kz.generate(cfg, [0, range(a.batch)] if cfg.n_subcarriers > 1 else range(a.batch))
dev = kz.HostBatch.from_contiguous(ch, orth_groups=a.groups, agg_cap=a.cap).to_device(a.dtype)
rng = ("philox", 7) if a.scheme in kz.STOCHASTIC_SCHEMES else None
times = []
for r in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if a.residual:
        res = kz.solve_batch(dev, a.scheme, mode="residual", epsilon=a.residual, max_iters=10000 * dev.n_users,
                             check_every=1, rng=rng)
    else:
        res = kz.solve_batch(dev, a.scheme, mode="lockstep", max_iters=a.iters, rng=rng)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
    print(f"{a.scheme} {a.dtype} B={a.batch} T={a.iters}: {times[-1]:.3f} ms (launches {res.launches})")
times.sort()
print(f"{a.scheme} {a.dtype} B={a.batch} T={a.iters}: min {times[0]:.3f} ms, median {times[len(times) // 2]:.3f} ms "
      f"over {len(times)} (launches {res.launches})")
if a.dump:
    import numpy as np
    np.savez(a.dump, v=res.v.cpu().numpy(), iters=res.iters.cpu().numpy(),
             flops=res.flops.cpu().numpy() if res.flops is not None else np.zeros(0))
