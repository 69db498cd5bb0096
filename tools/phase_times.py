"""Per-phase cycle breakdown of the lockstep kernels (timing build).

    python -m paper_2501_10689_b200.build --timing
    KZ_LIB_VARIANT=timing python tools/phase_times.py --scheme grk [--chunked]
Phases: 0 = setup; then one slot per CTA barrier inside an iteration, in order.
"""
import argparse
import os
import sys

os.environ.setdefault("KZ_LIB_VARIANT", "timing")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scheme", default="grk")
ap.add_argument("--dtype", default="c64")
ap.add_argument("--batch", type=int, default=296)
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--config", default="cfg2")
ap.add_argument("--cluster-w", type=int, default=0, help="warps per CTA of the cluster kernel (0: wide/chunked)")
ap.add_argument("--cluster-g", type=int, default=16, help="rhs per cluster of the cluster kernel (KZ_VERBOSE=1 shows the pick)")
ap.add_argument("--residual", type=float, default=0.0, help="residual-tolerance mode (solve_all semantics) instead of fixed T")
a = ap.parse_args()
cfg = kz.CONFIGS[a.config]
ch = kz.generate(cfg, [0, range(a.batch)] if cfg.n_subcarriers > 1 else range(a.batch))
dev = kz.HostBatch.from_contiguous(ch).to_device(a.dtype)
rng = ("philox", 3) if a.scheme in kz.STOCHASTIC_SCHEMES else None
if a.residual:
    def run(ws=None):
        return kz.solve_batch(dev, a.scheme, mode="residual", epsilon=a.residual, max_iters=10000 * dev.n_users,
                              check_every=1, rng=rng, workspace=ws)
else:
    def run(ws=None):
        return kz.solve_batch(dev, a.scheme, mode="lockstep", max_iters=a.iters, rng=rng, workspace=ws)
res = run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res = run(res.workspace)
if a.residual:
    a.iters = max(1, int(round(res.iters.double().mean().item())))
    print(f"residual mode: mean iters {res.iters.double().mean().item():.2f}, max {res.iters.max().item()}")
e1.record()
torch.cuda.synchronize()
B, K, Nt = dev.n_systems, dev.n_users, dev.n_antennas
import ctypes  # noqa: E402
from paper_2501_10689_b200 import _lib  # noqa: E402
lb = _lib.lib()
ws = res.workspace
cs = 16 if a.dtype == "c128" else 8
# generic layout total = offset of tstop; recompute from the end: tstop region starts at ws.numel() - extra
extra = ((B * K * 4 + 8 + 255) // 256 * 256) + B * K * 44 * 8
base = ws.numel() - extra
off = base + (B * K * 4 + 7) // 8 * 8
G = (32 if K > 16 and not os.environ.get("KZ_CHUNKED_C64") else 16) if a.dtype == "c64" else 8
ncta = B * ((K + G - 1) // G)
if a.cluster_w:
    CL = -(-Nt // (32 * a.cluster_w))
    ncta = min(B * K, B * -(-K // a.cluster_g) * CL)
raw = ws[off:off + ncta * 44 * 8].view(torch.int64).view(ncta, 44).cpu().numpy().astype(np.float64)
ph = raw[:, :12].copy()
wst = raw[:, 12:12 + Nt // 32] / a.iters  # per-warp refresh-end cycles per iteration
Nt_ = Nt
ns = ph[:, 10].copy()
smid = ph[:, 11].astype(int)
ph[:, 10:] = 0
tot = ph.sum(axis=1)
print(f"  CTA wall {ns.mean() / 1e3:.1f} us mean, cycles/ns {np.mean(tot / ns):.3f} GHz; SMs used {len(set(smid))}; "
      f"CTAs per SM max {np.bincount(smid).max()}")
print(f"{a.scheme} {a.dtype} B={B} T={a.iters} kernel {e0.elapsed_time(e1):.2f} ms; cycles/CTA mean {tot.mean():.3e}")
per_it = ph[:, 1:].mean(axis=0) / a.iters
if wst.max() > 0:
    print("  per-warp refresh end (cyc/iter, mean over CTAs):", " ".join(f"{x:.0f}" for x in wst.mean(axis=0)))
    print(f"  slowest warp per CTA: mean {wst.max(axis=1).mean():.0f}  fastest: {wst.min(axis=1).mean():.0f}")
print(f"  setup {ph[:, 0].mean():.0f} cyc ({ph[:, 0].mean() / tot.mean() * 100:.1f}%)")
marks = raw[:, 36:44]
if marks.max() > 0:  # KZ_SETUP_MARK checkpoints (cycles since kernel start, thread 0), as increments
    m = marks.mean(axis=0)
    print("  setup checkpoints (cyc since start, mean over CTAs):", " ".join(f"{x:.0f}" for x in m))
for q, v in enumerate(per_it, start=1):
    if v > 0:
        print(f"  phase {q}: {v:8.0f} cyc/iter ({v * a.iters / tot.mean() * 100:5.1f}%)")
