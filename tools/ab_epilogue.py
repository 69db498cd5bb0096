"""A/B of the epilogue paths (Gram form vs per-antenna windows, KZ_EPILOGUE_ANTENNA=1 in a child) on the
solver output of a config: beta, NMSE, sum-rate agreement and kernel time."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402

c, B, sc, T, dt = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), sys.argv[5]
tag = "antenna" if "KZ_EPILOGUE_ANTENNA" in os.environ else "gram"
cfg = kz.CONFIGS[c]
ch = kz.generate(cfg, [0, range(B)] if cfg.n_subcarriers > 1 else range(B))
dev = kz.HostBatch.from_contiguous(ch).to_device(dt)
rz = kz.rzf_batched(dev)
res = kz.solve_batch(dev, sc, mode="lockstep", max_iters=T, rng=("philox", 1) if sc in kz.STOCHASTIC_SCHEMES else None)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ep = kz.epilogue(dev, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True)
    e1.record()
    torch.cuda.synchronize()
print(f"{c} {sc} {dt} B={B}: epilogue {e0.elapsed_time(e1):.3f} ms ({tag})", flush=True)
np.savez(f"/tmp/ep_{tag}.npz", beta=ep["beta"].cpu().numpy(), nmse=ep["nmse"].cpu().numpy(),
         sr=ep["sum_rate"].cpu().numpy(), rates=ep["rates"].cpu().numpy())
if tag == "gram":
    subprocess.run([sys.executable] + sys.argv, env=dict(os.environ, KZ_EPILOGUE_ANTENNA="1"), check=True)
    a, b = np.load("/tmp/ep_gram.npz"), np.load("/tmp/ep_antenna.npz")
    for key in ("beta", "nmse", "sr", "rates"):
        print(f"  {key}: max rel diff {np.max(np.abs(a[key] / b[key] - 1)):.3e}")
    print("  nmse gram:", a["nmse"][:4], " antenna:", b["nmse"][:4])
