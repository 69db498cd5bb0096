"""RZF timings per config: blocked Gauss-Jordan kernel vs the legacy unblocked Cholesky kernel
(KZ_RZF_LEGACY=1, run in a child process), with the relative difference of V and beta."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402

B = {"cfg1": 1024, "cfg2": 1024, "cfg3": 512, "cfg4": 128, "cfg5": 256}
if __name__ == "__main__":
    tag = "legacy" if "KZ_RZF_LEGACY" in os.environ else "gj"
    confs = sys.argv[1].split(",")
    for c in confs:
        cfg = kz.CONFIGS[c]
        ch = kz.generate(cfg, [0, range(B[c])] if cfg.n_subcarriers > 1 else range(B[c]))
        dev = kz.HostBatch.from_contiguous(ch).to_device("c64")
        rz = kz.rzf_batched(dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rz = kz.rzf_batched(dev)
        e1.record()
        torch.cuda.synchronize()
        np.save(f"/tmp/rzf_{tag}_{c}.npy", rz["v"][:8].cpu().numpy())
        np.save(f"/tmp/rzfb_{tag}_{c}.npy", rz["beta"][:8].cpu().numpy())
        print(f"{c} B={B[c]} K={ch.n_users}: rzf {e0.elapsed_time(e1):.3f} ms ({tag})", flush=True)
    if tag == "gj":
        subprocess.run([sys.executable, __file__, sys.argv[1]], env=dict(os.environ, KZ_RZF_LEGACY="1"), check=True)
        for c in confs:
            a, b = np.load(f"/tmp/rzf_gj_{c}.npy"), np.load(f"/tmp/rzf_legacy_{c}.npy")
            ba, bb = np.load(f"/tmp/rzfb_gj_{c}.npy"), np.load(f"/tmp/rzfb_legacy_{c}.npy")
            print(f"{c}: rel V {np.linalg.norm(a - b) / np.linalg.norm(b):.2e}  rel beta {np.max(np.abs(ba / bb - 1)):.2e}")
