"""RZF and Gram-form epilogue timings with the Gram on the FP64 tensor cores (default) vs the CUDA-core pair sums
(KZ_GRAM_TC=0, child process), with the relative difference of V."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402

B = {"cfg1": 1024, "cfg2": 1024, "cfg3": 512, "cfg4": 128, "cfg5": 1024}


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


if __name__ == "__main__":
    tag = "cuda-core" if os.environ.get("KZ_GRAM_TC") == "0" else "tensor-core"
    confs = sys.argv[1].split(",")
    for c in confs:
        cfg = kz.CONFIGS[c]
        ch = kz.generate(cfg, [0, range(B[c])] if cfg.n_subcarriers > 1 else range(B[c]))
        for dt in ("c64", "c128"):
            dev = kz.HostBatch.from_contiguous(ch).to_device(dt)
            ms, rz = timed(lambda: kz.rzf_batched(dev))
            v = rz["v"].to(torch.complex64 if dt == "c64" else torch.complex128)
            ems, ep = timed(lambda: kz.epilogue(dev, v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True))
            np.save(f"/tmp/gtc_{tag}_{c}_{dt}.npy", rz["v"][:16].cpu().numpy())
            print(f"{c} {dt} B={B[c]} K={ch.n_users}: rzf {ms:.3f} ms, epilogue {ems:.3f} ms "
                  f"(gram form {ep['gram_form']}, {tag})", flush=True)
    if tag == "tensor-core":
        subprocess.run([sys.executable, __file__, sys.argv[1]], env=dict(os.environ, KZ_GRAM_TC="0"), check=True)
        for c in confs:
            for dt in ("c64", "c128"):
                a, b = np.load(f"/tmp/gtc_tensor-core_{c}_{dt}.npy"), np.load(f"/tmp/gtc_cuda-core_{c}_{dt}.npy")
                print(f"{c} {dt}: rel V {np.linalg.norm(a - b) / np.linalg.norm(b):.2e}")
