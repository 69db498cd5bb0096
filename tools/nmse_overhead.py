"""Per-iteration cost of the on-chip NMSE check: the same T iterations run fixed-T, with only the flop trace (one
cluster exchange, no F_ref reads) and NMSE-checked at an unreachable tolerance (two exchanges + F_ref reads)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402

B = int(os.environ.get("B", "256"))
T = 200
ch = kz.generate("cfg2", range(B))
host = kz.HostBatch.from_contiguous(ch)
rz = kz.rzf_batched(host.to_device("c128"), want_f=True)
for dt in ("c64", "c128"):
    dev = host.to_device(dt)
    for sc in ("grk", "ahk", "vr-oahk"):
        rng = ("philox", 3) if sc in kz.STOCHASTIC_SCHEMES else None
        for mode, kw in (("fixed", {}), ("flops-trace", dict(trace_cap=T, traces=("flops",))),
                         ("nmse eps=1e-30", dict(epsilon=1e-30, f_ref=rz["f"]))):
            run = lambda: kz.solve_batch(dev, sc, mode="lockstep", max_iters=T, rng=rng, **kw)  # noqa: E731
            r = run()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(3):
                r = run()
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) / 3 * 1e3
            print(f"{dt} {sc:8s} {mode:15s} {ms:7.2f} ms  outer {float(r.n_outer.float().mean()):.0f}  "
                  f"launches {r.launches}", flush=True)
