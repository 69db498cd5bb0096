"""Input preparation cost per config: host numpy generation + packing + partition + H2D versus
DeviceBatch.from_drops (host drop draws + on-device synthesis and partition)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402

for c, B in (("cfg2", 1024), ("cfg3", 256), ("cfg4", 64), ("cfg5", 256)):
    cfg = kz.CONFIGS[c]
    seeds = [0, range(B)] if cfg.n_subcarriers > 1 else range(B)
    kz.DeviceBatch.from_drops(kz.generate_drops(cfg, range(2) if cfg.n_subcarriers == 1 else [0, range(2)]), "c64")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev = kz.HostBatch.from_contiguous(kz.generate(cfg, seeds)).to_device("c64")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dr = kz.generate_drops(cfg, seeds)
    t2 = time.perf_counter()
    dev2 = kz.DeviceBatch.from_drops(dr, "c64")
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{c} B={B}: host path {1e3 * (t1 - t0):.1f} ms; drops {1e3 * (t2 - t1):.1f} ms + device build "
          f"{1e3 * (t3 - t2):.1f} ms  ({(t1 - t0) / (t3 - t1):.0f}x)", flush=True)
