import os, sys
sys.path.insert(0, os.getcwd())
import paper_2501_10689_b200 as kz
ch = kz.generate("cfg2", range(2))
dev = kz.HostBatch.from_contiguous(ch).to_device("c64")
print("val range", dev.problem.val_lo, dev.problem.val_hi, flush=True)
a = kz.solve_batch(dev, "vr-oahk", mode="lockstep", max_iters=5)
print("tma", a.tma_staging, flush=True)
