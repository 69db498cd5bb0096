import sys, os
sys.path.insert(0, "/root/repo")
import torch, paper_2501_10689_b200 as kz
c = sys.argv[1]
cfg = kz.CONFIGS[c]
ch = kz.generate(cfg, range(int(sys.argv[2])))
dev = kz.HostBatch.from_contiguous(ch).to_device("c64")
for _ in range(2):
    rz = kz.rzf_batched(dev)
torch.cuda.synchronize()
