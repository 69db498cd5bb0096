import os, sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import numpy as np
import oracle as O
import paper_2501_10689_b200 as kz
from paper_2501_10689_b200.channel import NearFieldConfig
from helpers import oracle_channel_contiguous

for nt, k, L in [(512, 64, 128), (512, 128, 128), (512, 256, 64), (1024, 128, 128), (1024, 256, 128), (4096, 64, 512)]:
    cfg = NearFieldConfig("dbg", nt, k, (L, L))
    ch = kz.generate(cfg, [0])
    chan = oracle_channel_contiguous(ch, 0)
    sys_ = O.AugmentedSystem.from_channel(chan, float(ch.reg[0]))
    host = kz.HostBatch.from_systems([sys_])
    dev = host.to_device("c128")
    for mode in ("residual", "lockstep"):
        T = 8
        streams = kz.HostStreams("grk", [np.random.default_rng(3).spawn(k)], host.row_energy.reshape(1, k))
        if mode == "residual":
            res = kz.solve_batch(dev, "grk", mode="residual", max_iters=T, epsilon=1e-30, rng=streams, rows_cap=T)
        else:
            res = kz.solve_batch(dev, "grk", mode="lockstep", max_iters=T, rng=streams, rows_cap=T)
        run = O.run_precoding("grk", sys_, O.rzf_precoder(chan, float(ch.reg[0])), epsilon=0.0, max_iters=T,
                              rng=np.random.default_rng(3), traces=False)
        rows = res.rows[0].cpu().numpy()
        bad = sum(1 for c in range(k) if list(rows[c][rows[c] >= 0]) != run.rows[c])
        err = np.linalg.norm(res.v[0].cpu().numpy() - run.v) / np.linalg.norm(run.v)
        print(f"Nt={nt} K={k} L={L} {mode:9s}: divergent rhs {bad}/{k}, rel err {err:.2e}, launches {res.launches}", flush=True)
