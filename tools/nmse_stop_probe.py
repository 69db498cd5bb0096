import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, paper_2501_10689_b200 as kz
ch = kz.generate("cfg2", range(256))
host = kz.HostBatch.from_contiguous(ch)
for dt in ("c64", "c128"):
    dev = host.to_device(dt)
    rz = kz.rzf_batched(host.to_device("c128"), want_f=True)
    for sc in ("grk", "vr-oahk"):
        rng = ("philox", 3) if sc == "grk" else None
        for mode in ("fixed", "nmse"):
            kw = dict(mode="lockstep", max_iters=200, rng=rng)
            if mode == "nmse":
                kw.update(epsilon=1e-6, f_ref=rz["f"])
            r = kz.solve_batch(dev, sc, **kw); torch.cuda.synchronize()
            t0 = time.perf_counter(); r = kz.solve_batch(dev, sc, **kw); torch.cuda.synchronize(); t = time.perf_counter() - t0
            print(dt, sc, mode, f"{t*1e3:.1f} ms", "mean outer iters", float(r.n_outer.float().mean()) if r.n_outer is not None else None, "launches", r.launches)
