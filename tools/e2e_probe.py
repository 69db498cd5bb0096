"""Where the end-to-end step's extra time goes (bench.py e2e vs the device step): variants timed over 5 steps.

    python tools/e2e_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402

cfg = kz.CONFIGS["cfg2"]
B, T = 1024, 200
schemes = ["urk", "grk", "vr-ogrk", "ahk", "vr-oahk"]
host = kz.HostBatch.from_contiguous(kz.generate(cfg, range(B)))
dev = host.to_device("c64")
pinned = kz.pin_host(host, "c64")
stream = torch.cuda.current_stream()
copy_stream = torch.cuda.Stream()
outs = {sc: (torch.empty((B, 64, 64), dtype=torch.complex64).pin_memory(), torch.empty(B, dtype=torch.float64).pin_memory(),
             torch.empty(B, dtype=torch.float64).pin_memory()) for sc in schemes}
ws = None


def step(upload, d2h, s):
    global ws
    d = kz.DeviceBatch(host, "c64", pinned=pinned) if upload else dev
    rz = kz.rzf_batched(d)
    ews, gram = None, False
    for sc in schemes:
        res = kz.solve_batch(d, sc, mode="lockstep", max_iters=T, rng=("philox", s) if sc in kz.STOCHASTIC_SCHEMES else None,
                             workspace=ws)
        ws = res.workspace
        ep = kz.epilogue(d, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True, workspace=ews, gram_cached=gram)
        ews, gram = ep["workspace"], ep["gram_form"]
        if d2h:
            ev = torch.cuda.Event()
            ev.record(stream)
            copy_stream.wait_event(ev)
            with torch.cuda.stream(copy_stream):
                for src, dst in zip((res.v, ep["nmse"], ep["sum_rate"]), outs[sc]):
                    src.record_stream(copy_stream)
                    dst.copy_(src, non_blocking=True)
    stream.wait_stream(copy_stream)


for upload, d2h in ((False, False), (True, False), (False, True), (True, True)):
    step(upload, d2h, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(1, 6):
        step(upload, d2h, s)
    e1.record()
    torch.cuda.synchronize()
    st = torch.cuda.memory_stats()
    print(f"upload={upload} d2h={d2h}: {e0.elapsed_time(e1) / 5:.2f} ms/step; cudaMalloc retries "
          f"{st.get('num_alloc_retries', 0)}, segments {st.get('segment.all.current', 0)}")
