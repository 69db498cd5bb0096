"""Small invocations of every kernel of libkaczmarz_b200.so, for compute-sanitizer (one tool per run):

    compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_cases.py
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py
    compute-sanitizer --tool initcheck python tools/sanitize_cases.py

Covers: the wide register-resident kernel (all 7 schemes, incl. the TMEM-parked aggregation), the warp-per-rhs
RK kernel, the chunked lockstep kernel (complex128, all schemes), the cluster kernel (DSMEM inbox; lockstep and
residual mode), the global-memory generic kernel (NMSE stop with traces), RZF, both epilogue forms, channel
synthesis + partition.  Sizes are tiny (sanitizers replay every access).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402


def main():
    only = set(sys.argv[1:])
    T = 3
    ch2 = kz.generate("cfg2", range(2))
    host2 = kz.HostBatch.from_contiguous(ch2)
    d64, d128 = host2.to_device("c64"), host2.to_device("c128")
    if not only or "wide" in only:
        for sc in kz.SCHEMES:
            rng = ("philox", 1) if sc in kz.STOCHASTIC_SCHEMES else None
            kz.solve_batch(d64, sc, mode="lockstep", max_iters=T, rng=rng, rows_cap=T, want_iterates=True)
            kz.solve_batch(d128, sc, mode="lockstep", max_iters=T, rng=rng, rows_cap=T, want_iterates=True)
        torch.cuda.synchronize()
        print("wide / rkwarp / lockstep ok", flush=True)
    if not only or "cluster" in only:
        big = kz.NearFieldConfig("san", 1024, 40, (96, 400))
        chb = kz.generate(big, range(1))
        db = kz.HostBatch.from_contiguous(chb).to_device("c64")
        for sc in ("gk", "grk", "vr-ogrk", "ahk", "vr-oahk"):
            rng = ("philox", 2) if sc in kz.STOCHASTIC_SCHEMES else None
            kz.solve_batch(db, sc, mode="lockstep", max_iters=T, rng=rng, rows_cap=T, want_iterates=True)
            kz.solve_batch(db, sc, mode="residual", epsilon=1e-2, max_iters=50, rng=rng)
        torch.cuda.synchronize()
        print("cluster ok", flush=True)
    if not only or "dense" in only:
        rz = kz.rzf_batched(d128)
        res = kz.solve_batch(d64, "ahk", mode="lockstep", max_iters=T)
        kz.epilogue(d64, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True)               # Gram form
        kz.epilogue(d64, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True, want_f=True)  # per antenna
        ch1 = kz.generate("cfg1", range(2))
        d1 = kz.HostBatch.from_contiguous(ch1).to_device("c64")
        r1 = kz.solve_batch(d1, "grk", mode="lockstep", max_iters=T, rng=("philox", 3))
        kz.epilogue(d1, r1.v, rates=True)
        kz.epilogue(d1, r1.v, v_ref=kz.rzf_batched(d1)["v"], beta_ref=torch.ones(2, dtype=torch.float64, device="cuda"))
        torch.cuda.synchronize()
        print("rzf / epilogue ok", flush=True)
    if not only or "drops" in only:
        kz.DeviceBatch.from_drops(kz.generate_drops("cfg3", range(2)), dtype="c64")
        torch.cuda.synchronize()
        print("drops ok", flush=True)
    if not only or "generic" in only:
        # the global-memory kernel: NMSE-stopped lockstep with traces (complex128), per-rhs residual mode with
        # check_every
        ch1 = kz.generate("cfg1", range(2))
        d1 = kz.HostBatch.from_contiguous(ch1).to_device("c128")
        f_ref = kz.rzf_batched(d1, want_f=True)["f"]
        for sc in ("grk", "vr-oahk"):
            rng = ("philox", 4) if sc in kz.STOCHASTIC_SCHEMES else None
            kz.solve_batch(d1, sc, mode="lockstep", max_iters=20, epsilon=1e-3, f_ref=f_ref, rng=rng, trace_cap=20)
            kz.solve_batch(d1, sc, mode="residual", max_iters=50, epsilon=1e-3, check_every=2, rng=rng,
                           trace_cap=64, want_iterates=True)
        torch.cuda.synchronize()
        print("generic ok", flush=True)

if __name__ == "__main__":
    main()
