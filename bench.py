"""Benchmark of the batched Kaczmarz precoding hot path (BASELINE.json configs[1] = cfg2).

One step = one full pass of the cfg2 workload over this rank's realizations:
the direct RZF reference (K2), then for each of the five cfg2 schemes
(urk, grk, vr-ogrk, ahk, vr-oahk) a fixed-T (T=200) lockstep solve of every
(system, rhs) pair (K1) followed by the fused epilogue (K3: F = beta H V,
NMSE vs RZF, Eq. (7) sum-rate).  Inputs are seeded synthetic channels of the
cfg2 model (there is no dataset); realizations are sharded across ranks
(weak scaling, no data-path collective; the per-system NMSE / sum-rate
statistics are gathered at the end).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Kaczmarz precoder solves/s"
UNIT = "precoders/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--batch", type=int, default=0, help="realizations per rank (default: the config's)")
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--schemes", default="")
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c128", action="store_true", help="skip the complex128 oracle-mode step")
    return ap.parse_args()


# --------------------------------------------------------------------------- CPU reference leg

def _cpu_task(args):
    """One (scheme, realization) precoder with the oracle port: RZF + solve + assembly + metrics."""
    cfg_name, seed, scheme, iters = args
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        import oracle as O
        from paper_2501_10689_b200.channel import CONFIGS, generate, solver_seed_sequence
        cfg = CONFIGS[cfg_name]
        ch = generate(cfg, [seed])
        nt, k = ch.n_antennas, ch.n_users
        vrs = tuple(O.contiguous_region(int(ch.start[0, i]), int(ch.length[0, i]), nt) for i in range(k))
        chan = O.ChannelMatrix(h=ch.dense(0), vrs=vrs, cfg=O.ArrayConfig(nt, cfg.carrier_freq, nt))
        reg = float(ch.reg[0])
        sys_ = O.AugmentedSystem.from_channel(chan, reg)  # preprocessing, untimed (as the GPU batch build)
        t0 = time.perf_counter()
        ref = O.rzf_precoder(chan, reg)
        run = O.run_precoding(scheme, sys_, ref, epsilon=0.0, max_iters=iters,
                              rng=np.random.default_rng(solver_seed_sequence(seed)))
        O.nmse(run.precoder.f, ref.f)
        O.spectral_efficiency(chan.h, run.precoder.f, float(ch.snr_linear[0]))
        return time.perf_counter() - t0


def cpu_reference_steps(cfg_name, schemes, iters, steps, warmup, cores):
    """Each step: R = max(1, cores // len(schemes)) realizations x all schemes, in parallel
    on `cores` worker processes.  Returns (per-step wall times, precoders per step)."""
    import multiprocessing as mp
    r = max(1, cores // len(schemes))
    ctx = mp.get_context("fork")
    walls = []
    with ctx.Pool(processes=min(cores, r * len(schemes))) as pool:
        for s in range(warmup + steps):
            tasks = [(cfg_name, 10_000 + s * r + j, sc, iters) for j in range(r) for sc in schemes]
            t0 = time.perf_counter()
            pool.map(_cpu_task, tasks, chunksize=1)
            if s >= warmup:
                walls.append(time.perf_counter() - t0)
    return walls, r * len(schemes), r


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:  # pragma: no cover
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------------- algorithmic bytes

def h_elems_per_launch(host, scheme, iters):
    """H_eff elements the algorithm streams per rhs-iteration
    (sum over R_t of |Gamma_i| plus the projected row), summed over every
    (system, rhs) of one launch of T iterations.  Bytes = elems * sizeof(complex);
    real flops = 8 * elems (one complex MAC per streamed element)."""
    sup = host.support_sizes().astype(np.float64)        # (B, K)
    b, k = sup.shape
    tot_rows = sup.sum(axis=1)                            # sum_i |Gamma_i| per system
    mean_row = sup.mean(axis=1)
    if scheme in ("grk", "gk"):
        per = tot_rows + mean_row
    elif scheme in ("urk", "swor-erk"):
        per = 2 * mean_row
    elif scheme == "vr-ogrk":
        xs = np.zeros(b)
        for s in range(b):
            cp = host.coupled_ptr[s * k:(s + 1) * k + 1]
            idx = host.coupled_idx
            xs[s] = np.mean([sup[s, idx[cp[i]:cp[i + 1]]].sum() for i in range(k)])
        per = xs + mean_row
    else:  # ahk, vr-oahk: refresh + aggregation over every row
        per = 2 * tot_rows
    return float(iters * k * per.sum())


MICRO = os.path.join(ROOT, "profiles", "r01_microbench.json")


def measured_fp32_peak():
    """FP32 FFMA peak (TFLOP/s) from tools/microbench.cu as committed under profiles/."""
    try:
        with open(MICRO) as fh:
            for line in fh:
                d = json.loads(line)
                if d.get("probe") == "FFMA":
                    return float(d["chip_TFLOPs_fp32"]), "measured (tools/microbench.cu, profiles/r01_microbench.json)"
    except (OSError, ValueError):
        pass
    return 2 * 148 * 128 * 1.965e9 / 1e12, "nominal 148 SM x 128 FFMA/clk x 1.965 GHz"


def measured_fp32_reg3_peak():
    """FP32 FFMA rate when every FMA reads three registers (the kernels' form), tools/fma_forms.cu."""
    try:
        with open(MICRO) as fh:
            for line in fh:
                d = json.loads(line)
                if d.get("probe") == "FFMA reg3":
                    return float(d["chip_TFLOPs_fp32"])
    except (OSError, ValueError):
        pass
    return None


def measured_smem_peak():
    try:
        with open(MICRO) as fh:
            for line in fh:
                d = json.loads(line)
                if d.get("probe") == "LDS.128 distinct":
                    return float(d["chip_TBps"]) * 1e3
    except (OSError, ValueError):
        pass
    return 148 * 128 * 1.965e9 / 1e9


# --------------------------------------------------------------------------- main

def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2501_10689_b200.channel import CONFIGS
    cfg = CONFIGS[a.config]
    schemes = [s for s in a.schemes.split(",") if s] or list(cfg.schemes)
    iters = a.iters or cfg.n_iters
    B = a.batch or cfg.n_systems
    workload = (f"{a.config}: Nt={cfg.n_antennas} K={cfg.n_users} VR={cfg.vr_len[0]}"
                f"{'' if cfg.vr_len[0] == cfg.vr_len[1] else '-' + str(cfg.vr_len[1])}, "
                f"{len(schemes)} schemes ({','.join(schemes)}) x {B} realizations/rank, T={iters}, "
                "RZF + solve + F/NMSE/sum-rate epilogue")

    if a.impl == "reference":
        if rank != 0:
            return
        cores = host_cores()
        walls, per_step, r = cpu_reference_steps(a.config, schemes, iters, a.steps, a.warmup, cores)
        t = float(np.mean(walls))
        val = per_step / t
        line = {"metric": METRIC, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": a.gpus,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
                "config": {"workload": workload, "sample_per_step": f"{r} realizations x {len(schemes)} schemes",
                           "parallelism": f"process pool x{min(cores, per_step)}"},
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": min(cores, per_step), "kind": "port",
                                 "sample": f"{r} realizations x {len(schemes)} schemes per step, T={iters}, "
                                           "oracle/ numpy port of kaczprec (reference not installable on the box)"},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    # CPU baseline before any CUDA initialisation (fork-safe), rank 0 at N=1 only
    cpu_baseline = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cores = host_cores()
        walls, per_step, r = cpu_reference_steps(a.config, schemes, iters, 1, 0, cores)
        cpu_baseline = {"value": per_step / walls[0], "unit": UNIT, "cores": min(cores, per_step), "kind": "port",
                        "sample": f"{r} realization(s) x {len(schemes)} schemes (T={iters}, RZF+solve+assembly+"
                                  "metrics) with the oracle/ numpy port, one process per precoder"}

    import torch
    import torch.distributed as dist
    import paper_2501_10689_b200 as kz
    from paper_2501_10689_b200 import _lib

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev_id = torch.device("cuda", local)
    lo, hi = kz.shard_range(B * world, rank, world)  # weak scaling: B realizations per rank
    seeds = range(lo, hi)
    ch = kz.generate(cfg, seeds)
    host = kz.HostBatch.from_contiguous(ch)
    dev = host.to_device(a.dtype, device=dev_id)
    csize = 16 if a.dtype == "c128" else 8
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev_id)
    ws = torch.empty(_lib.lib().kz_solve_workspace_bytes(
        __import__("ctypes").byref(dev.problem), None), dtype=torch.uint8, device=dev_id)

    def step(d, seed, per_scheme_ms=None, collect=None):
        n_launch = 0
        rz = kz.rzf_batched(d)
        n_launch += rz["launches"]
        ews, gram = None, False  # the five epilogues of a step share H, so the Gram G0 is formed once
        for sc in schemes:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = kz.solve_batch(d, sc, mode="lockstep", max_iters=iters,
                                 rng=("philox", seed * 7919 + 17) if sc in kz.STOCHASTIC_SCHEMES else None,
                                 workspace=ws)
            e1.record(stream)
            ep = kz.epilogue(d, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True, workspace=ews,
                             gram_cached=gram)
            ews, gram = ep["workspace"], ep["gram_form"]
            n_launch += res.launches + ep["launches"]
            if per_scheme_ms is not None:
                per_scheme_ms.setdefault(sc, []).append((e0, e1))
            if collect is not None:
                collect[sc] = (res.v, ep["nmse"], ep["sum_rate"])
        return n_launch

    for w in range(a.warmup):
        step(dev, w)
    torch.cuda.synchronize()

    per_scheme = {}
    launches = 0
    step_ms = []
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for s in range(a.steps):
            flush.fill_(s & 0xFF)  # L2 flush (256 MiB write), outside the timed events
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launches += step(dev, 1000 + s, per_scheme)
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    t_rank = float(np.sum(step_ms)) / 1e3
    t = torch.tensor([t_rank], dtype=torch.float64, device=dev_id)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    ms_per_step = 1e3 * t_max / a.steps
    precoders = len(schemes) * B * world * a.steps
    value = precoders / t_max
    rhs_iters = len(schemes) * B * world * cfg.n_users * iters * a.steps / t_max

    # dominant kernel: the scheme solve with the largest launch time
    avg = {sc: float(np.mean([x.elapsed_time(y) for x, y in ev])) for sc, ev in per_scheme.items()}
    dom = max(avg, key=avg.get)
    elems_dom = h_elems_per_launch(host, dom, iters)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    fp32_peak, fp32_src = measured_fp32_peak()
    reg3_peak = measured_fp32_reg3_peak()
    smem_peak = measured_smem_peak()
    smem_ncu = None  # shared-memory bytes the dominant launch moves, from ncu counters (profiles/r01_ncu_smem.json)
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_smem.json")) as fh:
            rec = json.load(fh).get(dom)
        if rec and a.dtype == "c64" and cfg.name == "cfg2":
            sb = rec["shared_bytes_per_iteration"] * iters * B / rec["B"]
            smem_ncu = {"bytes_per_launch": sb, "achieved_GBps": sb / (avg[dom] / 1e3) / 1e9, "peak_GBps": smem_peak,
                        "frac": sb / (avg[dom] / 1e3) / 1e9 / smem_peak if smem_peak else None,
                        "ncu_pct_of_peak_sustained": rec["pct_of_peak_sustained_elapsed"],
                        "source": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum x 128 B of the ncu --set full capture "
                                  f"({rec['capture']}, B={rec['B']}, T={rec['T']}), scaled to this launch's T and B"}
    except (OSError, ValueError, KeyError):
        pass
    t_dom = avg[dom] / 1e3
    tflops = 8.0 * elems_dom / t_dom / 1e12
    bytes_dom = csize * elems_dom
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(dom)
    except (OSError, ValueError):
        pass
    # end to end through the public API: pinned host inputs in, per-system results out.
    # Every step copies its inputs H2D (kz.DeviceBatch from pinned host tensors), runs RZF + 5 x (solve +
    # epilogue) and reads each scheme's V, NMSE and sum-rate back into pinned host buffers.  As a serving loop
    # would, the upload of step s+1 runs on an upload stream while step s computes, and the D2H of scheme k
    # overlaps the solve of scheme k+1 on a copy stream; the timed region spans all n steps (first upload to
    # last read-back) and is divided by n.
    e2e = None
    if not a.no_e2e:
        pinned = kz.pin_host(host, a.dtype)
        copy_stream = torch.cuda.Stream(device=dev_id)
        up_stream = torch.cuda.Stream(device=dev_id)
        outs_h = {sc: (torch.empty((B, cfg.n_users, cfg.n_users), dtype=dev.complex_dtype).pin_memory(),
                       torch.empty(B, dtype=torch.float64).pin_memory(),
                       torch.empty(B, dtype=torch.float64).pin_memory()) for sc in schemes}
        h2d = sum(t.numel() * t.element_size() for t in pinned.values())
        d2h = sum(sum(t.numel() * t.element_size() for t in o) for o in outs_h.values())

        def upload():
            with torch.cuda.stream(up_stream):
                d = kz.DeviceBatch(host, a.dtype, device=dev_id, pinned=pinned)
                ev = torch.cuda.Event()
                ev.record(up_stream)
            for t in d.t.values():
                t.record_stream(stream)  # consumed on the compute stream
            return d, ev

        def e2e_step(d, ev, s):
            stream.wait_event(ev)
            rz = kz.rzf_batched(d)
            ews, gram = None, False
            for sc in schemes:
                res = kz.solve_batch(d, sc, mode="lockstep", max_iters=iters,
                                     rng=("philox", s * 104729 + 5) if sc in kz.STOCHASTIC_SCHEMES else None,
                                     workspace=ws)
                ep = kz.epilogue(d, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True, workspace=ews,
                                 gram_cached=gram)
                ews, gram = ep["workspace"], ep["gram_form"]
                done_ev = torch.cuda.Event()
                done_ev.record(stream)
                copy_stream.wait_event(done_ev)
                with torch.cuda.stream(copy_stream):
                    for src, dst in zip((res.v, ep["nmse"], ep["sum_rate"]), outs_h[sc]):
                        src.record_stream(copy_stream)
                        dst.copy_(src, non_blocking=True)

        e2e_step(*upload(), 0)  # untimed warm-up (allocator, pinned staging, streams)
        stream.wait_stream(copy_stream)
        torch.cuda.synchronize()
        n_e2e = max(1, min(a.steps, 5))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk_e2e:
            e0.record(stream)
            up_stream.wait_stream(stream)  # the first upload starts inside the timed region
            nxt = upload()
            for s in range(1, n_e2e + 1):
                cur = nxt
                if s < n_e2e:
                    nxt = upload()  # next step's inputs stream in while this step computes
                e2e_step(cur[0], cur[1], s)
                del cur
            stream.wait_stream(copy_stream)
            e1.record(stream)
            torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / n_e2e], dtype=torch.float64, device=dev_id)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": len(schemes) * B * world / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": float(te.item()),
               "steps": n_e2e, "clocks": clk_e2e.summary(),
               "path": "kz.DeviceBatch(pinned, upload stream, one step ahead) -> rzf_batched -> solve_batch + "
                       "epilogue per scheme -> V/NMSE/sum-rate to pinned host (copy stream)"}

    # final gather of per-system statistics (the only cross-GPU step)
    col = {}
    step(dev, 99, collect=col)
    stats = {}
    for sc in schemes:
        g = kz.gather_stats({"nmse": col[sc][1], "sum_rate": col[sc][2]}, B * world)
        stats[sc] = {"median_nmse": float(g["nmse"].median()), "mean_sum_rate": float(g["sum_rate"].mean()),
                     "systems": int(g["nmse"].numel())}

    # the same step in complex128 oracle mode (BASELINE cfg2 quotes both modes): one warm + one timed step
    c128 = None
    if not a.no_c128 and a.dtype == "c64":
        dev128 = host.to_device("c128", device=dev_id)
        step(dev128, 7)
        torch.cuda.synchronize()
        ev128 = {}
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(dev128, 8, ev128)
        e1.record(stream)
        torch.cuda.synchronize()
        t128 = e0.elapsed_time(e1)
        c128 = {"value": len(schemes) * B * world / (t128 / 1e3), "unit": UNIT, "ms_per_step": t128,
                "dtype": "complex128",
                "per_scheme_launch_ms": {sc: ev[0][0].elapsed_time(ev[0][1]) for sc, ev in ev128.items()},
                "note": "one timed step, same workload; the exact-arithmetic kernels of the oracle-mode parity tests"}
        del dev128

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "complex64" if a.dtype == "c64" else "complex128",
            "data": "synthetic (seeded cfg model: LoS spherical wavefront, contiguous VR, unit-norm columns)",
            "config": {"workload": workload, "global_batch": B * world, "realizations_per_rank": B,
                       "l2": "flushed between timed steps (256 MiB write outside the events)",
                       "rng": "on-device Philox4x32-10 row draws", "parallelism": f"realizations sharded x{world}"},
            "rhs_iterations_per_s": rhs_iters,
            "per_scheme_launch_ms": avg,
            "roofline": {"kernel": f"kz_solve[{dom}]", "bound": "fp32-fma", "achieved": tflops,
                         "peak": fp32_peak, "unit": "TFLOP/s", "frac": tflops / fp32_peak, "traffic": traffic,
                         "algorithmic_flops_per_launch": 8.0 * elems_dom, "peak_source": fp32_src,
                         "note": "H_eff is shared-memory resident and each streamed h element is reused by "
                                 "2 rhs in registers (8 FFMA per complex element), so the launch is CUDA-core "
                                 "FMA bound (SURVEY 8(d): report the FMA roofline); flops = 8 x streamed H_eff "
                                 "elements per rhs-iteration",
                         "ffma_3reg_view": ({"peak_TFLOPs": reg3_peak, "frac": tflops / reg3_peak,
                                             "peak_source": "tools/fma_forms.cu (profiles/r01_microbench.json): "
                                                            "FFMA with three register operands issues at 0.81/clk "
                                                            "per SMSP vs 0.97 for the immediate form"}
                                            if reg3_peak else None),
                         "smem_view": {"algorithmic_GBps": bytes_dom / t_dom / 1e9, "peak_GBps": smem_peak},
                         "smem_ncu": smem_ncu,
                         "hbm_view": {"algorithmic_GBps": bytes_dom / t_dom / 1e9, "peak_GBps": hbm_peak,
                                      "peak_source": "MEASURED_PEAKS.json hbm_gbs"}},
            "cpu_baseline": cpu_baseline, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "stats": stats, "complex128_oracle_mode": c128,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
