"""Benchmark of the batched Kaczmarz precoding hot path.

Headline (BASELINE.json configs[1] = cfg2, the config the metric is quoted on): one step = one full pass of the
cfg2 workload over this rank's realizations: the direct RZF reference (K2), then for each of the five cfg2
schemes (urk, grk, vr-ogrk, ahk, vr-oahk) a fixed-T (T=200) lockstep solve of every (system, rhs) pair (K1)
followed by the fused epilogue (K3: F = beta H V, NMSE vs RZF, Eq. (7) sum-rate).  Inputs are seeded synthetic
channels of the cfg model (there is no dataset); realizations are sharded across ranks (weak scaling, no
data-path collective; the per-system NMSE / sum-rate statistics are gathered at the end).

Sub-records on the N=1 line (rank 0, one GPU), each with its own warm-up, device-timed steps, clocks, roofline
and end-to-end figure:
  complex128_oracle_mode  the same cfg2 step with the exact-arithmetic (oracle-mode) kernels
  configs.cfg3            BASELINE configs[2]: Nt=1024, K=128, VR ~ U[128,512], VR-OAHK T=200, B=4096, c64
  configs.cfg4            BASELINE configs[3]: Nt=4096, K=256, VR=512, GRK + VR-OAHK to residual 1e-4
                          (solve_all semantics), B=16384 (the largest single-GPU config), c64
  configs.cfg3_grouped    cfg3's own variant: 4 orthogonal row groups, <= 8 hyperplanes per aggregated step
  configs.cfg2_nmse_stop  the reference's default run_precoding(epsilon=1e-6) on the cfg2 workload (NMSE stop
                          against RZF on the on-chip kernels, cap 10^4 K)
  configs.cfg5_T{10,20,50,100}  BASELINE configs[4]: wideband, 1024 subcarriers, AHK + VR-OAHK per T of the sweep
Every config record carries per_scheme_views: each scheme's solve time against the FP32-FMA roofline (algorithmic
flops) and the HBM roofline (compulsory bytes: H_eff once + V).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  python bench.py --config cfg4 --scaling strong     (torchrun: 16384 realizations split over the ranks)

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
NOMINAL_FP32_TFLOPS = 2 * 148 * 128 * 1.965e9 / 1e12  # 148 SMs x 128 FP32 lanes x 2 flops x max SM clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: --batch (default: the config's B) realizations per rank; strong: the config's B "
                         "split over the ranks")
    ap.add_argument("--batch", type=int, default=0, help="realizations per rank (weak) or in total (strong)")
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--schemes", default="")
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c128", action="store_true", help="skip the complex128 oracle-mode record")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg3 / cfg4 records")
    ap.add_argument("--config-steps", type=int, default=1, help="timed steps of the cfg3 / cfg4 records")
    return ap.parse_args()


# --------------------------------------------------------------------------- CPU reference leg

REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baseline", "_ref")


def reference_kind() -> str:
    """"reference" when the unmodified kaczprec package is installed in baseline/_ref (python -m pip install
    --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>; git-ignored, it
    travels to the GPU box with the snapshot), else "port" (oracle/, pinned bitwise to the reference)."""
    return "reference" if os.path.isdir(os.path.join(REF_DIR, "kaczprec")) else "port"


def _cpu_task(args):
    """One (scheme, realization) precoder on the CPU: RZF + solve + assembly + metrics, with the reference's own
    kaczprec (kind "reference") or the oracle port (kind "port"), through the same public calls."""
    cfg_name, seed, scheme, iters, kind = args
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        if kind == "reference":
            if REF_DIR not in sys.path:
                sys.path.insert(0, REF_DIR)
            import kaczprec.assembly as KA
            import kaczprec.channel as KC
            import kaczprec.metrics as KM
            import kaczprec.rzf as KR
            import kaczprec.solvers as KS

            def region(s, ln, nt):
                return KC.VisibilityRegion(frozenset(range(s, s + ln)), nt, 1)
            ArrayConfig, ChannelMatrix, AugmentedSystem = KC.ArrayConfig, KC.ChannelMatrix, KS.AugmentedSystem
            rzf_precoder, run_precoding, nmse, rate = KR.rzf_precoder, KS.run_precoding, KM.nmse, \
                KM.spectral_efficiency
            del KA
        else:
            import oracle as O
            region, ArrayConfig, ChannelMatrix, AugmentedSystem = (O.contiguous_region, O.ArrayConfig,
                                                                    O.ChannelMatrix, O.AugmentedSystem)
            rzf_precoder, run_precoding, nmse, rate = O.rzf_precoder, O.run_precoding, O.nmse, O.spectral_efficiency
        from paper_2501_10689_b200.channel import CONFIGS, generate, solver_seed_sequence
        cfg = CONFIGS[cfg_name]
        ch = generate(cfg, [seed])
        nt, k = ch.n_antennas, ch.n_users
        vrs = tuple(region(int(ch.start[0, i]), int(ch.length[0, i]), nt) for i in range(k))
        chan = ChannelMatrix(h=ch.dense(0), vrs=vrs, cfg=ArrayConfig(nt, cfg.carrier_freq, nt))
        reg = float(ch.reg[0])
        sys_ = AugmentedSystem.from_channel(chan, reg)  # preprocessing, untimed (as the GPU batch build)
        t0 = time.perf_counter()
        ref = rzf_precoder(chan, reg)
        run = run_precoding(scheme, sys_, ref, epsilon=0.0, max_iters=iters,
                            rng=np.random.default_rng(solver_seed_sequence(seed)))
        nmse(run.precoder.f, ref.f)
        rate(chan.h, run.precoder.f, float(ch.snr_linear[0]))
        return time.perf_counter() - t0


def cpu_reference_steps(cfg_name, schemes, iters, steps, warmup, cores):
    """Each step: R = max(1, cores // len(schemes)) realizations x all schemes, in parallel
    on `cores` worker processes.  Returns (per-step wall times, precoders per step)."""
    import multiprocessing as mp
    r = max(1, cores // len(schemes))
    kind = reference_kind()
    ctx = mp.get_context("fork")
    walls = []
    with ctx.Pool(processes=min(cores, r * len(schemes))) as pool:
        for s in range(warmup + steps):
            tasks = [(cfg_name, 10_000 + s * r + j, sc, iters, kind) for j in range(r) for sc in schemes]
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


# --------------------------------------------------------------------------- algorithmic work

def elems_per_rhs_iter(sup, scheme, coupled=None):
    """H_eff elements the algorithm streams per rhs-iteration, per system (B,): the refreshed rows R_t plus the
    projected row; real flops = 8 x elements (one complex MAC each), bytes = c x elements.
    sup: (B, K) support sizes; coupled: (ptr, idx) of the VR-OGRK coupled sets."""
    sup = sup.astype(np.float64)
    b, k = sup.shape
    tot_rows = sup.sum(axis=1)
    mean_row = sup.mean(axis=1)
    if scheme in ("grk", "gk"):
        return tot_rows + mean_row
    if scheme in ("urk", "swor-erk"):
        return 2 * mean_row
    if scheme == "vr-ogrk":
        ptr, idx = coupled
        xs = np.zeros(b)
        for s in range(b):
            cp = ptr[s * k:(s + 1) * k + 1]
            xs[s] = np.mean([sup[s, idx[cp[i]:cp[i + 1]]].sum() for i in range(k)])
        return xs + mean_row
    return 2 * tot_rows  # ahk, vr-oahk: refresh + aggregation over every row


MICRO = os.path.join(ROOT, "profiles", "r02_microbench.json")


def _micro(probe, key):
    try:
        with open(MICRO) as fh:
            for line in fh:
                d = json.loads(line)
                if d.get("probe") == probe:
                    return d
    except (OSError, ValueError):
        pass
    return None


def fp32_peak():
    """Roofline denominator: the nominal FP32 FMA peak at the maximum SM clock (148 SMs x 128 lanes x 2 flops
    x 1.965 GHz = 74.4 TFLOP/s); the measured FFMA rates (tools/microbench.cu, with their clocks) are views."""
    return NOMINAL_FP32_TFLOPS, "nominal: 148 SM x 128 FP32 lanes x 2 flops x 1.965 GHz (max SM clock)"


def smem_peak_gbps():
    d = _micro("LDS.128", None)
    return float(d["bytes_per_s"]) / 1e9 if d and "bytes_per_s" in d else 148 * 128 * 1.965


def measured_views():
    out = {}
    for probe in ("FFMA imm", "FFMA reg3", "LDS.128"):
        d = _micro(probe, None)
        if d:
            out[probe] = {k: d[k] for k in d if k != "probe"}
    return out or None


def reg_ffma_stream_view(achieved_tflops):
    """The dominant launch against the rate the refresh inner loop reaches in isolation (tools/refresh_forms.cu,
    profiles/r02_refresh_forms.json, form A = the kernel's 2 rhs x 16 antennas blocking; the FFMAs alone, form E,
    run at the same rate: register-operand FFMA streams stop at ~0.65 warp-instructions/clk per SM sub-partition
    on this B200, whatever the shared-memory traffic)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_refresh_forms.json")) as fh:
            for line in fh:
                d = json.loads(line)
                if d.get("form", "").startswith("A:"):
                    rate = float(d["ffma_per_clk_per_smsp"])
                    peak = NOMINAL_FP32_TFLOPS * rate
                    return {"ffma_per_clk_per_smsp": rate, "peak_TFLOPs": peak, "frac": achieved_tflops / peak,
                            "peak_source": "profiles/r02_refresh_forms.json form A x the nominal FP32 peak"}
    except (OSError, ValueError, KeyError):
        pass
    return None


def peaks_json():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


# --------------------------------------------------------------------------- workloads

class Workload:
    """One config's step on this rank's systems: inputs resident in HBM, per step RZF + per scheme (solve +
    epilogue), chunked over `chunk` systems (bounded per-call outputs / workspaces)."""

    def __init__(self, cfg, schemes, dtype, lo, hi, dev_id, chunk=0, device_inputs=False, orth_groups=1, agg_cap=0,
                 nmse_eps=0.0):
        import paper_2501_10689_b200 as kz
        self.kz, self.cfg, self.schemes, self.dtype = kz, cfg, schemes, dtype
        self.nmse_eps = nmse_eps  # > 0: run_precoding's NMSE stop against the RZF precoder (cap = the config's T)
        self.lo, self.hi, self.B = lo, hi, hi - lo
        self.dev_id = dev_id
        self.tol = cfg.extra.get("residual_tol")
        self.iters = cfg.n_iters
        # one drop per realization; a wideband config (cfg5) is one drop whose subcarriers are the systems
        seeds = [0, range(lo, hi)] if cfg.n_subcarriers > 1 else range(lo, hi)
        if device_inputs:  # drops -> channel entries + VR partition on the device
            self.host = None
            self.dev = kz.DeviceBatch.from_drops(kz.generate_drops(cfg, seeds), dtype=dtype, device=dev_id)
        else:
            self.host = kz.HostBatch.from_contiguous(kz.generate(cfg, seeds), orth_groups=orth_groups, agg_cap=agg_cap)
            self.dev = self.host.to_device(dtype, device=dev_id)
        self.chunk = chunk if 0 < chunk < self.B else self.B
        self.sup = (self.dev.t["seg_len"].cpu().numpy().reshape(self.B, cfg.n_users))
        self.ws = {}
        self.tma = {}  # per scheme: H_eff staged by TMA tensor copies in the last solve (kz_last_tma_staging)

    def coupled(self):
        if self.host is not None:
            return self.host.coupled_ptr, self.host.coupled_idx
        return self.dev.t["coupled_ptr"].cpu().numpy(), self.dev.t["coupled_idx"].cpu().numpy()

    def rng(self, sc, seed):
        return ("philox", seed) if sc in self.kz.STOCHASTIC_SCHEMES else None

    def step(self, dev, seed, events=None, collect=None, out_host=None, copy_stream=None, stream=None):
        """One step over `dev` (this workload's batch or an uploaded copy).  events[sc] gets the (start, end) of
        the scheme's solve launches; collect[sc] the per-system (V, NMSE, sum-rate, iters) of the last chunk
        set; out_host: pinned host buffers the results are copied into on copy_stream."""
        import torch
        kz = self.kz
        launches = 0
        k = self.cfg.n_users
        for lo in range(0, self.B, self.chunk):
            hi = min(self.B, lo + self.chunk)
            sub = dev.view(lo, hi) if (lo, hi) != (0, self.B) else dev
            rz = kz.rzf_batched(sub, want_f=self.nmse_eps > 0)
            launches += rz["launches"]
            ews, gram = None, False  # the epilogues of a chunk share H, so the Gram G0 is formed once
            for sc in self.schemes:
                e0, e1 = _events()
                e0.record(stream)
                if self.tol:
                    res = kz.solve_batch(sub, sc, mode="residual", epsilon=self.tol, max_iters=10_000 * k,
                                         rng=self.rng(sc, seed), workspace=self.ws.get(sc),
                                         system_base=self.lo + lo)
                elif self.nmse_eps > 0:
                    res = kz.solve_batch(sub, sc, mode="lockstep", max_iters=self.iters, epsilon=self.nmse_eps,
                                         f_ref=rz["f"], rng=self.rng(sc, seed), workspace=self.ws.get(sc),
                                         system_base=self.lo + lo)
                else:
                    res = kz.solve_batch(sub, sc, mode="lockstep", max_iters=self.iters, rng=self.rng(sc, seed),
                                         workspace=self.ws.get(sc), system_base=self.lo + lo)
                e1.record(stream)
                self.ws[sc] = res.workspace
                self.tma[sc] = res.tma_staging
                ep = kz.epilogue(sub, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True, workspace=ews,
                                 gram_cached=gram)
                ews, gram = ep["workspace"], ep["gram_form"]
                launches += res.launches + ep["launches"]
                if events is not None:
                    events.setdefault(sc, []).append((e0, e1))
                if collect is not None:
                    c = collect.setdefault(sc, {"nmse": [], "sum_rate": [], "iters": []})
                    c["nmse"].append(ep["nmse"])
                    c["sum_rate"].append(ep["sum_rate"])
                    c["iters"].append(res.iters)
                if out_host is not None:
                    done_ev = torch.cuda.Event()
                    done_ev.record(stream)
                    copy_stream.wait_event(done_ev)
                    with torch.cuda.stream(copy_stream):
                        for src, dst in zip((res.v, ep["nmse"], ep["sum_rate"]), out_host[sc]):
                            src.record_stream(copy_stream)
                            dst[lo:hi].copy_(src, non_blocking=True)
        return launches

    def out_buffers(self):
        import torch
        k = self.cfg.n_users
        cdt = torch.complex128 if self.dtype == "c128" else torch.complex64
        return {sc: (torch.empty((self.B, k, k), dtype=cdt).pin_memory(),
                     torch.empty(self.B, dtype=torch.float64).pin_memory(),
                     torch.empty(self.B, dtype=torch.float64).pin_memory()) for sc in self.schemes}

    def elems(self, sc, iters_tensor=None):
        """Algorithmic H elements of one solve launch (all systems)."""
        per = elems_per_rhs_iter(self.sup, sc, self.coupled() if sc == "vr-ogrk" else None)  # (B,)
        if iters_tensor is None:
            return float(per.sum() * self.cfg.n_users * self.iters)
        it = iters_tensor.double().sum(dim=1).cpu().numpy()  # rhs-iterations per system
        return float((per * it).sum())


def timed_steps(wl, steps, warmup, seed0, flush, world, stream, dist):
    """Warm-up, then `steps` device-timed steps (barrier + synchronize on both sides, L2 flushed between
    steps outside the events).  Returns (step ms list, per-scheme events, launches, clocks)."""
    import torch
    for w in range(warmup):
        wl.step(wl.dev, seed0 + w, stream=stream)
    torch.cuda.synchronize()
    per_scheme, launches, step_ms = {}, 0, []
    with ClockSampler(wl.dev_id.index or 0) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for s in range(steps):
            flush.fill_(s & 0xFF)  # L2 flush (256 MiB write), outside the timed events
            e0, e1 = _events()
            e0.record(stream)
            launches += wl.step(wl.dev, seed0 + 1000 + s, events=per_scheme, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    return step_ms, per_scheme, launches, clk.summary()


def e2e_run(wl, n_steps, seed0, stream, dev_id, warm_compute=True):
    """End to end through the public API: pinned host inputs in, per-system V / NMSE / sum-rate out.  Every step
    uploads its inputs (kz.DeviceBatch from pinned host tensors, on an upload stream one step ahead, as a serving
    loop would) and reads each scheme's results back into pinned host buffers on a copy stream; the timed region
    spans all n steps (first upload to last read-back) and is divided by n."""
    import torch
    kz = wl.kz
    pinned = {name: t.cpu().pin_memory() for name, t in wl.dev.t.items() if name in kz.DeviceBatch.FIELDS
              or name == "snr_linear"}
    copy_stream = torch.cuda.Stream(device=dev_id)
    up_stream = torch.cuda.Stream(device=dev_id)
    outs = wl.out_buffers()
    h2d = sum(t.numel() * t.element_size() for t in pinned.values())
    d2h = sum(sum(t.numel() * t.element_size() for t in o) for o in outs.values())
    host = wl.dev.host

    def upload():
        with torch.cuda.stream(up_stream):
            d = kz.DeviceBatch(host, wl.dtype, device=dev_id, pinned=pinned)
            ev = torch.cuda.Event()
            ev.record(up_stream)
        for t in d.t.values():
            t.record_stream(stream)  # consumed on the compute stream
        return d, ev

    def run_step(d, ev, s):
        stream.wait_event(ev)
        wl.step(d, seed0 + s, out_host=outs, copy_stream=copy_stream, stream=stream)

    if warm_compute:
        for _ in range(2):  # untimed warm-up (allocator steady state with one upload in flight, pinned staging, streams)
            run_step(*upload(), 0)
    else:  # the kernels ran already (device-timed steps): warm only the upload allocations
        d, _ = upload()
        torch.cuda.synchronize()
        del d
    stream.wait_stream(copy_stream)
    torch.cuda.synchronize()
    e0, e1 = _events()
    with ClockSampler(dev_id.index or 0) as clk:
        e0.record(stream)
        up_stream.wait_stream(stream)  # the first upload starts inside the timed region
        nxt = upload()
        for s in range(1, n_steps + 1):
            cur = nxt
            if s < n_steps:
                nxt = upload()  # next step's inputs stream in while this step computes
            run_step(cur[0], cur[1], s)
            del cur
        stream.wait_stream(copy_stream)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n_steps
    return {"ms_per_step": ms, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": n_steps,
            "clocks": clk.summary()}


def e2e_drops_run(wl, n_steps, seed0, stream, dev_id):
    """End to end from the user drops, input preparation included: every step draws the realizations' drops on the
    host (channel.generate_drops: positions, angles, VR starts; the seeded streams of the reference model), builds
    the batch on the device (DeviceBatch.from_drops on an upload stream: drop parameters over PCIe, channel
    synthesis + VR partition by kz_channel_synth / kz_partition_*), runs the step and reads V / NMSE / sum-rate back
    to pinned host memory.  The next step's drops are drawn and built while the current step computes (a serving
    loop); the host work sits inside the CUDA-event interval (the first step's preparation is timed in full)."""
    import torch
    kz = wl.kz
    copy_stream = torch.cuda.Stream(device=dev_id)
    up_stream = torch.cuda.Stream(device=dev_id)
    outs = wl.out_buffers()
    d2h = sum(sum(t.numel() * t.element_size() for t in o) for o in outs.values())
    seeds = range(wl.lo, wl.hi)
    h2d = [0]

    def upload():
        drops = kz.generate_drops(wl.cfg, seeds)
        h2d[0] = sum(v.nbytes for v in vars(drops).values() if isinstance(v, np.ndarray))  # drop parameters
        d = kz.DeviceBatch.from_drops(drops, dtype=wl.dtype, device=dev_id, stream=up_stream)
        ev = torch.cuda.Event()
        ev.record(up_stream)
        for t in d.t.values():
            t.record_stream(stream)
        return d, ev

    def run_step(d, ev, s):
        stream.wait_event(ev)
        wl.step(d, seed0 + s, out_host=outs, copy_stream=copy_stream, stream=stream)

    run_step(*upload(), 0)  # untimed warm-up
    stream.wait_stream(copy_stream)
    torch.cuda.synchronize()
    e0, e1 = _events()
    with ClockSampler(dev_id.index or 0) as clk:
        e0.record(stream)
        up_stream.wait_stream(stream)
        nxt = upload()
        for s in range(1, n_steps + 1):
            cur = nxt
            run_step(cur[0], cur[1], s)  # enqueued; the next step's drops are prepared meanwhile
            if s < n_steps:
                nxt = upload()
            del cur
        stream.wait_stream(copy_stream)
        e1.record(stream)
        torch.cuda.synchronize()
    return {"ms_per_step": e0.elapsed_time(e1) / n_steps, "h2d_bytes_per_step": int(h2d[0]),
            "d2h_bytes_per_step": int(d2h), "steps": n_steps, "clocks": clk.summary(),
            "path": "channel.generate_drops (host) -> DeviceBatch.from_drops (upload stream: kz_channel_synth + "
                    "kz_partition, one step ahead) -> rzf_batched -> solve_batch + epilogue per scheme -> "
                    "V/NMSE/sum-rate to pinned host (copy stream)"}


def roofline(wl, per_scheme, iters_by_scheme=None):
    """Dominant launch (largest mean solve time) against the FP32 FMA peak: achieved = algorithmic flops
    (8 x H elements the algorithm streams) / mean launch time (CUDA events on the launch stream)."""
    avg = {sc: float(np.mean([a.elapsed_time(b) for a, b in ev])) for sc, ev in per_scheme.items()}
    dom = max(avg, key=avg.get)
    n_launch_per_step = max(1, -(-wl.B // wl.chunk))
    it = iters_by_scheme.get(dom) if iters_by_scheme else None
    el = wl.elems(dom, it) / n_launch_per_step  # per launch (chunks are equal-sized but the last)
    t = avg[dom] / 1e3
    tflops = 8.0 * el / t / 1e12
    peak, src = fp32_peak()
    csize = 16 if wl.dtype == "c128" else 8
    return dom, avg, {"kernel": f"kz_solve[{dom}]", "bound": "fp32-fma", "achieved": tflops, "peak": peak,
                      "unit": "TFLOP/s", "frac": tflops / peak, "peak_source": src,
                      "algorithmic_flops_per_launch": 8.0 * el, "launch_ms": avg[dom],
                      # the north_star's "SMEM roofline when H is resident": algorithmic bytes (each streamed h
                      # element counted once per rhs) over the measured LDS.128 rate; physically each
                      # loaded element feeds two rhs, which is why the FMA view above is the binding one
                      "smem_view": {"algorithmic_GBps": csize * el / t / 1e9, "peak_GBps": smem_peak_gbps(),
                                    "frac": csize * el / t / 1e9 / smem_peak_gbps(),
                                    "peak_source": "profiles/r02_microbench.json LDS.128 (event-timed, full chip)"},
                      "hbm_view": {"algorithmic_GBps": csize * el / t / 1e9,
                                   "peak_GBps": float(peaks_json().get("hbm_gbs", 6550.7)),
                                   "peak_source": "MEASURED_PEAKS.json hbm_gbs"}}


def scheme_views(wl, per_scheme, iters_by_scheme, steps):
    """Every scheme's solve launches per step against both rooflines: FP32 FMA (algorithmic flops) and HBM
    (compulsory bytes: H_eff read once per launch + V written), so a launch that is staging-bound (few
    iterations per rhs, e.g. cfg4 VR-OAHK at ~2.4) is read against the bound that applies to it."""
    peak, _ = fp32_peak()
    hbm = float(peaks_json().get("hbm_gbs", 6550.7))
    csize = 16 if wl.dtype == "c128" else 8
    h_bytes = float(wl.sup.sum()) * csize
    v_bytes = float(wl.B) * wl.cfg.n_users ** 2 * csize
    out = {}
    for sc, ev in per_scheme.items():
        t = float(np.sum([a.elapsed_time(b) for a, b in ev])) / steps / 1e3
        fl = 8.0 * wl.elems(sc, iters_by_scheme.get(sc))
        out[sc] = {"solve_s_per_step": t, "fma_TFLOPs": fl / t / 1e12, "fma_frac": fl / t / 1e12 / peak,
                   "hbm_compulsory_GBps": (h_bytes + v_bytes) / t / 1e9,
                   "hbm_frac": (h_bytes + v_bytes) / t / 1e9 / hbm}
    return out


def config_record(name, dev_id, stream, flush, steps, warmup, dtype="c64", do_e2e=True, chunk=4096, n_systems=0,
                  schemes=None, orth_groups=1, agg_cap=0, iters=0, nmse_eps=0.0):
    """A BASELINE config other than the headline at its stated size on this GPU (N=1 sub-record); iters > 0
    overrides the config's T (cfg5's iteration-count sweep)."""
    import torch
    import paper_2501_10689_b200 as kz
    cfg = kz.CONFIGS[name]
    if iters:
        cfg = type(cfg)(**{**cfg.__dict__, "n_iters": iters})
    schemes = list(schemes or cfg.schemes)
    B = n_systems or cfg.n_systems
    t0 = time.perf_counter()
    grouped = orth_groups > 1 or agg_cap > 0
    wl = Workload(cfg, schemes, dtype, 0, B, dev_id, chunk=chunk, device_inputs=not grouped,
                  orth_groups=orth_groups, agg_cap=agg_cap, nmse_eps=nmse_eps)
    torch.cuda.synchronize()
    prep_s = time.perf_counter() - t0
    # warm-up on one chunk (kernel / allocator init), then full device-timed steps
    warm = Workload.__new__(Workload)
    warm.__dict__.update(wl.__dict__)
    warm.B = min(wl.B, wl.chunk)
    for w in range(max(1, warmup)):
        warm.step(wl.dev.view(0, warm.B), 11 + w, stream=stream)
    torch.cuda.synchronize()
    per_scheme, step_ms, collect = {}, [], {}
    with ClockSampler(dev_id.index or 0) as clk:
        for s in range(steps):
            flush.fill_(s & 0xFF)
            e0, e1 = _events()
            e0.record(stream)
            n_launch = wl.step(wl.dev, 2000 + s, events=per_scheme, collect=collect if s == steps - 1 else None,
                               stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    iters = {sc: torch.cat(c["iters"]) for sc, c in collect.items()}
    dom, avg, roof = roofline(wl, {sc: ev for sc, ev in per_scheme.items()}, iters)
    # per-launch mean over the chunks: report per-step totals per scheme
    per_step_solve = {sc: float(np.sum([a.elapsed_time(b) for a, b in ev])) / steps for sc, ev in per_scheme.items()}
    ms = float(np.mean(step_ms))
    rec = {"workload": (f"{name}: Nt={cfg.n_antennas} K={cfg.n_users} VR={cfg.vr_len[0]}"
                        f"{'' if cfg.vr_len[0] == cfg.vr_len[1] else '-' + str(cfg.vr_len[1])}, "
                        f"{','.join(schemes)} x {wl.B} realizations, "
                        + (f"{orth_groups} orthogonal groups, <= {agg_cap} hyperplanes per aggregated step, "
                           if grouped else "")
                        + (f"residual tolerance {wl.tol} (solve_all semantics)" if wl.tol else
                           f"run_precoding NMSE stop at {nmse_eps:g} vs RZF (cap {cfg.n_iters})" if nmse_eps else
                           f"T={cfg.n_iters}")
                        + ", RZF + solve + F/NMSE/sum-rate epilogue"),
           "value": len(schemes) * wl.B / (ms / 1e3), "unit": UNIT, "dtype": "complex64" if dtype == "c64"
           else "complex128", "steps": steps, "warmup": f"{max(1, warmup)} step(s) on the first {warm.B} systems",
           "ms_per_step": ms, "chunk_systems": wl.chunk, "solve_ms_per_step": per_step_solve,
           "mean_iters_per_rhs": {sc: float(t.double().mean()) for sc, t in iters.items()},
           "median_nmse": {sc: float(torch.cat(c["nmse"]).median()) for sc, c in collect.items()},
           "mean_sum_rate": {sc: float(torch.cat(c["sum_rate"]).mean()) for sc, c in collect.items()},
           "rhs_iterations_per_s": float(sum(float(t.double().sum()) for t in iters.values()) / (ms / 1e3)),
           "roofline": roof, "per_scheme_views": scheme_views(wl, per_scheme, iters, steps),
           "clocks": clk.summary(),
           "inputs": ("host packing (HostBatch.from_contiguous with the orthogonal groups)" if grouped else
                      "seeded drops -> kz_channel_synth / kz_partition on the device")
           + f" ({prep_s:.1f} s); L2 flushed between steps (256 MiB write)",
           "gpu_launches_per_step": n_launch, "tma_staging": dict(wl.tma)}
    if do_e2e:
        try:
            e = e2e_run(wl, 1, 3000, stream, dev_id, warm_compute=False)
            e["value"] = len(schemes) * wl.B / (e["ms_per_step"] / 1e3)
            e["unit"] = UNIT
            rec["e2e"] = e
        except RuntimeError as exc:  # pinned host memory for the whole input set not available
            rec["e2e"] = {"unavailable": str(exc)[:200]}
    del wl
    torch.cuda.empty_cache()
    return rec


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
    if a.iters:
        cfg = type(cfg)(**{**cfg.__dict__, "n_iters": a.iters})
    tol = cfg.extra.get("residual_tol")
    if a.scaling == "strong":
        n_total = a.batch or cfg.n_systems
    else:
        n_total = (a.batch or cfg.n_systems) * world
    workload = (f"{a.config}: Nt={cfg.n_antennas} K={cfg.n_users} VR={cfg.vr_len[0]}"
                f"{'' if cfg.vr_len[0] == cfg.vr_len[1] else '-' + str(cfg.vr_len[1])}, "
                f"{len(schemes)} schemes ({','.join(schemes)}) x {n_total} realizations"
                f"{'' if a.scaling == 'strong' else f' ({n_total // world}/rank)'}, "
                + (f"residual tolerance {tol}" if tol else f"T={iters}") + ", RZF + solve + F/NMSE/sum-rate epilogue")

    if a.impl == "reference":
        if rank != 0:
            return
        cores = host_cores()
        walls, per_step, r = cpu_reference_steps(a.config, schemes, iters, a.steps, a.warmup, cores)
        t = float(np.mean(walls))
        val = per_step / t
        line = {"metric": METRIC, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": a.gpus,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
                "scaling": a.scaling, "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
                "config": {"workload": workload, "sample_per_step": f"{r} realizations x {len(schemes)} schemes",
                           "parallelism": f"process pool x{min(cores, per_step)}"},
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": min(cores, per_step), "kind": reference_kind(),
                                 "sample": f"{r} realizations x {len(schemes)} schemes per step, T={iters}, "
                                           + ("the unmodified kaczprec package from baseline/_ref"
                                              if reference_kind() == "reference" else
                                              "oracle/ numpy port of kaczprec (pinned bitwise to the reference; "
                                              "baseline/_ref not installed)")},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    # CPU baseline before any CUDA initialisation (fork-safe), rank 0 at N=1 only
    cpu_baseline = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline and not tol:
        cores = host_cores()
        walls, per_step, r = cpu_reference_steps(a.config, schemes, iters, 1, 0, cores)
        kind = reference_kind()
        cpu_baseline = {"value": per_step / walls[0], "unit": UNIT, "cores": min(cores, per_step), "kind": kind,
                        "sample": f"{r} realization(s) x {len(schemes)} schemes (T={iters}, RZF+solve+assembly+"
                                  "metrics) with " + ("the unmodified kaczprec from baseline/_ref" if kind == "reference"
                                                      else "the oracle/ numpy port") + ", one process per precoder"}

    import torch
    import torch.distributed as dist
    import paper_2501_10689_b200 as kz

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev_id = torch.device("cuda", local)
    lo, hi = kz.shard_range(n_total, rank, world)  # contiguous block of realizations per rank
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev_id)
    big = cfg.n_antennas > 512
    wl = Workload(cfg, schemes, a.dtype, lo, hi, dev_id, chunk=4096 if big else 0, device_inputs=big)
    B = wl.B

    step_ms, per_scheme, launches, clocks = timed_steps(wl, a.steps, a.warmup, 0, flush, world, stream, dist)
    t_rank = float(np.sum(step_ms)) / 1e3
    t = torch.tensor([t_rank], dtype=torch.float64, device=dev_id)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    ms_per_step = 1e3 * t_max / a.steps
    precoders = len(schemes) * n_total * a.steps
    value = precoders / t_max

    # statistics of one more step: the final gather of per-system NMSE / sum-rate / iterations (the only
    # cross-GPU step)
    col = {}
    wl.step(wl.dev, 99, collect=col, stream=stream)
    stats, iters_dom = {}, {}
    for sc in schemes:
        c = {k: torch.cat(v) for k, v in col[sc].items()}
        iters_dom[sc] = c["iters"]
        g = kz.gather_stats({"nmse": c["nmse"], "sum_rate": c["sum_rate"],
                             "iters": c["iters"].double().mean(dim=1)}, n_total)
        stats[sc] = {"median_nmse": float(g["nmse"].median()), "mean_sum_rate": float(g["sum_rate"].mean()),
                     "mean_iters_per_rhs": float(g["iters"].mean()), "systems": int(g["nmse"].numel())}
    rhs_iters = sum(float(iters_dom[sc].double().sum()) for sc in schemes) * world * a.steps / t_max
    dom, avg, roof = roofline(wl, per_scheme, iters_dom if tol else None)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")) as fh:
            tj = json.load(fh)  # DRAM bytes per launch (tools/ncu_capture.sh: the cfg2 solve launches)
            traffic = tj.get(f"{a.config}/{dom}", tj.get(dom) if a.config == "cfg2" else None)
    except (OSError, ValueError):
        pass
    roof["traffic"] = traffic
    roof["measured_views"] = measured_views()
    roof["reg_ffma_stream_view"] = reg_ffma_stream_view(roof["achieved"])
    roof["note"] = ("H_eff is on-chip (shared memory, or a thread-block cluster's shared memory for Nt > 512) and "
                    "each streamed h element feeds 2 rhs in registers (8 FFMA per complex element), so the launch "
                    "is CUDA-core FP32-FMA bound (SURVEY 8(d): report the FMA roofline); flops = 8 x the H_eff "
                    "elements the algorithm streams per rhs-iteration")

    e2e = None
    if not a.no_e2e:
        e = e2e_run(wl, max(1, min(a.steps, 10)), 5000, stream, dev_id)
        te = torch.tensor([e["ms_per_step"]], dtype=torch.float64, device=dev_id)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e["ms_per_step"] = float(te.item())
        e2e = {"value": len(schemes) * n_total / (e["ms_per_step"] / 1e3), "unit": UNIT, **e,
               "path": "kz.DeviceBatch(pinned, upload stream, one step ahead) -> rzf_batched -> solve_batch + "
                       "epilogue per scheme -> V/NMSE/sum-rate to pinned host (copy stream)"}
        if world == 1 and a.config == "cfg2":
            ed = e2e_drops_run(wl, max(1, min(a.steps, 5)), 5500, stream, dev_id)
            e2e["with_input_preparation"] = {"value": len(schemes) * n_total / (ed["ms_per_step"] / 1e3),
                                             "unit": UNIT, **ed}

    # N=1 sub-records (rank 0, one GPU): the complex128 oracle mode of the same step, and cfg3 / cfg4
    c128 = configs = None
    if world == 1 and a.config == "cfg2" and a.dtype == "c64":
        if not a.no_c128:
            wl128 = Workload(cfg, schemes, "c128", lo, hi, dev_id)
            ms128, ev128, _, clk128 = timed_steps(wl128, a.steps, a.warmup, 7, flush, 1, stream, dist)
            e = None
            if not a.no_e2e:
                e = e2e_run(wl128, max(1, min(a.steps, 3)), 6000, stream, dev_id)
                e["value"] = len(schemes) * B / (e["ms_per_step"] / 1e3)
                e["unit"] = UNIT
            c128 = {"value": len(schemes) * B / (float(np.mean(ms128)) / 1e3), "unit": UNIT,
                    "ms_per_step": float(np.mean(ms128)), "steps": a.steps, "warmup": a.warmup,
                    "dtype": "complex128",
                    "per_scheme_launch_ms": {sc: float(np.mean([x.elapsed_time(y) for x, y in ev]))
                                             for sc, ev in ev128.items()},
                    "clocks": clk128, "e2e": e,
                    "note": "the same cfg2 step with the exact-arithmetic kernels of the oracle-mode parity tests "
                            "(complex128, numpy-faithful selection; like-for-like with the complex128 CPU arm)"}
            del wl128
            torch.cuda.empty_cache()
        if not a.no_configs:
            configs = {}
            for name in ("cfg3", "cfg4"):
                configs[name] = config_record(name, dev_id, stream, flush, a.config_steps, 1,
                                              do_e2e=not a.no_e2e)
            # BASELINE cfg3's own variant (orthogonal row groups + at most 8 hyperplanes per aggregated step;
            # no reference counterpart, CPU restatement oracle/grouped.py) on the cluster kernel's grouped path,
            # at the config's stated 4096 realizations
            configs["cfg3_grouped"] = config_record("cfg3", dev_id, stream, flush, a.config_steps, 1,
                                                    do_e2e=not a.no_e2e, n_systems=4096, schemes=["vr-oahk-g"],
                                                    orth_groups=4, agg_cap=8)
            # the reference's default precoder run (run_precoding(epsilon=1e-6), solvers.py:556-603) on the cfg2
            # workload: every scheme NMSE-stopped against the RZF precoder on the on-chip kernels (the reference's
            # own cap, 10^4 K outer iterations)
            configs["cfg2_nmse_stop"] = config_record("cfg2", dev_id, stream, flush, a.config_steps, 1,
                                                      do_e2e=not a.no_e2e, iters=10_000 * CONFIGS["cfg2"].n_users,
                                                      nmse_eps=1e-6)
            # cfg5: wideband OFDM, 1024 subcarriers of one drop, AHK and VR-OAHK at each T of its sweep
            for T in CONFIGS["cfg5"].extra["iter_sweep"]:
                configs[f"cfg5_T{T}"] = config_record("cfg5", dev_id, stream, flush, a.config_steps, 1,
                                                      do_e2e=not a.no_e2e, iters=T)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": a.scaling,
            "vs_baseline": None, "dtype": "complex64" if a.dtype == "c64" else "complex128",
            "data": "synthetic (seeded cfg model: LoS spherical wavefront, contiguous VR, unit-norm columns)",
            "config": {"workload": workload, "global_batch": n_total, "realizations_per_rank": B,
                       "l2": "flushed between timed steps (256 MiB write outside the events)",
                       "rng": "on-device Philox4x32-10 row draws keyed by (seed, global system, rhs, draw)",
                       "parallelism": f"realizations sharded x{world} ({a.scaling} scaling)"},
            "rhs_iterations_per_s": rhs_iters,
            "per_scheme_launch_ms": avg,
            "tma_staging": dict(wl.tma),
            "roofline": roof,
            "cpu_baseline": cpu_baseline, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "stats": stats, "complex128_oracle_mode": c128, "configs": configs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
