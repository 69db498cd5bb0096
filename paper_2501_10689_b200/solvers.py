"""GPU drop-in for the reference solver API (pkg/src/kaczprec/solvers.py).

Public functions keep the reference names, arguments and return types:

  run_precoding(scheme, sys, reference, epsilon=1e-6, max_iters=None, rng=None)   solvers.py:556
  solve(scheme, sys, rhs, stop, rng=None) -> (state, trace)                       solvers.py:460
  solve_all(scheme, sys, stop, rng=None) -> V                                     solvers.py:510

and add batched entry points that take many systems at once:

  solve_batch(dev_batch, scheme, ...)            one kz_solve call over B systems
  run_precoding_batched(scheme, batch, ...)      solve + epilogue (F, NMSE, sum-rate)

Every call runs `kz_solve` from libkaczmarz_b200.so; there is no CPU path.
Random row choices consume the caller's numpy Generator exactly as the
reference does (one `rng.spawn(K)` child per rhs; one `random()` per
greedy-weighted pick, one `integers(K)` per uniform pick, the energy-swor pool
draws) — the draws are evaluated on the host in chunks and streamed to the
device, so row sequences match the reference's.  `rng=("philox", seed)`
instead draws on the device (throughput mode; no reference counterpart).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .batch import DeviceBatch, HostBatch
from .metrics import CADD, CMUL
from .vrgraph import UserPartition, build_partition

SCHEMES = ("urk", "swor-erk", "gk", "grk", "vr-ogrk", "ahk", "vr-oahk")
# batched-API extension (BASELINE cfg3; no reference counterpart, CPU restatement in oracle/grouped.py): VR-OAHK with
# several orthogonal row groups and at most HostBatch.agg_cap hyperplanes per aggregated step
EXTENDED_SCHEMES = ("vr-oahk-g",)
STOCHASTIC_SCHEMES = frozenset({"urk", "swor-erk", "grk", "vr-ogrk"})
VR_SCHEMES = frozenset({"vr-ogrk", "vr-oahk", "vr-oahk-g"})
_UNIFORM_SCHEMES = frozenset({"grk", "vr-ogrk"})


def canonical_scheme(name: str, extended: bool = False) -> str:
    """solvers.py:48-52 (extended=True also accepts EXTENDED_SCHEMES, for the batched entry points)."""
    low = name.strip().lower()
    if low not in SCHEMES and not (extended and low in EXTENDED_SCHEMES):
        raise ValueError(f"unknown scheme {name!r}; expected one of {SCHEMES + (EXTENDED_SCHEMES if extended else ())}")
    return low


def display_scheme(name: str) -> str:
    return canonical_scheme(name).upper()


# ---------------------------------------------------------------------------
# problem description (solvers.py:59-109)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class AugmentedSystem:
    channel: object
    reg: float
    row_energies: np.ndarray
    supports: tuple
    eff_rows: tuple
    h_adj: np.ndarray
    partition: UserPartition

    @classmethod
    def from_channel(cls, chan, reg: float) -> "AugmentedSystem":
        if reg < 0.0:
            raise ValueError("regularisation must be non-negative")
        if chan.n_users < 1:
            raise ValueError("need at least one user")
        supports, eff = [], []
        for k, vr in enumerate(chan.vrs):
            idx = vr.antenna_indices
            outside = np.delete(chan.h[:, k], idx)
            if outside.size and np.any(outside != 0.0):
                raise ValueError(f"column {k} is nonzero outside its visibility region")
            supports.append(idx)
            eff.append(np.ascontiguousarray(chan.h[idx, k]))
        energies = np.array([np.sum(np.abs(e) ** 2) for e in eff]) + reg
        if np.any(energies == 0.0):
            raise ValueError("zero-energy row: empty channel with reg = 0")
        return cls(channel=chan, reg=float(reg), row_energies=energies, supports=tuple(supports),
                   eff_rows=tuple(eff), h_adj=np.ascontiguousarray(chan.h.conj().T),
                   partition=build_partition(chan.vrs))

    @property
    def n_users(self) -> int:
        return self.channel.h.shape[1]

    @property
    def n_antennas(self) -> int:
        return self.channel.h.shape[0]


@dataclass
class StoppingRule:
    """solvers.py:426-450."""

    mode: str = "oracle"
    epsilon: float = 1e-6
    reference: np.ndarray | None = None
    max_iters: int | None = None
    check_every: int = 1

    def __post_init__(self):
        if self.mode not in ("oracle", "residual"):
            raise ValueError(f"unknown stopping mode {self.mode!r}")
        if self.epsilon <= 0.0:
            raise ValueError("epsilon must be positive")
        if self.check_every < 1:
            raise ValueError("check_every must be >= 1")


class FlopCounter:
    """metrics.py:25-41 (batched totals come back from the device; the per-call primitives charge on the host,
    the charges depend only on sizes)."""

    __slots__ = ("total",)

    def __init__(self, total: int = 0):
        self.total = int(total)

    def cmul(self, n: int) -> None:
        self.total += CMUL * n

    def cadd(self, n: int) -> None:
        self.total += CADD * n

    def real(self, n: int) -> None:
        self.total += n


@dataclass
class SolverState:
    rhs: int
    col: np.ndarray
    coef: np.ndarray
    resid: np.ndarray
    counter: FlopCounter = field(default_factory=FlopCounter)
    iters: int = 0
    noop_steps: int = 0

    @classmethod
    def initial(cls, sys, rhs: int, col_buffer: np.ndarray | None = None) -> "SolverState":
        """solvers.py:129-136: m = 0, q = 0, r = e_rhs."""
        if not 0 <= rhs < sys.n_users:
            raise ValueError(f"rhs index {rhs} out of range")
        col = col_buffer if col_buffer is not None else np.zeros(sys.n_antennas, dtype=np.complex128)
        resid = np.zeros(sys.n_users, dtype=np.complex128)
        resid[rhs] = 1.0
        return cls(rhs=rhs, col=col, coef=np.zeros(sys.n_users, dtype=np.complex128), resid=resid)


@dataclass
class RunTrace:
    scheme: str
    seed: int | None = None
    nmse: list = field(default_factory=list)
    resid: list = field(default_factory=list)
    flops: list = field(default_factory=list)
    n_iters: int = 0
    converged: bool = True
    flops_analytic: float | None = None
    flops_measured: int | None = None
    sum_rate: float | None = None


@dataclass
class PrecodingRun:
    """solvers.py:540-553."""

    scheme: str
    v: np.ndarray
    precoder: object
    n_iters: int
    converged: bool
    nmse_trace: list
    resid_trace: list
    flops_trace: list
    flops_measured: int
    noop_steps: int


# ---------------------------------------------------------------------------
# host-evaluated row streams
# ---------------------------------------------------------------------------

class HostStreams:
    """Draw the reference's random row decisions chunk by chunk.

    gens[b][c] is the Generator the reference's InstanceRun for (system b, rhs c)
    would hold.  Per chunk, each rhs yields `n` draws:
      grk / vr-ogrk : Generator.random()           (solvers.py:237, via choice)
      urk           : Generator.integers(K)         (solvers.py:219)
      swor-erk      : pool pick index                (solvers.py:224-230)
    """

    def __init__(self, scheme: str, gens, energies: np.ndarray):
        self.scheme = scheme
        self.gens = gens
        self.energies = energies  # (B, K)
        b, k = energies.shape
        self.pools = [[[] for _ in range(k)] for _ in range(b)]

    @property
    def kind(self):
        return _lib.RNG_HOST_UNIFORM if self.scheme in _UNIFORM_SCHEMES else _lib.RNG_HOST_INDEX

    def chunk(self, n: int, active=None) -> np.ndarray:
        b, k = self.energies.shape
        if self.kind == _lib.RNG_HOST_UNIFORM:
            out = np.zeros((b, k, n), dtype=np.float64)
        else:
            out = np.zeros((b, k, n), dtype=np.int32)
        for s in range(b):
            for c in range(k):
                g = self.gens[s][c]
                if g is None or (active is not None and not active[s, c]):
                    continue
                if self.scheme in _UNIFORM_SCHEMES:
                    out[s, c] = g.random(n)
                elif self.scheme == "urk":
                    out[s, c] = g.integers(k, size=n)
                else:
                    pool = self.pools[s][c]
                    e = self.energies[s]
                    for t in range(n):
                        if not pool:
                            pool.extend(range(k))
                        w = e[pool]
                        out[s, c, t] = pool.pop(int(g.choice(len(pool), p=w / w.sum())))
        return out


# ---------------------------------------------------------------------------
# batched solve (one kz_solve call, chunked only for host streams)
# ---------------------------------------------------------------------------

@dataclass
class BatchResult:
    scheme: str
    dev: DeviceBatch
    v: object                 # torch (B, K, K) complex on device: v[b, i, c]
    iters: object             # torch (B, K) int32
    converged: object         # (B, K) uint8
    done: object
    noop_steps: object
    flops: object             # (B, K) int64
    n_outer: object           # (B,) int32
    sys_converged: object     # (B,) uint8
    rows: object = None       # (B, K, rows_cap) int32
    nmse_trace: object = None
    resid_trace: object = None
    flops_trace: object = None
    n_checks: object = None
    workspace: object = None
    launches: int = 0
    tma_staging: bool = False  # H_eff staged into shared memory by TMA tensor copies (kz_last_tma_staging)

    m: object = None          # (B, K rhs, Nt) final iterates when requested

    def iterates(self):
        """Final iterate block M (col = H coef) as (B, K rhs, Nt); needs want_iterates=True."""
        if self.m is None:
            raise ValueError("solve_batch(..., want_iterates=True) was not requested")
        return self.m


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def solve_batch(dev: DeviceBatch, scheme: str, *, mode: str = "lockstep", max_iters: int, epsilon: float = 0.0,
                check_every: int = 1, f_ref=None, v_ref=None, rng=None, rows_cap: int = 0, trace_cap: int = 0,
                rhs_mask=None, chunk: int | None = None, stream=None, workspace=None,
                want_iterates: bool = False, system_base: int = 0,
                traces=("nmse", "resid", "flops")) -> BatchResult:
    """Run `scheme` on every (system, rhs) of `dev` with one kz_solve launch.

    mode: "lockstep" (run_precoding), "residual" / "oracle" (solve / solve_all).
    rng : None, ("philox", seed), or a HostStreams.
    system_base: global index of system 0 of `dev` (Philox draws are keyed by the global system index, so a
    realization's rows do not depend on how the batch is chunked or sharded).
    traces: which per-outer-iteration traces trace_cap > 0 records (subset of nmse / resid / flops).  A lockstep
    complex64 run without the residual trace (NMSE-stopped or not) stays on the register-resident wide kernel.
    """
    import torch
    scheme = canonical_scheme(scheme, extended=True)
    if scheme == "vr-oahk" and getattr(dev.host, "orth_groups", 1) > 1:
        raise ValueError("this batch holds several orthogonal groups (orth_groups > 1): run vr-oahk-g on it, or "
                         "build the batch with orth_groups=1 for vr-oahk")
    lb = _lib.lib()
    b, k = dev.n_systems, dev.n_users
    d = dev.device
    cdt = dev.complex_dtype
    mode_id = {"lockstep": _lib.STOP_LOCKSTEP, "residual": _lib.STOP_RESIDUAL, "oracle": _lib.STOP_ORACLE}[mode]
    if scheme in STOCHASTIC_SCHEMES and rng is None:
        raise ValueError(f"scheme {scheme!r} draws rows at random; pass an rng")

    z = lambda *shape, dt: torch.zeros(shape, dtype=dt, device=d)  # noqa: E731
    res = BatchResult(scheme=scheme, dev=dev, v=z(b, k, k, dt=cdt), iters=z(b, k, dt=torch.int32),
                      converged=z(b, k, dt=torch.uint8), done=z(b, k, dt=torch.uint8),
                      noop_steps=z(b, k, dt=torch.int32), flops=z(b, k, dt=torch.int64),
                      n_outer=z(b, dt=torch.int32), sys_converged=z(b, dt=torch.uint8))
    paused = z(b, k, dt=torch.uint8)
    if want_iterates:
        res.m = z(b, k, dev.n_antennas, dt=cdt)
    if rows_cap:
        res.rows = torch.full((b, k, rows_cap), -1, dtype=torch.int32, device=d)
    if trace_cap:
        n = b if mode == "lockstep" else b * k
        bad = set(traces) - {"nmse", "resid", "flops"}
        if bad:
            raise ValueError(f"unknown traces {sorted(bad)!r}")
        if "nmse" in traces:
            res.nmse_trace = z(n, trace_cap, dt=torch.float64)
        if "resid" in traces:
            res.resid_trace = z(n, trace_cap, dt=torch.float64)
        if "flops" in traces:
            res.flops_trace = z(n, trace_cap, dt=torch.int64)
        res.n_checks = z(b, k, dt=torch.int32)

    stop = _lib.KzStop()
    stop.mode = mode_id
    stop.max_iters = int(max_iters)
    stop.check_every = int(check_every)
    stop.epsilon = float(epsilon)
    keep = []
    if f_ref is not None:
        f_ref = torch.as_tensor(f_ref).to(device=d, dtype=torch.complex128).contiguous()
        keep.append(f_ref)
        stop.f_ref = f_ref.data_ptr()
    if v_ref is not None:
        v_ref = torch.as_tensor(v_ref).to(device=d, dtype=torch.complex128).contiguous()
        keep.append(v_ref)
        stop.v_ref = v_ref.data_ptr()
    if rhs_mask is not None:
        m = torch.as_tensor(np.asarray(rhs_mask, dtype=np.uint8)).to(d)
        keep.append(m)
        stop.rhs_mask = m.data_ptr()

    out = _lib.KzOut()
    out.v = res.v.data_ptr()
    out.iters = res.iters.data_ptr()
    out.converged = res.converged.data_ptr()
    out.done = res.done.data_ptr()
    out.noop_steps = res.noop_steps.data_ptr()
    out.flops = res.flops.data_ptr()
    out.n_outer = res.n_outer.data_ptr()
    out.sys_converged = res.sys_converged.data_ptr()
    out.paused = paused.data_ptr()
    if want_iterates:
        out.iterates = res.m.data_ptr()
    if rows_cap:
        out.rows = res.rows.data_ptr()
        out.rows_cap = rows_cap
    if trace_cap:
        out.trace_cap = trace_cap
        ptr = lambda t: 0 if t is None else t.data_ptr()  # noqa: E731
        out.nmse_trace = ptr(res.nmse_trace)
        out.resid_trace = ptr(res.resid_trace)
        out.flops_trace = ptr(res.flops_trace)
        out.n_checks = res.n_checks.data_ptr()

    rg = _lib.KzRng()
    host = isinstance(rng, HostStreams)
    if rng is None:
        rg.kind = _lib.RNG_NONE
    elif host:
        rg.kind = rng.kind
    else:
        kind, seed = rng
        if kind != "philox":
            raise ValueError(f"unknown rng spec {rng!r}")
        rg.kind = _lib.RNG_PHILOX
        rg.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        rg.system_base = int(system_base)
    if host and scheme not in STOCHASTIC_SCHEMES:
        host = False
        rg.kind = _lib.RNG_NONE
    sp = _stream_ptr(stream)
    resume = 0
    base = 0
    if chunk is None:
        chunk = int(max_iters) if mode == "lockstep" else min(int(max_iters), 1024)
    launches = 0
    active = np.ones((b, k), dtype=bool) if rhs_mask is None else np.asarray(rhs_mask, dtype=bool).reshape(b, k)
    while True:
        if host:
            arr = torch.from_numpy(rng.chunk(chunk, active)).to(d)
            keep.append(arr)
            rg.stream_len = chunk
            rg.stream_base = base
            if rg.kind == _lib.RNG_HOST_UNIFORM:
                rg.uniforms = arr.data_ptr()
            else:
                rg.indices = arr.data_ptr()
        if not resume:
            # size the workspace for the kernel this call dispatches to (the on-chip kernels need only the stop
            # bookkeeping; the global-memory kernel holds every iterate)
            need = lb.kz_solve_workspace_bytes_for(C.byref(dev.problem), _lib.SCHEME_IDS[scheme], C.byref(stop),
                                                   C.byref(rg), C.byref(out))
            if workspace is None or workspace.numel() < need:
                workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=d)
            res.workspace = workspace
        _lib.check(lb.kz_solve(C.byref(dev.problem), _lib.SCHEME_IDS[scheme], C.byref(stop), C.byref(rg),
                               C.byref(out), workspace.data_ptr(), workspace.numel(), resume, sp))
        launches += lb.kz_last_launch_count()
        res.tma_staging = bool(lb.kz_last_tma_staging())
        if not host:
            break
        pz = paused.cpu().numpy().astype(bool)
        if not pz.any():
            break
        active = pz
        paused.zero_()
        base += chunk
        resume = 1
    res.launches = launches
    res._keep = keep
    return res


# ---------------------------------------------------------------------------
# flop bookkeeping that happens outside the kernels (run_precoding :579, :604-611)
# ---------------------------------------------------------------------------

def _assembly_flops_vr(sys) -> int:
    """assemble_vr counter charges for the channel's subarray grid (assembly.py:74-92)."""
    chan = sys.channel
    k = sys.n_users
    m = chan.cfg.subarray_size
    tot = 0
    for s in range(chan.cfg.n_subarrays):
        q = sum(1 for vr in chan.vrs if s in vr.visible_subarrays)
        if q:
            tot += 6 * m * q * k + 2 * m * (q - 1) * k
    return tot


def _assembly_flops_dense(nt: int, k: int) -> int:
    return 6 * nt * k * k + 2 * nt * k * (k - 1)


def _gens_for(rng, k):
    return rng.spawn(k) if rng is not None else [None] * k


def _f_ref_of(reference):
    return reference.f if hasattr(reference, "f") else np.asarray(reference)


# ---------------------------------------------------------------------------
# reference-signature entry points
# ---------------------------------------------------------------------------

def run_precoding(scheme: str, sys, reference, epsilon: float = 1e-6, max_iters: int | None = None,
                  rng: np.random.Generator | None = None) -> PrecodingRun:
    """Lockstep K-rhs run with NMSE stopping (solvers.py:556-623), on the GPU."""
    import torch
    from .assembly import epilogue
    from .rzf import Precoder
    scheme = canonical_scheme(scheme)
    k, nt = sys.n_users, sys.n_antennas
    cap = max_iters if max_iters is not None else 10_000 * k
    host = HostBatch.from_systems([sys])
    dev = host.to_device("c128")
    f_ref = np.asarray(_f_ref_of(reference), dtype=np.complex128)[None]
    streams = None
    if scheme in STOCHASTIC_SCHEMES:
        if rng is None:
            raise ValueError(f"scheme {scheme!r} draws rows at random; pass an rng")
        streams = HostStreams(scheme, [_gens_for(rng, k)], host.row_energy.reshape(1, k))
    res = solve_batch(dev, scheme, mode="lockstep", max_iters=cap, epsilon=epsilon, f_ref=f_ref, rng=streams,
                      trace_cap=cap)
    t = int(res.n_outer[0])
    setup = 4 * nt * k
    v = res.v[0].cpu().numpy()
    ep = epilogue(dev, res.v, want_f=True)
    f = ep["f"][0].cpu().numpy()
    asm = _assembly_flops_vr(sys) if scheme in VR_SCHEMES else _assembly_flops_dense(nt, k)
    flops_rhs = int(res.flops[0].sum())
    return PrecodingRun(
        scheme=display_scheme(scheme), v=v,
        precoder=Precoder(f=f, norm_factor=float(ep["beta"][0]), scheme=display_scheme(scheme)),
        n_iters=t, converged=bool(res.sys_converged[0]),
        nmse_trace=res.nmse_trace[0, :t].cpu().tolist(), resid_trace=res.resid_trace[0, :t].cpu().tolist(),
        flops_trace=[setup + int(x) for x in res.flops_trace[0, :t].cpu().tolist()],
        flops_measured=setup + flops_rhs + asm, noop_steps=int(res.noop_steps[0].sum()))


def _stored_resid(res: BatchResult, c: int) -> np.ndarray:
    """The stored row residuals the scheme left for rhs c of system 0 (SolverState.resid), read from the
    complex128 solve workspace at kz_solve_resid_offset."""
    import torch
    k = res.dev.n_users
    off = int(_lib.lib().kz_solve_resid_offset(C.byref(res.dev.problem))) + c * k * 16
    return res.workspace[off:off + k * 16].view(torch.complex128).cpu().numpy().copy()


def _state_from(res: BatchResult, c: int) -> SolverState:
    m = res.iterates()[0, c].cpu().numpy()
    return SolverState(rhs=c, col=m, coef=res.v[0, :, c].cpu().numpy(), resid=_stored_resid(res, c),
                       counter=FlopCounter(int(res.flops[0, c])), iters=int(res.iters[0, c]),
                       noop_steps=int(res.noop_steps[0, c]))


def solve(scheme: str, sys, rhs: int, stop: StoppingRule, rng: np.random.Generator | None = None):
    """Single-rhs run with oracle / residual stopping (solvers.py:460-507), on the GPU."""
    scheme = canonical_scheme(scheme)
    k = sys.n_users
    if not 0 <= rhs < k:
        raise ValueError(f"rhs index {rhs} out of range")
    v_ref = None
    if stop.mode == "oracle":
        if stop.reference is None:
            raise ValueError("oracle stopping needs the direct-solver reference column")
        ref = np.asarray(stop.reference)
        if float(np.linalg.norm(ref)) == 0.0:
            raise ValueError("oracle reference column is zero")
        v_ref = np.zeros((1, k, k), dtype=np.complex128)
        v_ref[0, :, rhs] = ref
    if scheme in STOCHASTIC_SCHEMES and rng is None:
        raise ValueError(f"scheme {scheme!r} draws rows at random; pass an rng")
    cap = stop.max_iters if stop.max_iters is not None else 10_000 * k
    host = HostBatch.from_systems([sys])
    dev = host.to_device("c128")
    streams = None
    if scheme in STOCHASTIC_SCHEMES:
        gens = [[rng if c == rhs else None for c in range(k)]]
        streams = HostStreams(scheme, gens, host.row_energy.reshape(1, k))
    mask = np.zeros(k, dtype=np.uint8)
    mask[rhs] = 1
    cap_trace = max(1, cap // stop.check_every + 1)
    res = solve_batch(dev, scheme, mode=stop.mode, max_iters=cap, epsilon=stop.epsilon,
                      check_every=stop.check_every, v_ref=v_ref, rng=streams, rhs_mask=mask,
                      trace_cap=min(cap_trace, 1 << 20), want_iterates=True)
    st = _state_from(res, rhs)
    n = int(res.n_checks[0, rhs])
    tr = RunTrace(scheme=display_scheme(scheme))
    tr.resid = res.resid_trace[rhs, :n].cpu().tolist()
    tr.flops = [int(x) for x in res.flops_trace[rhs, :n].cpu().tolist()]
    if stop.mode == "oracle":
        tr.nmse = res.nmse_trace[rhs, :n].cpu().tolist()
    tr.n_iters = st.iters
    tr.converged = bool(res.converged[0, rhs])
    tr.flops_measured = st.counter.total
    return st, tr


def solve_all(scheme: str, sys, stop: StoppingRule, rng: np.random.Generator | None = None) -> np.ndarray:
    """Per-column solves, rng.spawn(K) children (solvers.py:510-537), on the GPU."""
    scheme = canonical_scheme(scheme)
    k = sys.n_users
    v_ref = None
    if stop.mode == "oracle":
        ref = np.asarray(stop.reference)
        if ref.shape != (k, k):
            raise ValueError(f"oracle reference must be (K, K), got {ref.shape}")
        if np.any(np.linalg.norm(ref, axis=0) == 0.0):
            raise ValueError("oracle reference column is zero")
        v_ref = ref[None]
    if scheme in STOCHASTIC_SCHEMES and rng is None:
        raise ValueError(f"scheme {scheme!r} draws rows at random; pass an rng")
    cap = stop.max_iters if stop.max_iters is not None else 10_000 * k
    host = HostBatch.from_systems([sys])
    dev = host.to_device("c128")
    streams = None
    if scheme in STOCHASTIC_SCHEMES:
        streams = HostStreams(scheme, [_gens_for(rng, k)], host.row_energy.reshape(1, k))
    res = solve_batch(dev, scheme, mode=stop.mode, max_iters=cap, epsilon=stop.epsilon,
                      check_every=stop.check_every, v_ref=v_ref, rng=streams)
    return res.v[0].cpu().numpy()


# ---------------------------------------------------------------------------
# batched precoding (the throughput entry point)
# ---------------------------------------------------------------------------

def run_precoding_batched(scheme: str, dev: DeviceBatch, *, max_iters: int, rng=None, epsilon: float = 0.0,
                          f_ref=None, v_ref=None, beta_ref=None, rates: bool = True, want_f: bool = False,
                          rows_cap: int = 0, stream=None, workspace=None, chunk_systems: int = 0,
                          system_base: int = 0) -> dict:
    """Fixed-T (epsilon = 0) or NMSE-stopped lockstep precoding of every system in `dev`,
    followed by the fused epilogue (F = beta H V, NMSE vs beta_ref H V_ref, Eq. (7) rates).

    chunk_systems > 0 runs the batch as consecutive views of that many systems (bounded per-call workspaces
    and outputs; Philox draws keyed by the global system index, so the results equal the one-call run).
    system_base: global index of system 0 of `dev` (sharded callers)."""
    import torch
    from .assembly import epilogue
    b = dev.n_systems
    if chunk_systems <= 0 or chunk_systems >= b:
        res = solve_batch(dev, scheme, mode="lockstep", max_iters=max_iters, epsilon=epsilon, f_ref=f_ref, rng=rng,
                          rows_cap=rows_cap, stream=stream, workspace=workspace, system_base=system_base)
        ep = epilogue(dev, res.v, v_ref=v_ref, beta_ref=beta_ref, rates=rates, want_f=want_f, stream=stream)
        out = {"solve": res, **ep, "v": res.v}
        out["launches"] = res.launches + ep["launches"]
        return out
    if isinstance(rng, HostStreams):
        raise ValueError("chunk_systems needs on-device draws (rng=('philox', seed)) or a deterministic scheme")
    sl = lambda a, lo, hi: None if a is None else a[lo:hi]  # noqa: E731
    parts, eps_, launches = [], [], 0
    for lo in range(0, b, chunk_systems):
        hi = min(b, lo + chunk_systems)
        sub = dev.view(lo, hi)
        res = solve_batch(sub, scheme, mode="lockstep", max_iters=max_iters, epsilon=epsilon,
                          f_ref=sl(f_ref, lo, hi), rng=rng, rows_cap=rows_cap, stream=stream, workspace=workspace,
                          system_base=system_base + lo)
        workspace = res.workspace
        ep = epilogue(sub, res.v, v_ref=sl(v_ref, lo, hi), beta_ref=sl(beta_ref, lo, hi), rates=rates,
                      want_f=want_f, stream=stream)
        parts.append(res)
        eps_.append(ep)
        launches += res.launches + ep["launches"]
    cat = lambda xs: None if xs[0] is None else torch.cat(xs)  # noqa: E731
    res = BatchResult(scheme=parts[0].scheme, dev=dev, **{f: cat([getattr(p, f) for p in parts]) for f in (
        "v", "iters", "converged", "done", "noop_steps", "flops", "n_outer", "sys_converged", "rows")})
    res.launches = launches
    out = {"solve": res, "v": res.v, "launches": launches, "workspace": None, "gram_form": eps_[0]["gram_form"]}
    for key in ("f", "beta", "nmse", "rates", "sum_rate"):
        out[key] = cat([e[key] for e in eps_])
    return out


# ---------------------------------------------------------------------------
# per-call step primitives and InstanceRun (solvers.py:143-423): one rhs of one system, state on the GPU
# for the duration of each call (kz_residual_refresh / kz_project_rows / kz_ahk_step)
# ---------------------------------------------------------------------------

def _prim_device(sys) -> DeviceBatch:
    """The system as a one-system complex128 batch on the current GPU, built once per AugmentedSystem."""
    dev = sys.__dict__.get("_kz_prim_dev")
    if dev is None:
        dev = HostBatch.from_systems([sys]).to_device("c128")
        sys.__dict__["_kz_prim_dev"] = dev
    return dev


class _DeviceState:
    """col / coef / resid of a SolverState uploaded for one primitive call and written back in place."""

    def __init__(self, state: SolverState, sys):
        import torch
        self.state, self.dev = state, _prim_device(sys)
        d = self.dev.device
        self.col = torch.from_numpy(np.ascontiguousarray(state.col, dtype=np.complex128)).to(d)
        self.coef = torch.from_numpy(np.ascontiguousarray(state.coef, dtype=np.complex128)).to(d)
        self.resid = torch.from_numpy(np.ascontiguousarray(state.resid, dtype=np.complex128)).to(d)

    def rows(self, rows):
        import torch
        return torch.from_numpy(np.ascontiguousarray(rows, dtype=np.int32)).to(self.dev.device)

    def write_back(self, col=True, coef=True, resid=True):
        if col:
            self.state.col[...] = self.col.cpu().numpy()
        if coef:
            self.state.coef[...] = self.coef.cpu().numpy()
        if resid:
            self.state.resid[...] = self.resid.cpu().numpy()


def _sizes(sys, rows):
    return [int(np.asarray(sys.supports[i]).size) for i in rows]


def residual_refresh(state: SolverState, sys, rows=None, use_vr: bool = True) -> None:
    """solvers.py:143-170 on the GPU: r_i = s_i - h_i^H col - reg coef_i for `rows` (None: all)."""
    k, nt = sys.n_users, sys.n_antennas
    dense_all = rows is None and not use_vr
    idx = np.arange(k) if rows is None else np.asarray([int(r) for r in rows], dtype=np.int64)
    if idx.size == 0:
        return
    ds = _DeviceState(state, sys)
    r = ds.rows(idx)
    _lib.check(_lib.lib().kz_residual_refresh(C.byref(ds.dev.problem), 0, int(state.rhs), _lib.ptr(ds.col),
                                              _lib.ptr(ds.coef), _lib.ptr(ds.resid), _lib.ptr(r), int(idx.size),
                                              1 if dense_all else 0, _stream_ptr(None)))
    ds.write_back(col=False, coef=False)
    if dense_all:
        state.counter.cmul(k * nt)
        state.counter.cadd(k * (nt + 1))
        state.counter.real(2 * k)
        return
    for n in (_sizes(sys, idx) if use_vr else [nt] * idx.size):
        state.counter.cmul(n)
        state.counter.cadd(n + 1)
        state.counter.real(2)


def _project(state: SolverState, sys, rows, use_vr: bool) -> None:
    ds = _DeviceState(state, sys)
    r = ds.rows(rows)
    _lib.check(_lib.lib().kz_project_rows(C.byref(ds.dev.problem), 0, _lib.ptr(ds.col), _lib.ptr(ds.coef),
                                          _lib.ptr(ds.resid), _lib.ptr(r), len(rows), _stream_ptr(None)))
    ds.write_back()
    for n in (_sizes(sys, rows) if use_vr else [sys.n_antennas] * len(rows)):
        state.counter.real(2)
        state.counter.cmul(n)
        state.counter.cadd(n + 1)


def rk_step(state: SolverState, sys, i: int, use_vr: bool = True) -> None:
    """solvers.py:173-188 on the GPU: project onto row i with the stored residual."""
    _project(state, sys, [int(i)], use_vr)
    state.iters += 1


def orthogonal_block_step(state: SolverState, sys, rows, use_vr: bool = True) -> None:
    """solvers.py:312-332 on the GPU: exact projections onto the (pairwise orthogonal) rows, in order."""
    rows = [int(r) for r in rows]
    if rows:
        _project(state, sys, rows, use_vr)


@dataclass
class SelectionStrategy:
    """solvers.py:191-203: row-choice rule; `pool` holds the without-replacement epoch state."""

    variant: str
    pool: list = field(default_factory=list)

    _VARIANTS = ("uniform", "energy", "energy-swor", "greedy-max", "greedy-weighted")

    def __post_init__(self):
        if self.variant not in self._VARIANTS:
            raise ValueError(f"unknown selection variant {self.variant!r}")


def select_row(strategy: SelectionStrategy, state: SolverState, sys, rng: np.random.Generator | None = None):
    """solvers.py:205-237.  The draw consumes the caller's numpy Generator on the host, exactly as the
    reference (and as HostStreams does for the batched kernels); the K-entry residual it reads is the one the
    GPU primitives wrote back."""
    k = sys.n_users
    variant = strategy.variant
    if variant == "greedy-max":
        score = np.abs(state.resid) ** 2 / sys.row_energies
        state.counter.real(4 * k)
        if not score.any():
            return None
        return int(np.argmax(score))
    if rng is None:
        raise ValueError(f"selection variant {variant!r} needs an rng")
    if variant == "uniform":
        return int(rng.integers(k))
    if variant == "energy":
        w = sys.row_energies
        state.counter.real(k + 2)
        return int(rng.choice(k, p=w / w.sum()))
    if variant == "energy-swor":
        if not strategy.pool:
            strategy.pool = list(range(k))
        w = sys.row_energies[strategy.pool]
        state.counter.real(len(strategy.pool) + 2)
        return strategy.pool.pop(int(rng.choice(len(strategy.pool), p=w / w.sum())))
    w = np.abs(state.resid) ** 2
    state.counter.real(4 * k + 2)
    total = w.sum()
    if total == 0.0:
        return None
    return int(rng.choice(k, p=w / total))


@dataclass(frozen=True)
class AggregationWeights:
    """solvers.py:240-245: phi (K complex, zero off `rows`) and the sorted rows."""

    phi: np.ndarray
    rows: np.ndarray


def aggregation_weights(state: SolverState, sys, rows) -> AggregationWeights:
    """solvers.py:248-254: phi_i = r_i / e_i on the sorted rows."""
    rows = np.asarray(sorted(int(r) for r in rows), dtype=np.intp)
    phi = np.zeros(sys.n_users, dtype=np.complex128)
    phi[rows] = state.resid[rows] / sys.row_energies[rows]
    state.counter.real(2 * rows.size)
    return AggregationWeights(phi=phi, rows=rows)


def ahk_step(state: SolverState, sys, weights: AggregationWeights, use_vr: bool = True,
             union: np.ndarray | None = None) -> bool:
    """solvers.py:257-309 on the GPU: one projection onto the aggregated hyperplane; False (no-op flag) when
    phi vanishes or the aggregated row is zero."""
    import torch
    rows = np.asarray(weights.rows, dtype=np.int64)
    m = rows.size
    if m == 0 or not weights.phi[rows].any():
        state.noop_steps += 1
        return False
    state.counter.cmul(m)
    state.counter.cadd(max(m - 1, 0))
    nt = sys.n_antennas
    if use_vr:
        if union is None:
            union = np.unique(np.concatenate([np.asarray(sys.supports[i]) for i in rows]))
        for n in _sizes(sys, rows):
            state.counter.cmul(n)
            state.counter.cadd(n)
        span_size = int(np.asarray(union).size)
    else:
        state.counter.cmul(nt * m)
        state.counter.cadd(nt * max(m - 1, 0))
        span_size = nt
    state.counter.real(4 * span_size + 3 * m + 2)
    ds = _DeviceState(state, sys)
    d = ds.dev.device
    phi = torch.from_numpy(np.ascontiguousarray(weights.phi, dtype=np.complex128)).to(d)
    r = ds.rows(rows)
    span = ds.rows(np.asarray(union)) if use_vr else None
    stepped = torch.zeros(1, dtype=torch.int32, device=d)
    _lib.check(_lib.lib().kz_ahk_step(C.byref(ds.dev.problem), 0, _lib.ptr(ds.col), _lib.ptr(ds.coef),
                                      _lib.ptr(ds.resid), _lib.ptr(phi), _lib.ptr(r), int(m), _lib.ptr(span),
                                      0 if span is None else int(span.numel()), _lib.ptr(stepped),
                                      _stream_ptr(None)))
    if not int(stepped.item()):
        state.noop_steps += 1
        return False
    ds.write_back(resid=False)
    state.counter.real(2)
    state.counter.cmul(span_size)
    state.counter.cadd(span_size)
    state.counter.cmul(m)
    state.counter.cadd(m)
    return True


class InstanceRun:
    """solvers.py:345-423: one right-hand side advanced one scheme iteration at a time, composed from the GPU
    primitives above exactly as the reference composes its numpy ones."""

    def __init__(self, scheme: str, sys, rhs: int, rng: np.random.Generator | None,
                 col_buffer: np.ndarray | None = None):
        self.scheme = canonical_scheme(scheme)
        if self.scheme in STOCHASTIC_SCHEMES and rng is None:
            raise ValueError(f"scheme {self.scheme!r} draws rows at random; pass an rng")
        self.sys = sys
        self.rng = rng
        self.state = SolverState.initial(sys, rhs, col_buffer=col_buffer)
        self.done = False
        self.strategy = {"urk": SelectionStrategy("uniform"), "swor-erk": SelectionStrategy("energy-swor"),
                         "gk": SelectionStrategy("greedy-max"), "grk": SelectionStrategy("greedy-weighted"),
                         "vr-ogrk": SelectionStrategy("greedy-weighted")}.get(self.scheme)
        if self.scheme == "vr-ogrk":
            self.prev_row = None
            self.coupled = [np.asarray(sorted(c), dtype=np.intp) for c in sys.partition.coupled]
        if self.scheme == "vr-oahk":
            self.orth_rows = np.asarray(sys.partition.orthogonal_sorted, dtype=np.intp)
            self.non_rows = np.asarray(sys.partition.non_orthogonal, dtype=np.intp)
            self.non_union = (np.unique(np.concatenate([np.asarray(sys.supports[i]) for i in self.non_rows]))
                              if self.non_rows.size else None)
        if self.scheme == "ahk":
            self.all_rows = np.arange(sys.n_users)

    def step(self) -> None:
        if self.done:
            return
        scheme, state, sys = self.scheme, self.state, self.sys
        if scheme in ("urk", "swor-erk"):
            i = select_row(self.strategy, state, sys, self.rng)
            residual_refresh(state, sys, rows=(i,), use_vr=False)
            rk_step(state, sys, i, use_vr=False)
        elif scheme in ("gk", "grk"):
            residual_refresh(state, sys, use_vr=False)
            i = select_row(self.strategy, state, sys, self.rng)
            if i is None:
                self.done = True
                return
            rk_step(state, sys, i, use_vr=False)
        elif scheme == "vr-ogrk":
            if self.prev_row is not None:
                residual_refresh(state, sys, rows=self.coupled[self.prev_row], use_vr=True)
            i = select_row(self.strategy, state, sys, self.rng)
            if i is None:
                self.done = True
                return
            rk_step(state, sys, i, use_vr=True)
            self.prev_row = i
        elif scheme == "ahk":
            residual_refresh(state, sys, use_vr=False)
            weights = aggregation_weights(state, sys, self.all_rows)
            if not ahk_step(state, sys, weights, use_vr=False):
                self.done = True
                return
            state.iters += 1
        else:  # vr-oahk
            residual_refresh(state, sys, rows=self.orth_rows, use_vr=True)
            orthogonal_block_step(state, sys, self.orth_rows, use_vr=True)
            if self.non_rows.size:
                residual_refresh(state, sys, rows=self.non_rows, use_vr=True)
                weights = aggregation_weights(state, sys, self.non_rows)
                ahk_step(state, sys, weights, use_vr=True, union=self.non_union)
            state.iters += 1
