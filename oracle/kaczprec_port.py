"""Numpy restatement of the reference Kaczmarz precoding path (TEST ORACLE ONLY).

Every function cites the reference file:line it restates; paths are relative
to the reference checkout's `pkg/src/kaczprec/`.  The arithmetic is expressed
with the same numpy primitives the reference uses (BLAS `@`/`vdot`, SIMD
`abs`, `Generator.choice/integers/spawn`, LAPACK Cholesky) so that on the same
host the results are bitwise identical to the reference; the committed
fixtures in `tests/golden/` pin that claim.

Scope: channel model (only what the reference tests' instances need), the
VR overlap partition, the seven row-action schemes with their flop charges,
the three stopping drivers (`solve`, `solve_all`, `run_precoding`), the direct
RZF solve, precoder assembly, NMSE and sum-rate.  The config-shaped
near-field channel of BASELINE.json is *input generation*, not part of the
reference, and lives in the product package.

Additions over the reference (checker conveniences, no behavioural change):
each chain records the row it projected at every step (`rows_log`), and
`run_precoding` returns those logs, so the GPU's row sequences can be
compared exactly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np
import scipy.linalg

__all__ = [
    "SPEED_OF_LIGHT", "ArrayConfig", "VisibilityRegion", "ChannelMatrix",
    "contiguous_region", "random_channel", "power_control",
    "UserPartition", "build_partition",
    "SCHEMES", "STOCHASTIC_SCHEMES", "VR_SCHEMES", "canonical_scheme",
    "AugmentedSystem", "SolverState", "FlopCounter",
    "residual_refresh", "rk_step", "SelectionStrategy", "select_row",
    "aggregation_weights", "ahk_step", "orthogonal_block_step",
    "InstanceRun", "StoppingRule", "solve", "solve_all",
    "PrecodingRun", "run_precoding",
    "Precoder", "auxiliary_matrix", "rzf_precoder",
    "assemble_dense", "assemble_vr", "nmse", "spectral_efficiency",
    "flops_measured_for",
]

# --------------------------------------------------------------------------
# channel.py — just enough of the reference model to rebuild its test drops
# --------------------------------------------------------------------------

SPEED_OF_LIGHT = 2.99792458e8  # channel.py:18


@dataclass(frozen=True)
class ArrayConfig:
    """ULA at half-wavelength spacing split into equal subarrays (channel.py:26-70)."""

    n_antennas: int
    carrier_freq: float
    n_subarrays: int = 1

    def __post_init__(self):
        if self.n_antennas < 1 or self.carrier_freq <= 0:
            raise ValueError("bad array configuration")
        if self.n_subarrays < 1 or self.n_antennas % self.n_subarrays:
            raise ValueError("n_subarrays must divide n_antennas")

    @property
    def wavelength(self) -> float:
        return SPEED_OF_LIGHT / self.carrier_freq

    @property
    def spacing(self) -> float:
        return self.wavelength / 2.0

    @property
    def subarray_size(self) -> int:
        return self.n_antennas // self.n_subarrays


@dataclass(frozen=True)
class VisibilityRegion:
    """Set of visible subarrays (channel.py:135-172)."""

    visible_subarrays: frozenset
    n_subarrays: int
    subarray_size: int

    def __post_init__(self):
        if not self.visible_subarrays:
            raise ValueError("visibility region must contain at least one subarray")
        if any(not 0 <= s < self.n_subarrays for s in self.visible_subarrays):
            raise ValueError("subarray index out of range")

    @property
    def n_antennas(self) -> int:
        return self.n_subarrays * self.subarray_size

    @property
    def n_visible_antennas(self) -> int:
        return len(self.visible_subarrays) * self.subarray_size

    @cached_property
    def antenna_indices(self) -> np.ndarray:
        m = self.subarray_size
        return np.concatenate([np.arange(s * m, s * m + m) for s in sorted(self.visible_subarrays)])

    @cached_property
    def indicator(self) -> np.ndarray:
        mask = np.zeros(self.n_antennas)
        mask[self.antenna_indices] = 1.0
        return mask


def contiguous_region(start: int, length: int, n_antennas: int) -> VisibilityRegion:
    """A contiguous VR [start, start+length) on a 1-antenna subarray grid.

    This is how the BASELINE configs' arbitrarily aligned contiguous regions
    map exactly onto the reference's subarray model.
    """
    return VisibilityRegion(frozenset(range(start, start + length)), n_antennas, 1)


@dataclass(frozen=True)
class ChannelMatrix:
    """Column k = user k's masked channel (channel.py:228-250)."""

    h: np.ndarray
    vrs: tuple
    cfg: ArrayConfig

    @property
    def n_antennas(self) -> int:
        return self.h.shape[0]

    @property
    def n_users(self) -> int:
        return self.h.shape[1]


def _steering(angle: float, d0: float, cfg: ArrayConfig) -> np.ndarray:
    """Spherical steering vector, exact law-of-cosines distances (channel.py:73-131)."""
    n = cfg.n_antennas
    pos = np.arange(n, dtype=np.float64) - (n - 1) / 2.0
    d = cfg.spacing
    dist = np.sqrt(d0 * d0 + (pos * d) ** 2 - 2.0 * pos * d * d0 * math.cos(angle))
    phase = -2.0 * math.pi / cfg.wavelength * (dist - d0)
    return np.exp(1j * phase) / math.sqrt(n)


def random_channel(cfg: ArrayConfig, n_users: int, n_paths: int, p_visible: float,
                   rng: np.random.Generator, min_distance: float = 1.0,
                   max_distance: float = 50.0, angle_lo: float = math.pi / 6,
                   angle_hi: float = 5 * math.pi / 6) -> ChannelMatrix:
    """User drops + multipath + Bernoulli subarray VRs, in the reference's draw order.

    Draw order per user (channel.py:263-285): for each path angle, distance,
    two standard normals for the gain; then the VR mask redrawn until
    non-empty (channel.py:175-191).  Column = sqrt(Nt/L) * sum gain*steering,
    masked (channel.py:206-224, 252-260).
    """
    cols, vrs = [], []
    for _ in range(n_users):
        paths = []
        for _ in range(n_paths):
            angle = rng.uniform(angle_lo, angle_hi)
            dist = rng.uniform(min_distance, max_distance)
            gain = complex((rng.standard_normal() + 1j * rng.standard_normal()) / math.sqrt(2.0))
            paths.append((angle, dist, gain))
        while True:
            mask = rng.random(cfg.n_subarrays) < p_visible
            if mask.any():
                break
        vr = VisibilityRegion(frozenset(int(s) for s in np.flatnonzero(mask)),
                              cfg.n_subarrays, cfg.subarray_size)
        col = np.zeros(cfg.n_antennas, dtype=np.complex128)
        for angle, dist, gain in paths:
            col += gain * _steering(angle, dist, cfg)
        col = math.sqrt(cfg.n_antennas / len(paths)) * col
        cols.append(col * vr.indicator)
        vrs.append(vr)
    return ChannelMatrix(h=np.stack(cols, axis=1), vrs=tuple(vrs), cfg=cfg)


def power_control(chan: ChannelMatrix, snr_db: float):
    """Unit-norm columns, reg = 1/snr (channel.py:299-313)."""
    norms = np.linalg.norm(chan.h, axis=0)
    if np.any(norms == 0.0):
        raise ValueError("cannot power-control a user with an all-zero channel")
    snr_linear = 10.0 ** (snr_db / 10.0)
    return ChannelMatrix(h=chan.h / norms, vrs=chan.vrs, cfg=chan.cfg), 1.0 / snr_linear


# --------------------------------------------------------------------------
# vrgraph.py — overlap graph, min-degree greedy MIS, coupled sets
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class UserPartition:
    """Orthogonal / non-orthogonal split + coupled sets (vrgraph.py:60-82)."""

    orthogonal: frozenset
    non_orthogonal: tuple
    coupled: tuple
    subarray_users: tuple

    @property
    def orthogonal_sorted(self) -> tuple:
        return tuple(sorted(self.orthogonal))


def build_partition(vrs) -> UserPartition:
    """vrgraph.py:31-56 (graph + greedy MIS) and :84-114 (partition)."""
    n = len(vrs)
    nbrs = [set() for _ in range(n)]
    for i in range(n):
        for j in range(i + 1, n):
            if vrs[i].visible_subarrays & vrs[j].visible_subarrays:
                nbrs[i].add(j)
                nbrs[j].add(i)
    alive = set(range(n))
    chosen = set()
    while alive:
        # smallest residual degree, ties by lowest index (vrgraph.py:52-55)
        v = min(alive, key=lambda u: (len(nbrs[u] & alive), u))
        chosen.add(v)
        alive -= nbrs[v] | {v}
    n_sub = vrs[0].n_subarrays if vrs else 0
    per_sub = [[] for _ in range(n_sub)]
    for k, vr in enumerate(vrs):
        for s in vr.visible_subarrays:
            per_sub[s].append(k)
    return UserPartition(
        orthogonal=frozenset(chosen),
        non_orthogonal=tuple(k for k in range(n) if k not in chosen),
        coupled=tuple(frozenset(nbrs[k]) | {k} for k in range(n)),
        subarray_users=tuple(tuple(sorted(u)) for u in per_sub),
    )


# --------------------------------------------------------------------------
# metrics.py — flop counter, NMSE, sum-rate
# --------------------------------------------------------------------------

CMUL, CADD = 6, 2  # metrics.py:21-22


class FlopCounter:
    """metrics.py:25-41."""

    __slots__ = ("total",)

    def __init__(self):
        self.total = 0

    def cmul(self, n):
        self.total += CMUL * n

    def cadd(self, n):
        self.total += CADD * n

    def real(self, n):
        self.total += n


def nmse(f, f_ref) -> float:
    """||F_ref - F||_F / ||F_ref||_F (metrics.py:44-51)."""
    f_ref = np.asarray(f_ref)
    den = np.linalg.norm(f_ref)
    if den == 0.0:
        raise ValueError("reference precoder has zero norm")
    return float(np.linalg.norm(f_ref - np.asarray(f)) / den)


def spectral_efficiency(h, f, snr_linear: float):
    """Per-user rates of Eq. (7) and their sum (metrics.py:54-78)."""
    h = np.asarray(h)
    f = np.asarray(f)
    if h.shape != f.shape:
        raise ValueError("shape mismatch")
    if snr_linear <= 0.0:
        raise ValueError("snr_linear must be positive")
    if np.linalg.norm(f) > 1.0 + 1e-9:
        raise ValueError("precoder violates the unit power budget")
    power = np.abs(h.conj().T @ f) ** 2
    signal = np.diag(power).copy()
    rates = np.log2(1.0 + signal / (power.sum(axis=1) - signal + 1.0 / snr_linear))
    return rates, float(rates.sum())


# --------------------------------------------------------------------------
# rzf.py / assembly.py — direct solve and F = H V
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Precoder:
    """rzf.py:19-29."""

    f: np.ndarray
    norm_factor: float
    scheme: str = ""


def _as_h(h):
    return h.h if isinstance(h, ChannelMatrix) or hasattr(h, "vrs") else np.asarray(h)


def auxiliary_matrix(h, reg: float) -> np.ndarray:
    """(H^H H + reg I)^{-1} by Cholesky on all K canonical rhs (rzf.py:38-66)."""
    h = _as_h(h)
    if reg < 0.0:
        raise ValueError("regularisation must be non-negative")
    k = h.shape[1]
    gram = h.conj().T @ h + reg * np.eye(k)
    cho = scipy.linalg.cho_factor(gram, lower=True)
    return scipy.linalg.cho_solve(cho, np.eye(k, dtype=np.complex128))


def _unit_power(raw, scheme):
    """assembly.py:51-56 / rzf.py:79-83."""
    nrm = float(np.linalg.norm(raw))
    if nrm == 0.0:
        raise ValueError("degenerate precoder")
    beta = 1.0 / nrm
    return Precoder(f=raw * beta, norm_factor=beta, scheme=scheme)


def rzf_precoder(h, reg: float) -> Precoder:
    """beta * H (H^H H + reg I)^{-1}, ||F||_F = 1 (rzf.py:69-83)."""
    h = _as_h(h)
    return _unit_power(h @ auxiliary_matrix(h, reg), "rzf")


def assemble_dense(chan, v, counter=None, scheme=""):
    """F = H V then normalise (assembly.py:59-71)."""
    h = _as_h(chan)
    nt, k = h.shape
    if counter is not None:
        counter.cmul(nt * k * k)
        counter.cadd(nt * k * (k - 1))
    return _unit_power(h @ np.asarray(v), scheme)


def assemble_vr(chan, v, counter=None, scheme=""):
    """Subarray-blocked F = [H_s]_{Q_s} [V]_{Q_s,:} (assembly.py:20-48, 74-92)."""
    h = chan.h
    k = h.shape[1]
    m = chan.cfg.subarray_size
    v = np.asarray(v)
    blocks = []
    for s in range(chan.cfg.n_subarrays):
        users = np.asarray(sorted(u for u, vr in enumerate(chan.vrs) if s in vr.visible_subarrays),
                           dtype=np.intp)
        blk = h[s * m:(s + 1) * m, :]
        if users.size == 0:
            blocks.append(np.zeros((m, k), dtype=np.complex128))
            continue
        blocks.append(blk[:, users] @ v[users, :])
        if counter is not None:
            counter.cmul(m * users.size * k)
            counter.cadd(m * (users.size - 1) * k)
    return _unit_power(np.vstack(blocks), scheme)


# --------------------------------------------------------------------------
# solvers.py — the row-action path
# --------------------------------------------------------------------------

SCHEMES = ("urk", "swor-erk", "gk", "grk", "vr-ogrk", "ahk", "vr-oahk")  # solvers.py:39
STOCHASTIC_SCHEMES = frozenset({"urk", "swor-erk", "grk", "vr-ogrk"})    # solvers.py:42
VR_SCHEMES = frozenset({"vr-ogrk", "vr-oahk"})                            # solvers.py:45


def canonical_scheme(name: str) -> str:
    """solvers.py:48-52."""
    low = name.strip().lower()
    if low not in SCHEMES:
        raise ValueError(f"unknown scheme {name!r}; expected one of {SCHEMES}")
    return low


@dataclass(frozen=True)
class AugmentedSystem:
    """Row energies, supports, restricted rows, H^H and partition (solvers.py:59-109)."""

    channel: ChannelMatrix
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
        supports, rows = [], []
        for k, vr in enumerate(chan.vrs):
            idx = vr.antenna_indices
            leak = np.delete(chan.h[:, k], idx)
            if leak.size and np.any(leak != 0.0):
                raise ValueError(f"column {k} is nonzero outside its visibility region")
            supports.append(idx)
            rows.append(np.ascontiguousarray(chan.h[idx, k]))
        energies = np.array([np.sum(np.abs(r) ** 2) for r in rows]) + reg
        if np.any(energies == 0.0):
            raise ValueError("zero-energy row: empty channel with reg = 0")
        return cls(channel=chan, reg=float(reg), row_energies=energies,
                   supports=tuple(supports), eff_rows=tuple(rows),
                   h_adj=np.ascontiguousarray(chan.h.conj().T),
                   partition=build_partition(chan.vrs))

    @property
    def n_users(self) -> int:
        return self.channel.h.shape[1]

    @property
    def n_antennas(self) -> int:
        return self.channel.h.shape[0]


@dataclass
class SolverState:
    """Per-rhs iterate (col, coef), stored residuals, counters (solvers.py:112-136)."""

    rhs: int
    col: np.ndarray
    coef: np.ndarray
    resid: np.ndarray
    counter: FlopCounter = field(default_factory=FlopCounter)
    iters: int = 0
    noop_steps: int = 0

    @classmethod
    def initial(cls, sys: AugmentedSystem, rhs: int, col_buffer=None) -> "SolverState":
        if not 0 <= rhs < sys.n_users:
            raise ValueError(f"rhs index {rhs} out of range")
        col = col_buffer if col_buffer is not None else np.zeros(sys.n_antennas, np.complex128)
        resid = np.zeros(sys.n_users, dtype=np.complex128)
        resid[rhs] = 1.0
        return cls(rhs=rhs, col=col, coef=np.zeros(sys.n_users, np.complex128), resid=resid)


def residual_refresh(st: SolverState, sys: AugmentedSystem, rows=None, use_vr=True) -> None:
    """r_i = s_i - h_i^H col - reg q_i, dense zgemv or per-row VR vdot (solvers.py:143-170)."""
    k, nt = sys.n_users, sys.n_antennas
    if rows is None and not use_vr:
        st.resid[:] = -(sys.h_adj @ st.col) - sys.reg * st.coef
        st.resid[st.rhs] += 1.0
        st.counter.cmul(k * nt)
        st.counter.cadd(k * (nt + 1))
        st.counter.real(2 * k)
        return
    for i in (range(k) if rows is None else rows):
        if use_vr:
            idx = sys.supports[i]
            dot = np.vdot(sys.eff_rows[i], st.col[idx])
            n = idx.size
        else:
            dot = np.vdot(sys.channel.h[:, i], st.col)
            n = nt
        st.resid[i] = (1.0 if i == st.rhs else 0.0) - dot - sys.reg * st.coef[i]
        st.counter.cmul(n)
        st.counter.cadd(n + 1)
        st.counter.real(2)


def rk_step(st: SolverState, sys: AugmentedSystem, i: int, use_vr=True) -> None:
    """gamma = r_i/e_i; col += gamma h_i; q_i += gamma; r_i := 0 (solvers.py:173-188)."""
    gamma = st.resid[i] / sys.row_energies[i]
    st.counter.real(2)
    if use_vr:
        idx = sys.supports[i]
        st.col[idx] += gamma * sys.eff_rows[i]
        n = idx.size
    else:
        st.col += gamma * sys.channel.h[:, i]
        n = sys.n_antennas
    st.coef[i] += gamma
    st.counter.cmul(n)
    st.counter.cadd(n + 1)
    st.resid[i] = 0.0
    st.iters += 1


@dataclass
class SelectionStrategy:
    """solvers.py:191-202."""

    variant: str
    pool: list = field(default_factory=list)

    def __post_init__(self):
        if self.variant not in ("uniform", "energy", "energy-swor", "greedy-max", "greedy-weighted"):
            raise ValueError(f"unknown selection variant {self.variant!r}")


def select_row(strategy: SelectionStrategy, st: SolverState, sys: AugmentedSystem, rng=None):
    """The five row rules; None when a greedy rule sees no residual (solvers.py:205-237)."""
    k = sys.n_users
    kind = strategy.variant
    if kind == "greedy-max":
        score = np.abs(st.resid) ** 2 / sys.row_energies
        st.counter.real(4 * k)
        return int(np.argmax(score)) if score.any() else None
    if rng is None:
        raise ValueError(f"selection variant {kind!r} needs an rng")
    if kind == "uniform":
        return int(rng.integers(k))
    if kind == "energy":
        w = sys.row_energies
        st.counter.real(k + 2)
        return int(rng.choice(k, p=w / w.sum()))
    if kind == "energy-swor":
        if not strategy.pool:
            strategy.pool = list(range(k))
        w = sys.row_energies[strategy.pool]
        st.counter.real(len(strategy.pool) + 2)
        return strategy.pool.pop(int(rng.choice(len(strategy.pool), p=w / w.sum())))
    w = np.abs(st.resid) ** 2
    st.counter.real(4 * k + 2)
    total = w.sum()
    if total == 0.0:
        return None
    return int(rng.choice(k, p=w / total))


@dataclass(frozen=True)
class AggregationWeights:
    """solvers.py:240-245."""

    phi: np.ndarray
    rows: np.ndarray


def aggregation_weights(st: SolverState, sys: AugmentedSystem, rows) -> AggregationWeights:
    """phi_i = r_i / e_i on sorted rows (solvers.py:248-254)."""
    rows = np.asarray(sorted(int(r) for r in rows), dtype=np.intp)
    phi = np.zeros(sys.n_users, dtype=np.complex128)
    phi[rows] = st.resid[rows] / sys.row_energies[rows]
    st.counter.real(2 * rows.size)
    return AggregationWeights(phi=phi, rows=rows)


def ahk_step(st: SolverState, sys: AugmentedSystem, w: AggregationWeights, use_vr=True,
             union=None) -> bool:
    """Projection onto the phi-aggregated hyperplane (solvers.py:257-309)."""
    rows = w.rows
    phi_r = w.phi[rows]
    m = rows.size
    if m == 0 or not phi_r.any():
        st.noop_steps += 1
        return False
    num = np.vdot(phi_r, st.resid[rows])
    st.counter.cmul(m)
    st.counter.cadd(max(m - 1, 0))
    nt = sys.n_antennas
    if use_vr:
        if union is None:
            union = np.unique(np.concatenate([sys.supports[i] for i in rows]))
        y = np.zeros(nt, dtype=np.complex128)
        for i in rows:  # scatter in ascending row order
            idx = sys.supports[i]
            y[idx] += w.phi[i] * sys.eff_rows[i]
            st.counter.cmul(idx.size)
            st.counter.cadd(idx.size)
        span = union
        span_size = span.size
    else:
        y = sys.channel.h[:, rows] @ phi_r
        st.counter.cmul(nt * m)
        st.counter.cadd(nt * max(m - 1, 0))
        span = None
        span_size = nt
    den = float(np.sum(np.abs(y) ** 2)) + sys.reg * float(np.sum(np.abs(phi_r) ** 2))
    st.counter.real(4 * span_size + 3 * m + 2)
    if den == 0.0:
        st.noop_steps += 1
        return False
    gamma = num / den
    st.counter.real(2)
    if span is None:
        st.col += gamma * y
    else:
        st.col[span] += gamma * y[span]
    st.counter.cmul(span_size)
    st.counter.cadd(span_size)
    st.coef[rows] += gamma * phi_r
    st.counter.cmul(m)
    st.counter.cadd(m)
    return True


def orthogonal_block_step(st: SolverState, sys: AugmentedSystem, rows, use_vr=True) -> None:
    """Simultaneous exact projections on pairwise-disjoint rows (solvers.py:312-332)."""
    for i in rows:
        phi = st.resid[i] / sys.row_energies[i]
        st.counter.real(2)
        if use_vr:
            idx = sys.supports[i]
            st.col[idx] += phi * sys.eff_rows[i]
            n = idx.size
        else:
            st.col += phi * sys.channel.h[:, i]
            n = sys.n_antennas
        st.coef[i] += phi
        st.counter.cmul(n)
        st.counter.cadd(n + 1)
        st.resid[i] = 0.0


class InstanceRun:
    """One rhs advanced one scheme iteration per `step()` (solvers.py:345-423).

    `rows_log` (oracle addition) records each projected row of the RK family.
    """

    def __init__(self, scheme, sys: AugmentedSystem, rhs: int, rng, col_buffer=None):
        self.scheme = canonical_scheme(scheme)
        if self.scheme in STOCHASTIC_SCHEMES and rng is None:
            raise ValueError(f"scheme {self.scheme!r} draws rows at random; pass an rng")
        self.sys, self.rng = sys, rng
        self.state = SolverState.initial(sys, rhs, col_buffer=col_buffer)
        self.done = False
        self.rows_log = []
        self.strategy = {
            "urk": "uniform", "swor-erk": "energy-swor", "gk": "greedy-max",
            "grk": "greedy-weighted", "vr-ogrk": "greedy-weighted",
        }.get(self.scheme)
        if self.strategy is not None:
            self.strategy = SelectionStrategy(self.strategy)
        part = sys.partition
        if self.scheme == "vr-ogrk":
            self.prev_row = None
            self.coupled = [np.asarray(sorted(c), dtype=np.intp) for c in part.coupled]
        if self.scheme == "vr-oahk":
            self.orth_rows = np.asarray(part.orthogonal_sorted, dtype=np.intp)
            self.non_rows = np.asarray(part.non_orthogonal, dtype=np.intp)
            self.non_union = (np.unique(np.concatenate([sys.supports[i] for i in self.non_rows]))
                              if self.non_rows.size else None)

    def step(self) -> None:
        if self.done:
            return
        st, sys, sc = self.state, self.sys, self.scheme
        if sc in ("urk", "swor-erk"):
            i = select_row(self.strategy, st, sys, self.rng)
            residual_refresh(st, sys, rows=(i,), use_vr=False)
            rk_step(st, sys, i, use_vr=False)
            self.rows_log.append(i)
        elif sc in ("gk", "grk"):
            residual_refresh(st, sys, use_vr=False)
            i = select_row(self.strategy, st, sys, self.rng)
            if i is None:
                self.done = True
                return
            rk_step(st, sys, i, use_vr=False)
            self.rows_log.append(i)
        elif sc == "vr-ogrk":
            if self.prev_row is not None:
                residual_refresh(st, sys, rows=self.coupled[self.prev_row], use_vr=True)
            i = select_row(self.strategy, st, sys, self.rng)
            if i is None:
                self.done = True
                return
            rk_step(st, sys, i, use_vr=True)
            self.prev_row = i
            self.rows_log.append(i)
        elif sc == "ahk":
            residual_refresh(st, sys, use_vr=False)
            w = aggregation_weights(st, sys, range(sys.n_users))
            if not ahk_step(st, sys, w, use_vr=False):
                self.done = True
                return
            st.iters += 1
        else:  # vr-oahk
            residual_refresh(st, sys, rows=self.orth_rows, use_vr=True)
            orthogonal_block_step(st, sys, self.orth_rows, use_vr=True)
            if self.non_rows.size:
                residual_refresh(st, sys, rows=self.non_rows, use_vr=True)
                w = aggregation_weights(st, sys, self.non_rows)
                ahk_step(st, sys, w, use_vr=True, union=self.non_union)
            st.iters += 1


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


@dataclass
class RunTrace:
    """metrics.py:227-240 (fields the solvers fill)."""

    scheme: str
    nmse: list = field(default_factory=list)
    resid: list = field(default_factory=list)
    flops: list = field(default_factory=list)
    n_iters: int = 0
    converged: bool = True
    flops_measured: int | None = None
    rows: list = field(default_factory=list)


def _true_residual_norm(st: SolverState, sys: AugmentedSystem) -> float:
    """solvers.py:453-457."""
    r = -(sys.h_adj @ st.col) - sys.reg * st.coef
    r[st.rhs] += 1.0
    return float(np.linalg.norm(r))


def solve(scheme, sys: AugmentedSystem, rhs: int, stop: StoppingRule, rng=None):
    """Single-rhs driver with oracle / residual stopping (solvers.py:460-507)."""
    scheme = canonical_scheme(scheme)
    if stop.mode == "oracle":
        if stop.reference is None:
            raise ValueError("oracle stopping needs the direct-solver reference column")
        ref = np.asarray(stop.reference)
        ref_norm = float(np.linalg.norm(ref))
        if ref_norm == 0.0:
            raise ValueError("oracle reference column is zero")
    cap = stop.max_iters if stop.max_iters is not None else 10_000 * sys.n_users
    run = InstanceRun(scheme, sys, rhs, rng)
    trace = RunTrace(scheme=scheme.upper())
    converged = False
    while True:
        run.step()
        if run.state.iters % stop.check_every == 0 or run.done:
            rn = _true_residual_norm(run.state, sys)
            trace.resid.append(rn)
            trace.flops.append(run.state.counter.total)
            if stop.mode == "oracle":
                err = float(np.linalg.norm(run.state.coef - ref)) / ref_norm
                trace.nmse.append(err)
                if err < stop.epsilon:
                    converged = True
                    break
            elif rn <= stop.epsilon:
                converged = True
                break
        if run.done:
            converged = True
            break
        if run.state.iters >= cap:
            break
    trace.n_iters = run.state.iters
    trace.converged = converged
    trace.flops_measured = run.state.counter.total
    trace.rows = run.rows_log
    return run.state, trace


def solve_all(scheme, sys: AugmentedSystem, stop: StoppingRule, rng=None, traces=None):
    """Per-column solves with rng.spawn(K) children (solvers.py:510-537).

    `traces` (oracle addition): optional list that receives each column's RunTrace.
    """
    scheme = canonical_scheme(scheme)
    k = sys.n_users
    kids = rng.spawn(k) if rng is not None else [None] * k
    ref = stop.reference
    if stop.mode == "oracle":
        ref = np.asarray(ref)
        if ref.shape != (k, k):
            raise ValueError(f"oracle reference must be (K, K), got {ref.shape}")
    v = np.empty((k, k), dtype=np.complex128)
    for c in range(k):
        rule = StoppingRule(mode=stop.mode, epsilon=stop.epsilon,
                            reference=ref[:, c] if stop.mode == "oracle" else None,
                            max_iters=stop.max_iters, check_every=stop.check_every)
        st, tr = solve(scheme, sys, c, rule, rng=kids[c])
        v[:, c] = st.coef
        if traces is not None:
            traces.append(tr)
    return v


@dataclass
class PrecodingRun:
    """solvers.py:540-553 (+ `rows`: per-rhs projected-row logs, oracle addition)."""

    scheme: str
    v: np.ndarray
    precoder: Precoder
    n_iters: int
    converged: bool
    nmse_trace: list
    resid_trace: list
    flops_trace: list
    flops_measured: int
    noop_steps: int
    rows: list = field(default_factory=list)
    iters: list = field(default_factory=list)


def run_precoding(scheme, sys: AugmentedSystem, reference, epsilon=1e-6, max_iters=None,
                  rng=None, traces=True) -> PrecodingRun:
    """Lockstep K-rhs driver with per-outer-iteration NMSE stop (solvers.py:556-623).

    `traces=False` (oracle addition) skips the per-iteration NMSE/residual
    instrumentation when epsilon == 0 (fixed-T mode), where it cannot change
    the outcome; used only to keep the CPU baseline honest about solver time.
    """
    scheme = canonical_scheme(scheme)
    k, nt = sys.n_users, sys.n_antennas
    f_ref = reference.f if hasattr(reference, "f") else np.asarray(reference)
    kids = rng.spawn(k) if rng is not None else [None] * k
    cols = np.zeros((nt, k), dtype=np.complex128, order="F")
    runs = [InstanceRun(scheme, sys, c, kids[c], col_buffer=cols[:, c]) for c in range(k)]
    setup = 4 * nt * k
    cap = max_iters if max_iters is not None else 10_000 * k
    nmse_tr, resid_tr, flops_tr = [], [], []
    eye = np.eye(k)
    converged = False
    t = 0
    instrument = traces or epsilon > 0.0
    while True:
        t += 1
        for run in runs:
            run.step()
        if instrument:
            mnorm = float(np.linalg.norm(cols))
            err = nmse(cols / mnorm if mnorm > 0.0 else cols, f_ref)
            coefs = np.stack([r.state.coef for r in runs], axis=1)
            r_full = eye - sys.h_adj @ cols - sys.reg * coefs
            nmse_tr.append(err)
            resid_tr.append(float(np.linalg.norm(r_full)))
            flops_tr.append(setup + sum(r.state.counter.total for r in runs))
            if err < epsilon:
                converged = True
                break
        if t >= cap or all(r.done for r in runs):
            break
    v = np.stack([r.state.coef for r in runs], axis=1)
    acc = FlopCounter()
    if scheme in VR_SCHEMES:
        prec = assemble_vr(sys.channel, v, counter=acc, scheme=scheme.upper())
    else:
        prec = assemble_dense(sys.channel, v, counter=acc, scheme=scheme.upper())
    return PrecodingRun(
        scheme=scheme.upper(), v=v, precoder=prec, n_iters=t, converged=converged,
        nmse_trace=nmse_tr, resid_trace=resid_tr, flops_trace=flops_tr,
        flops_measured=setup + sum(r.state.counter.total for r in runs) + acc.total,
        noop_steps=sum(r.state.noop_steps for r in runs),
        rows=[r.rows_log for r in runs], iters=[r.state.iters for r in runs],
    )


def flops_measured_for(run: PrecodingRun) -> int:
    return run.flops_measured
