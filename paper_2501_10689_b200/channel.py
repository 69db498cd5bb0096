"""Seeded near-field channels for the BASELINE.json configurations (input generation).

The reference's own channel model (pkg/src/kaczprec/channel.py) draws
Bernoulli subarray visibility and multipath gains; the BASELINE configs
instead specify a line-of-sight spherical wavefront with amplitude
lambda/(4 pi r) masked to one contiguous visibility region at a random start.
Per SURVEY.md §9 the columns are normalised to unit norm (the reference's
power-control convention, channel.py:299-313) and the ridge weight is
xi = K / SNR_linear.  A contiguous VR [s, s+L) is represented exactly in the
reference model as VisibilityRegion(range(s, s+L)) on a one-antenna subarray
grid, which is what `to_reference_layout` produces.

Realization b uses numpy.random.default_rng(seed_b); the solver streams use
SeedSequence(entropy=seed_b, spawn_key=(1,)) as the reference harness does
(experiments.py:226-228).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SPEED_OF_LIGHT = 2.99792458e8


@dataclass(frozen=True)
class NearFieldConfig:
    name: str
    n_antennas: int
    n_users: int
    vr_len: tuple            # (lo, hi) inclusive; lo == hi for a fixed length
    carrier_freq: float = 30e9
    snr_db: float = 10.0
    r_min: float = 5.0
    r_max: float = 50.0
    theta_max_deg: float = 60.0
    n_subcarriers: int = 1   # > 1: wideband OFDM, one drop, one system per subcarrier
    bandwidth: float = 0.0
    schemes: tuple = ()
    n_iters: int = 0
    n_systems: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def wavelength(self) -> float:
        return SPEED_OF_LIGHT / self.carrier_freq

    @property
    def reg(self) -> float:
        return self.n_users / 10.0 ** (self.snr_db / 10.0)

    @property
    def snr_linear(self) -> float:
        return 10.0 ** (self.snr_db / 10.0)


CONFIGS = {
    "cfg1": NearFieldConfig("cfg1", 256, 16, (64, 64), schemes=("grk",), n_iters=50, n_systems=100),
    "cfg2": NearFieldConfig("cfg2", 512, 64, (128, 128),
                            schemes=("urk", "grk", "vr-ogrk", "ahk", "vr-oahk"), n_iters=200, n_systems=1024),
    "cfg3": NearFieldConfig("cfg3", 1024, 128, (128, 512), schemes=("vr-oahk",), n_iters=200, n_systems=4096),
    "cfg4": NearFieldConfig("cfg4", 4096, 256, (512, 512), schemes=("grk", "vr-oahk"), n_iters=0,
                            n_systems=16384, extra={"residual_tol": 1e-4}),
    "cfg5": NearFieldConfig("cfg5", 2048, 128, (512, 512), n_subcarriers=1024, bandwidth=400e6,
                            schemes=("ahk", "vr-oahk"), n_iters=100, n_systems=1024,
                            extra={"iter_sweep": (10, 20, 50, 100)}),
}


@dataclass
class ContiguousChannels:
    """B systems with one contiguous support per user, values packed per row.

    heff[row_val_ptr[b*K+i] : row_val_ptr[b*K+i+1]] = H_b[start[b,i] : start[b,i]+length[b,i], i]
    """

    n_antennas: int
    n_users: int
    start: np.ndarray        # (B, K) int32
    length: np.ndarray       # (B, K) int32
    heff: np.ndarray         # (n_val,) complex128
    row_val_ptr: np.ndarray  # (B*K+1,) int64
    reg: np.ndarray          # (B,) float64
    snr_linear: np.ndarray   # (B,) float64

    @property
    def n_systems(self) -> int:
        return self.start.shape[0]

    def dense(self, b: int) -> np.ndarray:
        """Dense (Nt, K) channel of system b (zeros off the VRs)."""
        k = self.n_users
        h = np.zeros((self.n_antennas, k), dtype=np.complex128)
        for i in range(k):
            r = b * k + i
            s, ln = int(self.start[b, i]), int(self.length[b, i])
            h[s:s + ln, i] = self.heff[self.row_val_ptr[r]:self.row_val_ptr[r + 1]]
        return h

    def subset(self, systems) -> "ContiguousChannels":
        systems = np.asarray(systems, dtype=np.int64)
        k = self.n_users
        rows = (systems[:, None] * k + np.arange(k)[None, :]).ravel()
        lens = (self.row_val_ptr[rows + 1] - self.row_val_ptr[rows])
        ptr = np.zeros(rows.size + 1, dtype=np.int64)
        np.cumsum(lens, out=ptr[1:])
        vals = np.concatenate([self.heff[self.row_val_ptr[r]:self.row_val_ptr[r + 1]] for r in rows])
        return ContiguousChannels(self.n_antennas, k, self.start[systems], self.length[systems], vals, ptr,
                                  self.reg[systems], self.snr_linear[systems])


def _user_drop(cfg: NearFieldConfig, rng: np.random.Generator):
    k, nt = cfg.n_users, cfg.n_antennas
    r0 = rng.uniform(cfg.r_min, cfg.r_max, k)
    theta = rng.uniform(-math.radians(cfg.theta_max_deg), math.radians(cfg.theta_max_deg), k)
    lo, hi = cfg.vr_len
    length = np.full(k, lo, dtype=np.int64) if lo == hi else rng.integers(lo, hi + 1, k)
    start = rng.integers(0, nt - length + 1)
    return r0, theta, start.astype(np.int64), length.astype(np.int64)


def _entries(cfg: NearFieldConfig, r0, theta, start, length, wavelength):
    """lambda/(4 pi r) exp(-j 2 pi r / lambda) on each user's VR, unit-norm per user."""
    nt = cfg.n_antennas
    d = cfg.wavelength / 2.0  # element spacing fixed by the carrier
    cols = []
    for i in range(r0.size):
        n = np.arange(start[i], start[i] + length[i], dtype=np.float64) - (nt - 1) / 2.0
        x = n * d
        axis_angle = math.pi / 2.0 - theta[i]
        r = np.sqrt(r0[i] * r0[i] + x * x - 2.0 * x * r0[i] * math.cos(axis_angle))
        h = wavelength / (4.0 * math.pi * r) * np.exp(-2j * math.pi * r / wavelength)
        cols.append(h / np.linalg.norm(h))
    return cols


def generate(cfg: NearFieldConfig | str, seeds) -> ContiguousChannels:
    """Channels for realizations `seeds` (narrowband) or, for a wideband config,
    all subcarriers of the single drop `seeds[0]` (one system per subcarrier)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    seeds = list(seeds)
    k = cfg.n_users
    starts, lens, vals = [], [], []
    if cfg.n_subcarriers > 1:
        r0, theta, start, length = _user_drop(cfg, np.random.default_rng(seeds[0]))
        m = cfg.n_subcarriers
        sc = seeds[1] if len(seeds) > 1 else range(m)
        for mi in sc:
            f = cfg.carrier_freq + (mi - (m - 1) / 2.0) * cfg.bandwidth / m
            vals.extend(_entries(cfg, r0, theta, start, length, SPEED_OF_LIGHT / f))
            starts.append(start)
            lens.append(length)
    else:
        for s in seeds:
            r0, theta, start, length = _user_drop(cfg, np.random.default_rng(s))
            vals.extend(_entries(cfg, r0, theta, start, length, cfg.wavelength))
            starts.append(start)
            lens.append(length)
    start = np.asarray(starts, dtype=np.int32)
    length = np.asarray(lens, dtype=np.int32)
    ptr = np.zeros(start.size + 1, dtype=np.int64)
    np.cumsum(length.ravel(), out=ptr[1:])
    b = start.shape[0]
    return ContiguousChannels(cfg.n_antennas, k, start, length, np.concatenate(vals), ptr,
                              np.full(b, cfg.reg), np.full(b, cfg.snr_linear))


@dataclass
class Drops:
    """User drops of B systems (the inputs of on-device channel synthesis):
    everything `generate` draws, without the channel entries."""

    n_antennas: int
    n_users: int
    r0: np.ndarray           # (B, K) float64 distance to the array centre (m)
    theta: np.ndarray        # (B, K) float64 angle from broadside (rad)
    start: np.ndarray        # (B, K) int32 first visible antenna
    length: np.ndarray       # (B, K) int32 VR length
    wavelength: np.ndarray   # (B,) float64 per system (subcarrier)
    element_spacing: float   # lambda_carrier / 2
    reg: np.ndarray          # (B,)
    snr_linear: np.ndarray   # (B,)

    @property
    def n_systems(self) -> int:
        return self.start.shape[0]


def generate_drops(cfg: NearFieldConfig | str, seeds) -> Drops:
    """The drops `generate(cfg, seeds)` uses, from the same seeded streams (same draw order)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    seeds = list(seeds)
    r0s, ths, starts, lens, lams = [], [], [], [], []
    if cfg.n_subcarriers > 1:
        r0, theta, start, length = _user_drop(cfg, np.random.default_rng(seeds[0]))
        m = cfg.n_subcarriers
        for mi in (seeds[1] if len(seeds) > 1 else range(m)):
            f = cfg.carrier_freq + (mi - (m - 1) / 2.0) * cfg.bandwidth / m
            r0s.append(r0); ths.append(theta); starts.append(start); lens.append(length)
            lams.append(SPEED_OF_LIGHT / f)
    else:
        for s in seeds:
            r0, theta, start, length = _user_drop(cfg, np.random.default_rng(s))
            r0s.append(r0); ths.append(theta); starts.append(start); lens.append(length)
            lams.append(cfg.wavelength)
    b = len(starts)
    return Drops(cfg.n_antennas, cfg.n_users, np.asarray(r0s, dtype=np.float64), np.asarray(ths, dtype=np.float64),
                 np.asarray(starts, dtype=np.int32), np.asarray(lens, dtype=np.int32),
                 np.asarray(lams, dtype=np.float64), cfg.wavelength / 2.0, np.full(b, cfg.reg),
                 np.full(b, cfg.snr_linear))


def solver_seed_sequence(seed: int) -> np.random.SeedSequence:
    """Solver RNG of realization `seed`, distinct from its channel draw (experiments.py:226-228)."""
    return np.random.SeedSequence(entropy=seed, spawn_key=(1,))
