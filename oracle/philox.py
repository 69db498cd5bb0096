"""TEST INFRASTRUCTURE ONLY (the checker, never the product): a numpy restatement of the device's counter-based
row draws, so the oracle can be fed exactly the draws the throughput kernels consume.

The product's throughput mode (`rng=("philox", seed)`, KZ_RNG_PHILOX in include/kaczmarz_b200.h) draws on the
device with Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2, 3", SC'11; the published
round function and Weyl key schedule, restated from the paper, not from any library source):

  counter  = (draw & 0xffffffff, draw >> 32, rhs, system)     key = (seed & 0xffffffff, seed >> 32)
  round    : (hi0, lo0) = mulhilo(0xD2511F53, c0); (hi1, lo1) = mulhilo(0xCD9E8D57, c2)
             c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); k += (0x9E3779B9, 0xBB67AE85)
  10 rounds; uniform = ((o0 << 32 | o1) >> 11) * 2^-53  (53 random bits in [0, 1))

`system` is the GLOBAL realization index (kz_rng.system_base + local index), so draws do not depend on chunking
or sharding.  `PhiloxGenerator(seed, system)` is a numpy-Generator-shaped stand-in for the reference's `rng`
argument: `spawn(K)` gives one child per rhs (as `run_precoding` / `solve_all` do, solvers.py:520,573), and each
child's n-th draw is the device's draw n of that (system, rhs):

  child.random()            the uniform                        (grk / vr-ogrk via choice)
  child.choice(n, p=...)    numpy Generator.choice's algorithm on that uniform: cdf = cumsum(p), cdf /= cdf[-1],
                            searchsorted(cdf, u, side="right")  (checked against numpy itself in
                            tests/test_oracle_golden.py)
  child.integers(n)         floor(u * n) clamped to n - 1      (urk, the device's uniform row draw)
"""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr: np.ndarray, key0, key1) -> np.ndarray:
    """Philox4x32-10 of counters ctr (..., 4) uint32 under key (key0, key1) (scalars or arrays broadcasting
    against ctr[..., 0]); returns (..., 4) uint32."""
    c = [np.asarray(ctr[..., j], dtype=np.uint32).copy() for j in range(4)]
    k0 = np.asarray(key0, dtype=np.uint32).copy()
    k1 = np.asarray(key1, dtype=np.uint32).copy()
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = M0 * c[0].astype(np.uint64)
            p1 = M1 * c[2].astype(np.uint64)
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & _MASK32).astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & _MASK32).astype(np.uint32)
            c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
            k0 = k0 + W0
            k1 = k1 + W1
    return np.stack(c, axis=-1)


def philox_uniform(seed: int, system, rhs, draw) -> np.ndarray:
    """Device draw `draw` of (system, rhs) under `seed` (kz_common.cuh philox_uniform), broadcast over the
    index arrays; float64 in [0, 1)."""
    system, rhs, draw = np.broadcast_arrays(np.asarray(system, dtype=np.uint64), np.asarray(rhs, dtype=np.uint64),
                                            np.asarray(draw, dtype=np.uint64))
    ctr = np.stack([(draw & _MASK32).astype(np.uint32), (draw >> np.uint64(32)).astype(np.uint32),
                    rhs.astype(np.uint32), system.astype(np.uint32)], axis=-1)
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    o = philox4x32_10(ctr, seed & 0xFFFFFFFF, seed >> 32)
    bits = (o[..., 0].astype(np.uint64) << np.uint64(32) | o[..., 1].astype(np.uint64)) >> np.uint64(11)
    return bits.astype(np.float64) * (1.0 / 9007199254740992.0)


class PhiloxStream:
    """The draws of one (system, rhs), consumed in order (a Generator-shaped child)."""

    BLOCK = 256

    def __init__(self, seed: int, system: int, rhs: int):
        self.seed, self.system, self.rhs = int(seed), int(system), int(rhs)
        self.n = 0
        self._buf = np.empty(0)
        self._base = 0

    def _next(self) -> float:
        d = self.n
        if not (self._base <= d < self._base + self._buf.size):
            self._base = d
            self._buf = philox_uniform(self.seed, self.system, self.rhs, np.arange(d, d + self.BLOCK))
        self.n += 1
        return float(self._buf[d - self._base])

    def random(self, size=None):
        if size is None:
            return self._next()
        return np.array([self._next() for _ in range(int(np.prod(size)))]).reshape(size)

    def integers(self, n, size=None):
        def one():
            i = int(self._next() * n)
            return n - 1 if i >= n else i
        if size is None:
            return one()
        return np.array([one() for _ in range(int(np.prod(size)))]).reshape(size)

    def choice(self, n, p=None):
        if p is None:
            return self.integers(n)
        cdf = np.cumsum(np.asarray(p, dtype=np.float64))
        cdf /= cdf[-1]
        return int(np.searchsorted(cdf, self._next(), side="right"))


class PhiloxGenerator:
    """Parent stand-in for the `rng` of run_precoding / solve_all: spawn(K) -> one PhiloxStream per rhs."""

    def __init__(self, seed: int, system: int):
        self.seed, self.system = int(seed), int(system)

    def spawn(self, k: int):
        return [PhiloxStream(self.seed, self.system, c) for c in range(k)]
