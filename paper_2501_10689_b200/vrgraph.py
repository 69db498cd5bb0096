"""User partition from visibility-region overlap (host input preparation).

Same result as the reference's `build_partition` (pkg/src/kaczprec/vrgraph.py:31-114):
overlap graph on users, maximal independent set by repeated minimum-residual-
degree removal with lowest-index tie-break (vrgraph.py:43-56), coupled sets
X_k = N(k) ∪ {k}, non-orthogonal users in ascending order.  The graph is built
from support intervals with vectorised numpy instead of pairwise set
intersections, so contiguous visibility regions cost O(K^2) comparisons.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class UserPartition:
    orthogonal: frozenset
    non_orthogonal: tuple
    coupled: tuple  # tuple of frozensets
    subarray_users: tuple = ()

    @property
    def n_users(self) -> int:
        return len(self.coupled)

    @property
    def orthogonal_sorted(self) -> tuple:
        return tuple(sorted(self.orthogonal))


def overlap_from_intervals(start: np.ndarray, length: np.ndarray) -> np.ndarray:
    """(K, K) bool adjacency of half-open intervals [start, start+length), no self loops."""
    s = np.asarray(start, dtype=np.int64)
    e = s + np.asarray(length, dtype=np.int64)
    adj = (s[:, None] < e[None, :]) & (s[None, :] < e[:, None])
    np.fill_diagonal(adj, False)
    return adj


def overlap_from_segments(segments) -> np.ndarray:
    """Adjacency for general supports given per user as lists of (start, length) runs."""
    k = len(segments)
    adj = np.zeros((k, k), dtype=bool)
    for i in range(k):
        for j in range(i + 1, k):
            hit = False
            for si, li in segments[i]:
                for sj, lj in segments[j]:
                    if si < sj + lj and sj < si + li:
                        hit = True
                        break
                if hit:
                    break
            adj[i, j] = adj[j, i] = hit
    return adj


def greedy_mis(adj: np.ndarray) -> np.ndarray:
    """Min-degree greedy maximal independent set (vrgraph.py:43-56); sorted indices."""
    k = adj.shape[0]
    alive = np.ones(k, dtype=bool)
    chosen = []
    idx = np.arange(k)
    while alive.any():
        deg = (adj & alive[None, :]).sum(axis=1)
        key = np.where(alive, deg * (k + 1) + idx, np.iinfo(np.int64).max)
        v = int(np.argmin(key))
        chosen.append(v)
        alive &= ~adj[v]
        alive[v] = False
    return np.asarray(sorted(chosen), dtype=np.int64)


def grouped_mis(adj: np.ndarray, n_groups: int) -> list:
    """Orthogonal row groups for the grouped VR-OAHK variant (BASELINE cfg3): O_1 = greedy_mis(adj), O_g = the same
    greedy on the subgraph induced by the rows not yet grouped (lowest original index on ties, since the induced
    subgraph keeps the ascending order).  Each group is pairwise VR-disjoint.  Returns ascending index arrays."""
    k = adj.shape[0]
    rem = np.arange(k)
    groups = []
    for _ in range(max(1, n_groups)):
        if rem.size == 0:
            break
        loc = greedy_mis(adj[np.ix_(rem, rem)])
        groups.append(rem[loc])
        rem = np.setdiff1d(rem, rem[loc])
    return groups


def partition_from_adjacency(adj: np.ndarray) -> UserPartition:
    k = adj.shape[0]
    orth = greedy_mis(adj)
    in_o = np.zeros(k, dtype=bool)
    in_o[orth] = True
    coupled = tuple(frozenset(np.flatnonzero(adj[i]).tolist()) | {i} for i in range(k))
    return UserPartition(orthogonal=frozenset(orth.tolist()),
                         non_orthogonal=tuple(np.flatnonzero(~in_o).tolist()),
                         coupled=coupled)


def build_partition(vrs) -> UserPartition:
    """Drop-in for kaczprec.vrgraph.build_partition on VisibilityRegion-like objects."""
    segs = []
    for vr in vrs:
        subs = sorted(vr.visible_subarrays)
        runs = []
        for s in subs:
            if runs and runs[-1][0] + runs[-1][1] == s:
                runs[-1][1] += 1
            else:
                runs.append([s, 1])
        segs.append([(a, b) for a, b in runs])
    adj = overlap_from_segments(segs)
    part = partition_from_adjacency(adj)
    n_sub = vrs[0].n_subarrays if vrs else 0
    per_sub = [[] for _ in range(n_sub)]
    for k, vr in enumerate(vrs):
        for s in vr.visible_subarrays:
            per_sub[s].append(k)
    return UserPartition(part.orthogonal, part.non_orthogonal, part.coupled,
                         tuple(tuple(sorted(u)) for u in per_sub))
