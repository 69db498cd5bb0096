"""TEST INFRASTRUCTURE ONLY (the checker, never the product): CPU restatement of the BASELINE cfg3 variant of
VR-OAHK that the reference does not implement -- "orthogonal row groups built from disjoint VRs and an aggregation
of up to 8 hyperplanes per step" (BASELINE.json configs[2]).  Built from the reference's
own primitives as restated in oracle/kaczprec_port.py:

  partition   O_1 = the reference's min-degree greedy independent set of the VR overlap graph
              (vrgraph.py:43-56, 84-114); O_g = the same greedy on the graph induced by the rows not yet grouped,
              for g = 2..n_groups (indices mapped back, lowest-index ties as in the reference); N = the rest,
              ascending.  Each O_g is pairwise VR-disjoint, so its rows are mutually orthogonal.
  iteration   for each O_g in order: residual_refresh(O_g) + orthogonal_block_step(O_g)   (solvers.py:414-416)
              then N in consecutive ascending blocks of at most `agg_cap` rows, each:
              residual_refresh(block) + aggregation_weights(block) + ahk_step(block, union of the block supports)
              (solvers.py:417-421, 248-309; Eqs. 40-45 of PAPER.md:461-472 with V replaced by the block);
              iters += 1 once per iteration.
With n_groups = 1 and agg_cap >= |N| this is exactly the reference's vr-oahk (InstanceRun.step, solvers.py:414-421):
tests/test_oracle_golden.py checks that limit bitwise against the restated reference path.
"""

from __future__ import annotations

import numpy as np

from .kaczprec_port import (FlopCounter, PrecodingRun, SolverState, aggregation_weights, ahk_step, assemble_vr,
                            nmse, orthogonal_block_step, residual_refresh)


def _overlap_sets(vrs):
    n = len(vrs)
    nbrs = [set() for _ in range(n)]
    for i in range(n):
        for j in range(i + 1, n):
            if vrs[i].visible_subarrays & vrs[j].visible_subarrays:
                nbrs[i].add(j)
                nbrs[j].add(i)
    return nbrs


def _greedy_mis(nbrs, alive):
    """vrgraph.py:43-56 on the subgraph induced by `alive`: smallest residual degree, lowest index on ties."""
    alive = set(alive)
    chosen = set()
    while alive:
        v = min(alive, key=lambda u: (len(nbrs[u] & alive), u))
        chosen.add(v)
        alive -= nbrs[v] | {v}
    return chosen


def grouped_partition(vrs, n_groups: int):
    """(groups: list of ascending row tuples O_1..O_g, non: ascending tuple N)."""
    if n_groups < 1:
        raise ValueError("n_groups must be >= 1")
    nbrs = _overlap_sets(vrs)
    remaining = set(range(len(vrs)))
    groups = []
    for _ in range(n_groups):
        if not remaining:
            break
        o = _greedy_mis(nbrs, remaining)
        groups.append(tuple(sorted(o)))
        remaining -= o
    return groups, tuple(sorted(remaining))


def n_blocks(n_rows: int, agg_cap: int) -> int:
    return 0 if n_rows == 0 else -(-n_rows // agg_cap)


class GroupedRun:
    """One rhs of the grouped VR-OAHK variant, advanced one iteration per step() (InstanceRun's contract)."""

    def __init__(self, sys, rhs: int, groups, non, agg_cap: int, col_buffer=None):
        if agg_cap < 1:
            raise ValueError("agg_cap must be >= 1")
        self.sys = sys
        self.state = SolverState.initial(sys, rhs, col_buffer=col_buffer)
        self.done = False
        self.groups = [np.asarray(g, dtype=np.intp) for g in groups]
        non = np.asarray(non, dtype=np.intp)
        self.blocks = [non[s:s + agg_cap] for s in range(0, non.size, agg_cap)]
        self.unions = [np.unique(np.concatenate([sys.supports[i] for i in blk])) for blk in self.blocks]

    def step(self) -> None:
        st, sys = self.state, self.sys
        for g in self.groups:
            residual_refresh(st, sys, rows=g, use_vr=True)
            orthogonal_block_step(st, sys, g, use_vr=True)
        for blk, un in zip(self.blocks, self.unions):
            residual_refresh(st, sys, rows=blk, use_vr=True)
            w = aggregation_weights(st, sys, blk)
            ahk_step(st, sys, w, use_vr=True, union=un)
        st.iters += 1


def run_precoding_grouped(sys, reference, n_groups: int, agg_cap: int, max_iters: int) -> PrecodingRun:
    """Fixed-T lockstep run of the variant over all K rhs (run_precoding's fixed-T path, solvers.py:556-623 with
    epsilon = 0); the precoder is assembled per subarray as for the VR schemes (assembly.py:74-92)."""
    k, nt = sys.n_users, sys.n_antennas
    groups, non = grouped_partition(sys.channel.vrs, n_groups)
    cols = np.zeros((nt, k), dtype=np.complex128, order="F")
    runs = [GroupedRun(sys, c, groups, non, agg_cap, col_buffer=cols[:, c]) for c in range(k)]
    for _ in range(max_iters):
        for r in runs:
            r.step()
    v = np.stack([r.state.coef for r in runs], axis=1)
    acc = FlopCounter()
    prec = assemble_vr(sys.channel, v, counter=acc, scheme="VR-OAHK-G")
    f_ref = reference.f if hasattr(reference, "f") else np.asarray(reference)
    return PrecodingRun(
        scheme="VR-OAHK-G", v=v, precoder=prec, n_iters=max_iters, converged=False,
        nmse_trace=[nmse(prec.f, f_ref)], resid_trace=[], flops_trace=[],
        flops_measured=4 * nt * k + sum(r.state.counter.total for r in runs) + acc.total,
        noop_steps=sum(r.state.noop_steps for r in runs), rows=[[] for _ in runs],
        iters=[r.state.iters for r in runs])
