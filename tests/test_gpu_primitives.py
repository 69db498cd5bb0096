"""Per-call step primitives and InstanceRun (solvers.py:143-423) on the GPU against the oracle port.

The reference composes InstanceRun.step from residual_refresh / select_row / rk_step / aggregation_weights /
ahk_step / orthogonal_block_step; the GPU mirror composes the same calls over kz_residual_refresh,
kz_project_rows and kz_ahk_step.  complex128: col and coef within 1e-10 relative after every step (resid, a
difference of O(1) terms, within 1e-10 relative or 1e-13 absolute), identical
iteration / no-op counts, done flags and FlopCounter totals (the draws consume the same Generator).
Inputs: the reference test drop (Bernoulli subarray VRs: multi-segment supports) and a cfg1-shaped drop.
"""

import numpy as np
import pytest

import oracle as O
from helpers import load, oracle_channel_contiguous, oracle_channel_from_mask
from oracle.kaczprec_port import AggregationWeights as OAW

pytestmark = pytest.mark.gpu

REL = 1e-10


def _kz():
    import paper_2501_10689_b200 as kz
    return kz


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (n if n > 0 else 1.0)


def ref_system():
    z = load("ref_lockstep.npz")
    chan = oracle_channel_from_mask(z["h"], z["vr_mask"], z["n_subarrays"])
    return O.AugmentedSystem.from_channel(chan, float(z["reg"]))


def cfg1_system():
    kz = _kz()
    ch = kz.generate(kz.CONFIGS["cfg1"], [3])
    return O.AugmentedSystem.from_channel(oracle_channel_contiguous(ch, 0), float(ch.reg[0]))


def same_state(a, b):
    assert rel(a.col, b.col) <= REL
    assert rel(a.coef, b.coef) <= REL
    # r = s - H^H m - xi q cancels O(1) terms: near convergence compare it on the scale of those terms
    assert rel(a.resid, b.resid) <= REL or np.max(np.abs(a.resid - b.resid)) <= 1e-13
    assert a.iters == b.iters
    assert a.noop_steps == b.noop_steps
    assert a.counter.total == b.counter.total


@pytest.mark.parametrize("make", [ref_system, cfg1_system], ids=["ref-subarray", "cfg1-contiguous"])
@pytest.mark.parametrize("scheme", O.SCHEMES)
def test_instance_run_steps_match_oracle(scheme, make):
    kz = _kz()
    sys_ = make()
    k = sys_.n_users
    for rhs in (0, k - 1):
        a = O.InstanceRun(scheme, sys_, rhs, np.random.default_rng(11))
        b = kz.InstanceRun(scheme, sys_, rhs, np.random.default_rng(11))
        for _ in range(25):
            a.step()
            b.step()
            assert a.done == b.done
            same_state(b.state, a.state)
            if a.done:
                break


def test_residual_refresh_forms():
    kz = _kz()
    sys_ = ref_system()
    k = sys_.n_users
    rng = np.random.default_rng(5)
    for rows, use_vr in ((None, False), (None, True), ([2, 0], True), ([1, 3], False)):
        a = O.SolverState.initial(sys_, 1)
        a.col[:] = rng.standard_normal(sys_.n_antennas) + 1j * rng.standard_normal(sys_.n_antennas)
        a.coef[:] = rng.standard_normal(k) + 1j * rng.standard_normal(k)
        b = kz.SolverState(rhs=1, col=a.col.copy(), coef=a.coef.copy(), resid=a.resid.copy())
        O.residual_refresh(a, sys_, rows=rows, use_vr=use_vr)
        kz.residual_refresh(b, sys_, rows=rows, use_vr=use_vr)
        same_state(b, a)


def test_overlapping_block_is_applied_in_order():
    """orthogonal_block_step on rows whose supports overlap: the reference applies them one after another."""
    kz = _kz()
    sys_ = ref_system()
    rows = [0, 1, 2, 3]
    a = O.SolverState.initial(sys_, 2)
    O.residual_refresh(a, sys_)
    b = kz.SolverState(rhs=2, col=a.col.copy(), coef=a.coef.copy(), resid=a.resid.copy(),
                       counter=kz.FlopCounter(a.counter.total))
    O.orthogonal_block_step(a, sys_, rows)
    kz.orthogonal_block_step(b, sys_, rows)
    same_state(b, a)


def test_ahk_step_noops_and_forms():
    kz = _kz()
    sys_ = ref_system()
    k = sys_.n_users
    a = O.SolverState.initial(sys_, 0)
    b = kz.SolverState.initial(sys_, 0)
    # phi identically zero on the rows: no-op flag, state untouched
    wa = O.aggregation_weights(a, sys_, [1, 2])
    wb = kz.aggregation_weights(b, sys_, [1, 2])
    assert not O.ahk_step(a, sys_, wa)
    assert not kz.ahk_step(b, sys_, wb)
    same_state(b, a)
    # empty row set
    assert not kz.ahk_step(b, sys_, kz.AggregationWeights(phi=np.zeros(k, complex), rows=np.zeros(0, np.intp)))
    assert not O.ahk_step(a, sys_, OAW(phi=np.zeros(k, complex), rows=np.zeros(0, np.intp)))
    same_state(b, a)
    for use_vr in (True, False):
        O.residual_refresh(a, sys_, use_vr=False)
        kz.residual_refresh(b, sys_, use_vr=False)
        wa = O.aggregation_weights(a, sys_, range(k))
        wb = kz.aggregation_weights(b, sys_, range(k))
        assert O.ahk_step(a, sys_, wa, use_vr=use_vr)
        assert kz.ahk_step(b, sys_, wb, use_vr=use_vr)
        same_state(b, a)


@pytest.mark.parametrize("scheme", O.SCHEMES)
def test_solve_returns_the_reference_state(scheme):
    """solve() returns SolverState like the reference (solvers.py:460-507): col, coef, the stored residuals
    the scheme left (stale where the scheme does not refresh), iters, noop steps, flop total."""
    kz = _kz()
    sys_ = ref_system()
    vref = O.auxiliary_matrix(sys_.channel, sys_.reg)
    for mode in ("residual", "oracle"):
        kw = dict(epsilon=1e-8) if mode == "residual" else dict(epsilon=1e-6, reference=vref[:, 2])
        a, ta = O.solve(scheme, sys_, 2, O.StoppingRule(mode=mode, **kw), rng=np.random.default_rng(4))
        b, tb = kz.solve(scheme, sys_, 2, kz.StoppingRule(mode=mode, **kw), rng=np.random.default_rng(4))
        assert ta.n_iters == tb.n_iters and ta.converged == tb.converged
        same_state(b, a)


def test_integration_md_flow():
    """The INTEGRATION.md drop-in flow end to end (oracle channel objects stand in for kaczprec's)."""
    kz = _kz()
    cfg = O.ArrayConfig(256, 100e9, 16)
    chan, reg = O.power_control(O.random_channel(cfg, 16, 5, 0.35, np.random.default_rng(0)), 0.0)
    sys_ = kz.AugmentedSystem.from_channel(chan, reg)
    ref = kz.rzf_precoder(chan, reg)
    run = kz.run_precoding("vr-oahk", sys_, ref, epsilon=1e-6)
    assert run.converged and run.nmse_trace[-1] < 1e-6
    st, tr = kz.solve("gk", sys_, 0, kz.StoppingRule(mode="residual", epsilon=1e-8))
    assert tr.converged
    V = kz.solve_all("grk", sys_, kz.StoppingRule(mode="residual", epsilon=1e-8), rng=np.random.default_rng(7))
    f = kz.assemble_vr(kz.SubarrayChannel.from_channel(chan), V).f
    assert kz.nmse(f, ref.f) < 1e-6
    r = kz.InstanceRun("vr-oahk", sys_, rhs=0, rng=None)
    for _ in range(10):
        r.step()
    assert r.state.iters == 10
