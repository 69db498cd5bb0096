"""The INTEGRATION.md drop-in example end to end on a GPU (oracle channel objects stand in for kaczprec's):

    python tools/integration_example.py
"""
import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import oracle as O
import paper_2501_10689_b200 as kz
cfg = O.ArrayConfig(256, 100e9, 16)
chan, reg = O.power_control(O.random_channel(cfg, 16, 5, 0.35, np.random.default_rng(0)), 0.0)
sys_ = kz.AugmentedSystem.from_channel(chan, reg)
ref = kz.rzf_precoder(chan, reg)
run = kz.run_precoding("vr-oahk", sys_, ref, epsilon=1e-6)
st, tr = kz.solve("gk", sys_, 0, kz.StoppingRule(mode="residual", epsilon=1e-8))
V = kz.solve_all("grk", sys_, kz.StoppingRule(mode="residual", epsilon=1e-8), rng=np.random.default_rng(7))
f = kz.assemble_vr(kz.SubarrayChannel.from_channel(chan), V).f
print(run.n_iters, run.nmse_trace[-1], run.flops_measured, kz.nmse(f, ref.f), tr.n_iters, st.resid[:2])
r = kz.InstanceRun("vr-oahk", sys_, rhs=0, rng=None)
for _ in range(10): r.step()
st2 = kz.SolverState.initial(sys_, 3)
kz.residual_refresh(st2, sys_, use_vr=False)
i = kz.select_row(kz.SelectionStrategy("greedy-weighted"), st2, sys_, np.random.default_rng(1))
kz.rk_step(st2, sys_, i)
w = kz.aggregation_weights(st2, sys_, range(sys_.n_users))
kz.ahk_step(st2, sys_, w, use_vr=False)
kz.orthogonal_block_step(st2, sys_, sys_.partition.orthogonal_sorted)
print("instance run iters", r.state.iters, "step api ok", st2.iters, st2.counter.total)
