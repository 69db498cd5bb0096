import os, sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import numpy as np
import oracle as O
import paper_2501_10689_b200 as kz
from helpers import oracle_channel_contiguous

ch = kz.generate("cfg4", [0])
chan = oracle_channel_contiguous(ch, 0)
sys_ = O.AugmentedSystem.from_channel(chan, float(ch.reg[0]))
k = sys_.n_users
host = kz.HostBatch.from_systems([sys_])
dev = host.to_device("c128")
run = O.run_precoding("grk", sys_, O.rzf_precoder(chan, float(ch.reg[0])), epsilon=0.0, max_iters=8,
                      rng=np.random.default_rng(3), traces=False)
for chunk in (8, 64, 1024):
    streams = kz.HostStreams("grk", [np.random.default_rng(3).spawn(k)], host.row_energy.reshape(1, k))
    res = kz.solve_batch(dev, "grk", mode="lockstep", max_iters=8, rng=streams, rows_cap=8, chunk=chunk)
    rows = res.rows[0].cpu().numpy()
    bad = [c for c in range(k) if list(rows[c][rows[c] >= 0]) != run.rows[c]]
    print("chunk", chunk, "divergent", len(bad), "first", bad[:3], flush=True)
    if bad:
        c = bad[0]
        print("  gpu", list(rows[c]), "oracle", run.rows[c])
# dense refresh check: residuals after 1 step for rhs 0 from the GPU iterate vs oracle
streams = kz.HostStreams("grk", [np.random.default_rng(3).spawn(k)], host.row_energy.reshape(1, k))
res = kz.solve_batch(dev, "grk", mode="lockstep", max_iters=2, rng=streams, rows_cap=2, want_iterates=True)
m = res.iterates()[0].cpu().numpy()
q = res.v[0].cpu().numpy()
kids = np.random.default_rng(3).spawn(k)
for c in range(3):
    r_gpu = -(sys_.h_adj @ m[c]) - sys_.reg * q[:, c]
    r_gpu[c] += 1
    runc = O.InstanceRun("grk", sys_, c, kids[c])
    runc.step(); runc.step()
    st = runc.state
    r_or = -(sys_.h_adj @ st.col) - sys_.reg * st.coef
    r_or[c] += 1
    print(c, "col diff", np.linalg.norm(m[c] - st.col), "coef diff", np.linalg.norm(q[:, c] - st.coef), runc.rows_log)
