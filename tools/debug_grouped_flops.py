import os, sys, subprocess, numpy as np
sys.path.insert(0, os.getcwd())
code = r'''
import numpy as np, torch, paper_2501_10689_b200 as kz
ch = kz.generate("cfg3", [6, 7])
host = kz.HostBatch.from_contiguous(ch, orth_groups=GROUPS, agg_cap=CAP)
for T in (3, 6):
    res = kz.solve_batch(host.to_device("c64"), "vr-oahk-g", mode="lockstep", max_iters=T)
    np.save(f"/tmp/fl_TAG_{T}.npy", res.flops.cpu().numpy()); np.save(f"/tmp/no_TAG_{T}.npy", res.noop_steps.cpu().numpy())
print("launches", res.launches)
'''
for tag, env in (("clu", {}), ("gen", {"KZ_DISABLE_CLUSTER": "1"})):
    c = code.replace("GROUPS", "4").replace("CAP", "8").replace("TAG", tag)
    r = subprocess.run([sys.executable, "-c", c], env=dict(os.environ, **env), capture_output=True, text=True)
    print(tag, r.stdout.strip(), r.stderr[-500:])
for T in (3, 6):
    a, b = np.load(f"/tmp/fl_clu_{T}.npy"), np.load(f"/tmp/fl_gen_{T}.npy")
    na, nb = np.load(f"/tmp/no_clu_{T}.npy"), np.load(f"/tmp/no_gen_{T}.npy")
    d = b - a
    print("T", T, "total diff", d.sum(), "rhs differing", np.count_nonzero(d), "unique diffs", np.unique(d)[:20], "noop diff", (nb - na).sum())
    print("  per system", d.sum(axis=1), "rows of first differing", np.argwhere(d != 0)[:5].tolist(), d[d != 0][:8])
