"""Cluster-kernel debugging: AHK iteration counts / noop steps on a large-array drop, c64 cluster vs
c64 generic (KZ_DISABLE_CLUSTER in a child process) vs c128."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2501_10689_b200 as kz  # noqa: E402


def run(dtype, scheme, T, cfg):
    ch = kz.generate(cfg, range(3))
    dev = kz.HostBatch.from_contiguous(ch).to_device(dtype)
    res = kz.solve_batch(dev, scheme, mode="lockstep", max_iters=T)
    return res.iters.cpu().numpy(), res.noop_steps.cpu().numpy(), res.v.cpu().numpy()


if __name__ == "__main__":
    cfg = kz.NearFieldConfig("t_large", int(os.environ.get("NT", 1024)), 40, (96, 400))
    scheme = os.environ.get("SCHEME", "ahk")
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        it, no, v = run("c64", scheme, 25, cfg)
        np.save("/tmp/child_v.npy", v)
        print("generic c64 iters", it[0].tolist(), "noop", no.sum())
        sys.exit(0)
    it, no, v = run("c64", scheme, 25, cfg)
    print("cluster c64 iters", it[0].tolist(), "noop", no.sum())
    env = dict(os.environ, KZ_DISABLE_CLUSTER="1")
    subprocess.run([sys.executable, __file__, "child"], env=env, check=True)
    vg = np.load("/tmp/child_v.npy")
    it2, no2, v2 = run("c128", scheme, 25, cfg)
    print("c128 iters", it2[0].tolist(), "noop", no2.sum())
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    print("rel cluster-c128", rel(v, v2), "generic64-c128", rel(vg, v2), "cluster-generic", rel(v, vg))
