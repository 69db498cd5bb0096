"""Race and memory checks of the on-chip kernels without compute-sanitizer (closed on this GPU pool):

* determinism: every fast path (wide register-resident kernel, warp-per-rhs RK kernel, chunked complex128 lockstep
  kernel, cluster kernel staged and streamed, generic kernel) run twice on the same inputs gives bitwise equal
  V, iteration and flop counters.  The kernels are atomic-free and reduce in fixed orders, so a shared-memory
  race (a partial read before its writer's barrier, a DSMEM inbox read before the cluster barrier, the TMEM
  park / reload of the aggregation schemes) shows up as run-to-run differences;
* bounds: tools/sanitize_cases.py (small invocations of every kernel) under the bounds-checked build
  (libkaczmarz_b200_checked.so, -DKZ_CHECKED: shared / DSMEM / TMEM / piece-list indices checked against their
  allocations, trap on violation) exits cleanly.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _kz():
    import paper_2501_10689_b200 as kz
    return kz


def _twice(dev, scheme, **kw):
    import torch
    kz = _kz()
    rng = ("philox", 11) if scheme in kz.STOCHASTIC_SCHEMES else None
    a = kz.solve_batch(dev, scheme, rng=rng, **kw)
    b = kz.solve_batch(dev, scheme, rng=rng, **kw)
    torch.cuda.synchronize()
    for name in ("v", "iters", "flops", "noop_steps"):
        x, y = getattr(a, name), getattr(b, name)
        assert torch.equal(x, y), (scheme, name)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_register_resident_kernels_are_deterministic(dtype):
    """cfg2 shape (wide kernel in c64: all seven schemes incl. the TMEM-parked aggregation; chunked lockstep and
    warp-per-rhs kernels in c128)."""
    kz = _kz()
    dev = kz.HostBatch.from_contiguous(kz.generate("cfg2", range(3))).to_device(dtype)
    for scheme in kz.SCHEMES:
        _twice(dev, scheme, mode="lockstep", max_iters=40)


@pytest.mark.parametrize("stream", ["0", "2"])
def test_cluster_kernel_is_deterministic(stream):
    """The cluster kernel (DSMEM inbox, owner pushes, cluster barriers) staged and streamed, fixed T and residual
    mode; run in a subprocess because the variant choice is read once per process (KZ_CLUSTER_STREAM)."""
    code = (
        "import paper_2501_10689_b200 as kz, torch\n"
        "ch = kz.generate(kz.NearFieldConfig('det', 2048, 64, (256, 256)), range(2))\n"
        "dev = kz.HostBatch.from_contiguous(ch).to_device('c64')\n"
        "for sc in ('gk', 'grk', 'vr-ogrk', 'ahk', 'vr-oahk'):\n"
        "    rng = ('philox', 5) if sc in kz.STOCHASTIC_SCHEMES else None\n"
        "    for kw in (dict(mode='lockstep', max_iters=30), dict(mode='residual', epsilon=1e-3, max_iters=5000)):\n"
        "        a = kz.solve_batch(dev, sc, rng=rng, **kw); b = kz.solve_batch(dev, sc, rng=rng, **kw)\n"
        "        torch.cuda.synchronize()\n"
        "        assert a.launches <= 3 and b.launches == a.launches\n"
        "        for n in ('v', 'iters', 'flops', 'noop_steps'):\n"
        "            assert torch.equal(getattr(a, n), getattr(b, n)), (sc, kw['mode'], n)\n"
        "print('ok')\n")
    env = dict(os.environ, KZ_CLUSTER_STREAM=stream)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


def test_bounds_checked_build_runs_every_kernel():
    """tools/sanitize_cases.py under libkaczmarz_b200_checked.so (built by __graft_entry__.build()); skipped only if
    the checked library was not built."""
    from paper_2501_10689_b200 import build as B
    if not os.path.exists(B.lib_path("checked")):
        pytest.skip("libkaczmarz_b200_checked.so not built (python -m paper_2501_10689_b200.build --checked)")
    env = dict(os.environ, KZ_LIB_VARIANT="checked")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert "[kz checked]" not in r.stdout + r.stderr
    for phase in ("wide / rkwarp / lockstep ok", "cluster ok", "rzf / epilogue ok", "drops ok", "generic ok"):
        assert phase in r.stdout


def test_cluster_rhs_grouping_is_bitwise_neutral():
    """Residual-mode greedy runs group a cluster's rhs by coupled-set size (KZ_CLUSTER_RHS_ORDER=1, the default);
    every rhs's arithmetic is unchanged, so V / iterations / flops equal the index-order run (=0) bit for bit."""
    code = (
        "import numpy as np, paper_2501_10689_b200 as kz, torch\n"
        "dev = kz.HostBatch.from_contiguous(kz.generate('cfg4', range(1))).to_device('c64')\n"
        "r = kz.solve_batch(dev, 'grk', mode='residual', epsilon=1e-4, max_iters=256 * 10000, rng=('philox', 9))\n"
        "np.savez(OUT, v=r.v.cpu().numpy(), it=r.iters.cpu().numpy(), fl=r.flops.cpu().numpy())\n")
    outs = []
    for order in ("0", "1"):
        path = f"/tmp/kz_rhs_order_{order}.npz"
        env = dict(os.environ, KZ_CLUSTER_RHS_ORDER=order)
        r = subprocess.run([sys.executable, "-c", code.replace("OUT", repr(path))], cwd=ROOT, env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        import numpy as np
        outs.append(np.load(path))
    for key in ("v", "it", "fl"):
        assert (outs[0][key] == outs[1][key]).all(), key


def test_cluster_rhs_grouping_ragged_rhs_count():
    """The grouped slot assignment with K not a multiple of the rhs per cluster (K = 40: a partly empty second
    cluster per system) and both greedy schemes that take it (gk, grk): bitwise equal to the index order."""
    code = (
        "import numpy as np, paper_2501_10689_b200 as kz, torch\n"
        "ch = kz.generate(kz.NearFieldConfig('rag', 1024, 40, (96, 400)), range(3))\n"
        "dev = kz.HostBatch.from_contiguous(ch).to_device('c64')\n"
        "out = {}\n"
        "for sc in ('gk', 'grk'):\n"
        "    rng = ('philox', 4) if sc == 'grk' else None\n"
        "    r = kz.solve_batch(dev, sc, mode='residual', epsilon=1e-4, max_iters=40 * 10000, rng=rng)\n"
        "    assert bool(r.converged.all())\n"
        "    out[sc + '_v'] = r.v.cpu().numpy(); out[sc + '_it'] = r.iters.cpu().numpy()\n"
        "np.savez(OUT, **out)\n")
    import numpy as np
    res = []
    for order in ("0", "1"):
        path = f"/tmp/kz_rhs_rag_{order}.npz"
        r = subprocess.run([sys.executable, "-c", code.replace("OUT", repr(path))], cwd=ROOT,
                           env=dict(os.environ, KZ_CLUSTER_RHS_ORDER=order), capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        res.append(np.load(path))
    for key in res[0].files:
        assert (res[0][key] == res[1][key]).all(), key
