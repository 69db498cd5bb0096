"""Batched Gram on the FP64 tensor cores (kz_dense.cuh kz_gram_tc_kernel, DMMA m8n8k4): the RZF Gram
H^H H + xi I (rzf.py:38-40) and the epilogue's G0 = H^H H for contiguous supports.

Checks: the RZF auxiliary matrix V = (H^H H + xi I)^{-1} and beta against the complex128 oracle
(oracle.auxiliary_matrix / rzf_precoder, themselves pinned to the reference) at 1e-10 for every BASELINE config
shape -- cfg2 (K = 64), a ragged K = 37 (the last 8-row block half empty), cfg3 (ragged VR lengths 128-512),
cfg4 (Nt = 4096, K = 256: 32 x 32 blocks, the kernel's maximum) and cfg5 subcarriers -- that the tensor-core
path ran (two launches: Gram + Gauss-Jordan), and the Gram-form epilogue (G0 from the tensor cores) against the
per-antenna epilogue on the same V (beta, NMSE, sum-rate to 1e-11).
"""

import dataclasses

import numpy as np
import pytest

import oracle as O
from helpers import oracle_channel_contiguous

pytestmark = pytest.mark.gpu


def _kz():
    import paper_2501_10689_b200 as kz
    return kz


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("cfg,systems", [("cfg2", range(4)), ("k37", range(3)), ("cfg3", range(2)),
                                         ("cfg4", range(1)), ("cfg5", range(2))])
def test_rzf_tensor_core_gram_matches_oracle(cfg, systems):
    kz = _kz()
    c = dataclasses.replace(kz.CONFIGS["cfg2"], name="k37", n_users=37) if cfg == "k37" else cfg
    ch = kz.generate(c, [0, systems] if cfg == "cfg5" else systems)  # cfg5: one drop, subcarriers
    dev = kz.HostBatch.from_contiguous(ch).to_device("c128")
    rz = kz.rzf_batched(dev)
    assert rz["launches"] == 2, rz["launches"]  # tensor-core Gram + blocked Gauss-Jordan
    v = rz["v"].cpu().numpy()
    beta = rz["beta"].cpu().numpy()
    for b in range(len(systems)):
        chan = oracle_channel_contiguous(ch, b)
        reg = float(ch.reg[b])
        vo = O.auxiliary_matrix(chan.h, reg)
        assert _rel(v[b], vo) <= 1e-10
        assert beta[b] == pytest.approx(O.rzf_precoder(chan.h, reg).norm_factor, rel=1e-10)


def test_rzf_tensor_core_gram_c64_inputs():
    """complex64 batches: the Gram of the fp32 rows in fp64 (products exact) -- V equals the complex128 batch's
    V built from the same fp32-rounded rows."""
    kz = _kz()
    ch = kz.generate("cfg2", range(3))
    host = kz.HostBatch.from_contiguous(ch)
    d64 = host.to_device("c64")
    rz = kz.rzf_batched(d64)
    v = rz["v"].cpu().numpy()
    for b in range(3):
        chan = oracle_channel_contiguous(ch, b)
        h32 = chan.h.astype(np.complex64).astype(np.complex128)
        assert _rel(v[b], O.auxiliary_matrix(h32, float(ch.reg[b]))) <= 1e-10


def test_epilogue_gram_form_with_tensor_core_g0():
    kz = _kz()
    ch = kz.generate("cfg2", range(6))
    dev = kz.HostBatch.from_contiguous(ch).to_device("c128")
    rz = kz.rzf_batched(dev)
    res = kz.solve_batch(dev, "grk", mode="lockstep", max_iters=10, rng=("philox", 5))  # NMSE ~1e-2, no floor
    g = kz.epilogue(dev, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True)
    a = kz.epilogue(dev, res.v, v_ref=rz["v"], beta_ref=rz["beta"], rates=True, want_f=True)
    assert g["gram_form"] and not a["gram_form"]
    assert g["launches"] == 2  # tensor-core G0 + the Gram-form epilogue
    assert np.all(g["nmse"].cpu().numpy() > 1e-4)
    for key in ("beta", "nmse", "sum_rate"):
        x, y = g[key].cpu().numpy(), a[key].cpu().numpy()
        np.testing.assert_allclose(x, y, rtol=1e-11, atol=0)
