"""Multi-rank host logic on CPU: gloo, world size 2 (the NCCL path on the GPU
box runs the same code).  Each rank builds its own contiguous shard of
realizations, computes per-system statistics and the final gather must
reproduce the single-process result in global order."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_10689_b200.shard import gather_stats, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _per_system_stats(seeds):
    import oracle as O
    import paper_2501_10689_b200 as kz
    from helpers import oracle_channel_contiguous
    ch = kz.generate("cfg1", seeds)
    host = kz.HostBatch.from_contiguous(ch)
    n_orth = np.diff(host.orth_ptr).astype(np.float64)
    energy = host.row_energy.reshape(len(seeds), -1).sum(axis=1)
    # a real (if small) per-system computation: oracle RZF sum-rate on the rank's own systems
    rate = []
    for b in range(len(seeds)):
        chan = oracle_channel_contiguous(ch, b)
        f = O.rzf_precoder(chan, float(ch.reg[b])).f
        rate.append(O.spectral_efficiency(chan.h, f, float(ch.snr_linear[b]))[1])
    return {"n_orth": torch.tensor(n_orth), "energy": torch.tensor(energy),
            "sum_rate": torch.tensor(np.asarray(rate)), "seed": torch.tensor(np.asarray(seeds, dtype=np.float64))}


def _worker(rank, world, port, n_total, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(n_total, rank, world)
    stats = _per_system_stats(list(range(lo, hi)))
    out = gather_stats(stats, n_total)
    if rank == 0:
        q.put({k: v.numpy() for k, v in out.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [6, 7])
def test_two_rank_gather_matches_single_process(n_total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = _per_system_stats(list(range(n_total)))
    for k, v in want.items():
        np.testing.assert_array_equal(got[k], v.numpy(), err_msg=k)


def test_shard_range_partitions():
    for n in (0, 1, 5, 16384):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
