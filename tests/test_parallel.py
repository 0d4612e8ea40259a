"""CPU: batch sharding + all-gather of the multi-GPU batched Pfaffian path
(world size 2, gloo).  The per-rank compute is the oracle here (CPU test);
on the GPU box it is the batched CUDA kernel."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2411_09859_b200.inputs import skew_lower
from paper_2411_09859_b200.parallel import pfaffian_batched_distributed, shard_range


def _oracle_compute(xs):
    out = [oracle.pfaffian_slog(*(lambda r: (r.tau, r.pivots))(oracle.ltlt_blk_piv(x, b=x.shape[0])), x.shape[0])
           for x in xs]
    return np.array([s for s, _ in out]), np.array([l for _, l in out])


def _make(i):
    return skew_lower(16, i)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, l = pfaffian_batched_distributed(11, _make, compute=_oracle_compute)
    q.put((rank, s, l))
    dist.destroy_process_group()


def test_shard_range_covers_batch():
    for batch in (0, 1, 7, 8192):
        for world in (1, 2, 3, 8):
            spans = [shard_range(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_two_rank_gloo_matches_single_process():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    ref_s, ref_l = _oracle_compute(np.stack([_make(i) for i in range(11)]))
    for _rank, s, l in res:
        assert np.array_equal(s, ref_s)
        assert np.allclose(l, ref_l, rtol=0, atol=0)
