"""CPU: host logic of the block-cyclic multi-GPU driver (no device needed).

* the block-cyclic partition covers every column exactly once;
* the column-filtered GEMM's owned-tile tables (C ABI, host only) cover each
  lower tile column exactly as the owners' column sets do, with `partial`
  exactly on tiles that straddle an owner boundary;
* the ld padding keeps every block a whole number of VMM granules;
* world-size-2 gloo: partitions agree across ranks, and the SCM_RIGHTS fd
  exchange that carries the VMM handles delivers every peer's descriptors.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2411_09859_b200.dist import BlockCyclic, owner_table, padded_ld


@pytest.mark.parametrize("n,nbd,G", [(1, 1, 1), (1000, 128, 3), (49152, 512, 8), (777, 100, 4), (5, 64, 8)])
def test_block_cyclic_partition(n, nbd, G):
    bc = BlockCyclic(n, nbd, G)
    cols = np.concatenate([bc.columns_of(r) for r in range(G)])
    assert np.array_equal(np.sort(cols), np.arange(n))
    for r in range(G):
        assert all(bc.owner(c) == r for c in bc.columns_of(r)[:50])


@pytest.mark.parametrize("n,cbase,nbd,G", [(1000, 0, 128, 2), (900, 37, 100, 3), (4000, 1234, 512, 8),
                                           (130, 5, 64, 4), (49152 - 600, 600, 512, 8)])
def test_owner_tables_cover_lower_tiles(n, cbase, nbd, G):
    nt = (n + 127) // 128
    seen = np.zeros(nt, dtype=int)
    total = 0
    for r in range(G):
        tiles, rows = owner_table(n, cbase, nbd, G, r)
        first = 0
        for tj, f, part in rows:
            assert f == first
            first += nt - tj
            cols = np.arange(cbase + tj * 128, cbase + min(n, tj * 128 + 128))
            own = (cols // nbd) % G == r
            assert own.any() and bool(part) == (not own.all())
            seen[tj] += 1
        assert tiles == first
        total += tiles
    # every tile column is covered by each owner that has a column in it
    for tj in range(nt):
        cols = np.arange(cbase + tj * 128, cbase + min(n, tj * 128 + 128))
        assert seen[tj] == len(set(((cols // nbd) % G).tolist()))
    assert total >= nt * (nt + 1) // 2


def test_padded_ld():
    gran = 2 << 20
    for n, nbd in [(1000, 128), (49152, 512), (777, 100), (4096, 256)]:
        ld = padded_ld(n, nbd, gran)
        assert ld >= n and (nbd * ld * 8) % gran == 0 and ld - n < gran // np.gcd(gran, nbd * 8)


def _fd_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2411_09859_b200.dist import exchange_fds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fds = []
    for k in range(230):   # more than one SCM_RIGHTS message
        fd = os.memfd_create(f"r{rank}k{k}")
        os.write(fd, f"rank{rank}-blk{k}".encode())
        fds.append(fd)
    got = exchange_fds(fds, rank, world)
    seen = {}
    for peer, pfds in got.items():
        seen[peer] = [os.pread(f, 64, 0).decode() for f in pfds]
    parts = [None] * world
    bc = BlockCyclic(1000, 128, world)
    dist.all_gather_object(parts, bc.columns_of(rank).tolist())
    q.put((rank, seen, sorted(c for p in parts for c in p) == list(range(1000))))
    dist.destroy_process_group()


def test_two_rank_fd_exchange_and_partition():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fd_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, seen, cover in res:
        peer = 1 - rank
        assert seen == {peer: [f"rank{peer}-blk{k}" for k in range(230)]}
        assert cover
