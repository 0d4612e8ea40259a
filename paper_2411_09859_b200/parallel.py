"""Multi-GPU partitioning for the paths that shard.

* Batched factorizations / Pfaffians (config 4) shard naturally: rank r of W
  owns the contiguous matrices [r*B/W, (r+1)*B/W) (per-matrix seeds stay the
  global indices), computes them on its own GPU with the batched kernel, and
  the per-matrix (sign, log|Pf|) are all-gathered -- no communication during
  compute.
* A single matrix of configs 2/3 is run as independent replicas (no
  collective); config 5's one large matrix uses the 1-D block-cyclic driver in
  dist.py (peer-mapped column blocks, one stream barrier per panel phase).

The compute function is injectable so the host logic can be tested on CPU
with the gloo backend.
"""

from __future__ import annotations

import numpy as np


def shard_range(batch, rank, world):
    """Contiguous near-equal slice [lo, hi) of `batch` items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = batch * rank // world
    hi = batch * (rank + 1) // world
    return lo, hi


def gpu_pfaffian_compute(xs):
    """Default per-rank compute: the batched CUDA kernel."""
    from .apps import pfaffian_batched
    return pfaffian_batched(xs)


def pfaffian_batched_distributed(batch, make_matrix, compute=gpu_pfaffian_compute, group=None):
    """(sign, log|Pf|) of `batch` matrices, sharded across the ranks of the
    default torch.distributed group; every rank returns the full arrays."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(batch, rank, world)
    if hi > lo:
        xs = np.stack([make_matrix(i) for i in range(lo, hi)])
        sign, logabs = compute(xs)
    else:
        sign, logabs = np.zeros(0), np.zeros(0)
    if world == 1:
        return np.asarray(sign, dtype=np.float64), np.asarray(logabs, dtype=np.float64)
    # pad to the largest shard, gather, then trim (shards differ by at most one)
    cap = max(shard_range(batch, r, world)[1] - shard_range(batch, r, world)[0] for r in range(world))
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    local = torch.zeros((2, cap), dtype=torch.float64, device=dev)
    local[0, : hi - lo] = torch.as_tensor(np.asarray(sign, dtype=np.float64))
    local[1, : hi - lo] = torch.as_tensor(np.asarray(logabs, dtype=np.float64))
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local, group=group)
    out_s, out_l = [], []
    for r in range(world):
        a, b = shard_range(batch, r, world)
        out_s.append(parts[r][0, : b - a].cpu().numpy())
        out_l.append(parts[r][1, : b - a].cpu().numpy())
    return np.concatenate(out_s), np.concatenate(out_l)
