"""A batch of independent queries over several GPUs.

A single traversal does not shard without a per-round label exchange, but a
batch of queries (configs 3 and 5) does: every rank — one process per GPU
under torch.distributed, each holding the whole graph (config 5: 7 GB of the
180 GB) — runs its share of the batch as one batched traversal on its own GPU
(replicas: no collective on the data path), and the labels are gathered on one
rank afterwards. Rank r takes queries r, r + W, r + 2W, ... so a batch sorted
by anything is split evenly.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np


def shard_of(k: int, rank: int, world: int) -> List[int]:
    """Query indices rank `rank` runs out of a batch of k (interleaved)."""
    return list(range(rank, k, world))


def sharded_query_batch(g, kind: str, vertices: Sequence[int], windows: Sequence,
                        group=None, dst: int = 0, ordering=None,
                        run: Optional[Callable] = None) -> Optional[np.ndarray]:
    """Runs `kind` for every (vertices[q], windows[q]) across the ranks of the
    default (or given) torch.distributed process group and returns the (k, n)
    int64 labels on rank `dst` (None on the other ranks) — the same array as
    query_batch(g, kind, vertices, windows) on one GPU.

    `run(vertices, windows) -> (len, n) int64` replaces the local batched
    traversal (tests of the sharding logic without a GPU)."""
    import torch
    import torch.distributed as dist

    from . import query_batch

    k = len(vertices)
    if len(windows) != k:
        raise ValueError("one window per query")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = shard_of(k, rank, world)
    if run is None:
        def run(vs, ws):
            return query_batch(g, kind, vs, ws, ordering=ordering)
    n = None
    local = run([vertices[q] for q in mine], [windows[q] for q in mine]) if mine else None
    if local is not None:
        n = local.shape[1]
    # every rank needs n and the padded row count for the gather
    n_t = torch.tensor([n if n is not None else -1], dtype=torch.int64)
    gather_dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    n_t = n_t.to(gather_dev)
    dist.all_reduce(n_t, op=dist.ReduceOp.MAX, group=group)
    n = int(n_t.item())
    rows = (k + world - 1) // world
    buf = np.zeros((rows, n), np.int64)
    if local is not None:
        buf[:len(mine)] = local
    t = torch.from_numpy(buf).to(gather_dev)
    parts = [torch.empty_like(t) for _ in range(world)] if rank == dst else None
    dist.gather(t, parts, dst=dst, group=group)
    if rank != dst:
        return None
    out = np.empty((k, n), np.int64)
    for r in range(world):
        idx = shard_of(k, r, world)
        if idx:
            out[idx] = parts[r].cpu().numpy()[:len(idx)]
    return out
