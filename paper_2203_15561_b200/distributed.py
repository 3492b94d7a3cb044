"""Multi-GPU sharding across processes (one process per GPU, torchrun style).

The reference's only parallel construct is align_batch's process pool over
independent pairs (pkg/src/bitalign/window.py:152-163): results in input
order, identical at any degree.  Here each rank aligns a longest-first (LPT)
shard of the pairs on its own GPU -- there is no exchange on the data path --
and the per-slot outcomes are gathered to the destination rank(s) with one
object collective at the end, so the result is identical at any world size.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from ._abi import num_windows


def shard_indices(pattern_lens: Sequence[int] | np.ndarray, window: int, overlap: int,
                  world_size: int, rank: int) -> np.ndarray:
    """Pair indices owned by `rank`: greedy LPT over the exact per-pair cost
    proxy (#windows from |P| alone), deterministic on every rank."""
    if not 0 <= rank < world_size:
        raise ValueError(f"rank {rank} out of range for world size {world_size}")
    lens = np.asarray(pattern_lens, dtype=np.int64)
    cost = np.maximum(num_windows(lens, window, overlap).astype(np.int64), 1)
    order = np.argsort(-cost, kind="stable")
    loads = np.zeros(world_size, dtype=np.int64)
    owner = np.empty(lens.shape[0], dtype=np.int64)
    for idx in order:
        s = int(np.argmin(loads))
        owner[idx] = s
        loads[s] += int(cost[idx])
    return np.nonzero(owner == rank)[0]


def align_batch_distributed(pairs, cfg, *, aligner: Callable | None = None, dst: int | None = 0,
                            group=None):
    """align_batch over all ranks of the default (or given) process group.

    Every rank passes the same `pairs`; rank r aligns its LPT shard with
    `aligner(shard_pairs, cfg)` (default: the GPU align_batch on this rank's
    device) and the outcomes are gathered in input order to rank `dst`
    (None: to every rank).  Returns the full list where gathered, else None.
    """
    import torch.distributed as dist

    if aligner is None:
        from .window import align_batch as aligner  # noqa: N813
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lens = np.fromiter((len(p) for p, _ in pairs), dtype=np.int64, count=len(pairs))
    idx = shard_indices(lens, cfg.window, cfg.overlap, world, rank)
    mine = aligner([pairs[i] for i in idx.tolist()], cfg) if len(idx) else []
    payload = (idx.tolist(), mine)
    if dst is None:
        parts = [None] * world
        dist.all_gather_object(parts, payload, group=group)
    else:
        parts = [None] * world if rank == dst else None
        dist.gather_object(payload, parts, dst=dst, group=group)
        if rank != dst:
            return None
    out = [None] * len(pairs)
    for shard_idx, outcomes in parts:
        for i, o in zip(shard_idx, outcomes):
            out[i] = o
    return out
