"""Multi-GPU plumbing for the bound-propagation path: one process per GPU, independent sentences.

The ε search of one sentence never talks to another sentence, so the corpus is
sharded into contiguous, disjoint blocks of sentence ids per rank and there is no data-path
collective ("scaling": "weak").  torch.distributed (NCCL on GPUs, gloo in the CPU tests) is used
only for the barrier, the max-over-ranks of device times, and gathering per-sentence results.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Optional


@dataclass(frozen=True)
class RankInfo:
    rank: int
    world: int
    local_rank: int


def rank_info() -> RankInfo:
    """RANK / WORLD_SIZE / LOCAL_RANK as set by torchrun (defaults: single process)."""
    return RankInfo(int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
                    int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str = "nccl", device_index: Optional[int] = None):
    """Initialises torch.distributed when WORLD_SIZE > 1; returns the module or None."""
    info = rank_info()
    if info.world <= 1:
        return None
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        kw = {}
        if backend == "nccl" and device_index is not None:
            kw["device_id"] = torch.device("cuda", device_index)
        dist.init_process_group(backend=backend, **kw)
    return dist


def sentence_block(rank: int, step: int, steps_per_rank: int, batch: int) -> range:
    """Globally unique sentence ids of (rank, step): rank-major contiguous blocks."""
    base = (rank * steps_per_rank + step) * batch
    return range(base, base + batch)


def shard(n_items: int, rank: int, world: int) -> range:
    """Contiguous, balanced split of [0, n_items) over `world` ranks (first ranks get the remainder)."""
    q, r = divmod(n_items, world)
    start = rank * q + min(rank, r)
    return range(start, start + q + (1 if rank < r else 0))


def max_over_ranks(values, dist=None, device=None):
    """Element-wise max of a list of floats over ranks (identity for a single process)."""
    vals = [float(v) for v in values]
    if dist is None:
        return vals
    import torch
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def run_sharded(n_items: int, work: Callable[[range], list], dist=None) -> Optional[list]:
    """Runs `work` on this rank's shard of [0, n_items) and gathers all results on rank 0
    in item order (None on the other ranks)."""
    info = rank_info() if dist is not None else RankInfo(0, 1, 0)
    mine = work(shard(n_items, info.rank, info.world))
    if dist is None:
        return mine
    parts = [None] * info.world
    dist.all_gather_object(parts, mine)
    if info.rank != 0:
        return None
    out = []
    for p in parts:
        out.extend(p)
    return out
