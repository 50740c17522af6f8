"""Multi-GPU plumbing for the bound-propagation path: one process per GPU.

Sentence sharding (c2-c4): the ε search of one sentence never talks to another sentence (SURVEY
§8(e)), so the corpus is sharded into contiguous, disjoint blocks of sentence ids per rank and
there is no data-path collective ("scaling": "weak").  torch.distributed (NCCL on GPUs, gloo in
the CPU tests) is used only for the barrier, the max-over-ranks of device times, and gathering
per-sentence results.

Column sharding (c5): the perturbation columns of every Λ are split over the ranks and the
library all-reduces the concretization partials with NCCL inside the pass
(fg_model_shard_nccl); torch.distributed only carries the 128-byte NCCL unique id.
`column_range` / `reduce_op` mirror the library's split and reduction (include/faith_gpu.h).
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


def column_range(pert_dim: int, rank: int, world: int) -> range:
    """Perturbation columns owned by `rank` in the column-sharded pass (faith_gpu.h: rank r owns
    [r*D/world, (r+1)*D/world); D must be a multiple of 4*world for float4 rows)."""
    if pert_dim % (4 * world):
        raise ValueError(f"pert_dim {pert_dim} is not a multiple of 4*world ({4 * world})")
    w = pert_dim // world
    return range(rank * w, (rank + 1) * w)


def reduce_op(norm: str) -> str:
    """All-reduce op of the concretization partials for perturbation norm p: the dual q-norm of
    a row split by columns is a SUM of |.| (q = l1, p = linf), a SUM of squares (q = l2) or a MAX
    of |.| (q = linf, p = l1)."""
    return {"linf": "sum", "l2": "sum", "l1": "max"}[norm]


def partial_norms(rows, norm: str):
    """Raw partial dual-norm of each row of `rows` [n, d_local] (before the l2 square root)."""
    import numpy as np
    a = np.abs(np.asarray(rows, dtype=np.float64))
    if norm == "linf":
        return a.sum(axis=-1)
    if norm == "l2":
        return (a * a).sum(axis=-1)
    return a.max(axis=-1, initial=0.0)


def finish_norms(partials, norm: str):
    import numpy as np
    return np.sqrt(partials) if norm == "l2" else partials


def shard_model_columns(model, dist=None):
    """Column-shards `model` (faith_gpu.Model) over the torch.distributed world with the
    library's NCCL exchange: rank 0 creates the NCCL unique id, every rank receives it through
    torch.distributed and joins the communicator.  Single process: world-size-1 communicator."""
    from paper_2209_12708_b200 import faith_gpu as F
    info = rank_info() if dist is not None else RankInfo(0, 1, 0)
    box = [F.nccl_unique_id() if info.rank == 0 else None]
    if dist is not None:
        dist.broadcast_object_list(box, src=0)
    model.shard_columns_nccl(info.rank, info.world, box[0])
    return info
