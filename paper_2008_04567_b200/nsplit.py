"""N-split inference (BASELINE.json configs[4]: "ResNet-50 end-to-end
conv forward batch 256 split along N across 8xB200"): the batch is cut into contiguous shards, one
per rank; every rank holds the (replicated, inference-constant) weights and runs the convolutions
of its shard with plans built for the shard's batch. There is no collective in the data path; the
outputs stay sharded. A shard's result equals the same images' rows of a one-process run of the
whole batch when both use the same kernel configuration (the per-output reduction order does not
depend on where an image sits in the batch; tests/test_nsplit_gpu.py checks this bit for bit).
"""
from __future__ import annotations

import torch

from .conv import Conv2dPlan


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard of rank `rank`: (first image, image count). Sizes differ by at most one
    (the first n_total % world ranks get one more image); every image belongs to exactly one rank."""
    if world < 1 or not 0 <= rank < world or n_total < world:
        raise ValueError(f"cannot split N={n_total} over world={world} (rank {rank})")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def shard_batch(x: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """The rank's rows of a batch (leading dimension N), as a contiguous tensor."""
    s, c = shard_range(x.shape[0], rank, world)
    return x[s:s + c].contiguous()


def shard_plan(layer, rank: int, world: int, n_total: int | None = None, **plan_kw) -> Conv2dPlan:
    """A Conv2dPlan for this rank's shard of a layer whose batch is n_total (default layer.n)."""
    n_total = layer.n if n_total is None else n_total
    _, count = shard_range(n_total, rank, world)
    return Conv2dPlan(count, layer.c, layer.h, layer.w, layer.k, layer.r, layer.s, layer.stride, layer.pad,
                      layer.dil, layer.groups, **plan_kw)
