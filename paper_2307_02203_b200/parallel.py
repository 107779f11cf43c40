"""Multi-GPU sharding: one process per GPU, vertex- or pair-range shards, NCCL gather.

Every workload on the hot path partitions into independent units (query
vertices, reference x vertex pairs, vertex pairs -- SURVEY.md 8(e)), so each
rank computes a contiguous range on its own GPU with no exchange during
compute; the only collective is the result assembly (an all-gather of equal,
padded shards -- NCCL over NVLink on the GPU box, gloo in the CPU tests).

The reference's only parallelism is a ProcessPoolExecutor over 4096-point
chunks for the MI ground truth (measures.py:303-310), bit-identical for any
``workers``; here too results do not depend on the number of ranks.
"""

from __future__ import annotations

import math

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple:
    """Contiguous range [v0, v1) of rank ``rank`` out of ``world`` (ceil split)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    shard = math.ceil(n / world) if n else 0
    v0 = min(n, rank * shard)
    return v0, min(n, v0 + shard)


def shard_size(n: int, world: int) -> int:
    return math.ceil(n / world) if n else 0


def gather_shards(local, n_total: int, group=None):
    """All-gather equal-size padded shards; returns the assembled (n_total, ...) tensor
    on every rank.  ``local`` holds this rank's [v0, v1) rows (may be shorter than
    the shard size on the last rank)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    shard = shard_size(n_total, world)
    pad = torch.zeros((shard,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((shard * world,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return out[:n_total]


def reconstruct_field_sharded(model, ref, role, dims, group=None):
    """reconstruct_field split over the ranks of ``group`` (one GPU each).

    Returns the full float32 field (CUDA tensor) on every rank; per-vertex
    arithmetic is independent of the split, so it equals the 1-GPU result bitwise.
    """
    import torch.distributed as dist
    from .service import reconstruct_field_device
    V = int(np.prod(dims))
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    v0, v1 = shard_range(V, rank, world)
    local = reconstruct_field_device(model, ref, role, dims, v0, v1)
    return gather_shards(local, V, group)


def ground_truth_field_sharded(field_obj, measure, var_mu, var_nu, ref, dims, group=None):
    """ground_truth_field_device split over the ranks of ``group``."""
    import torch.distributed as dist
    from .measures import ground_truth_field_device
    V = int(np.prod(dims))
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    v0, v1 = shard_range(V, rank, world)
    local = ground_truth_field_device(field_obj, measure, var_mu, var_nu, ref, dims, v0, v1)
    return gather_shards(local, V, group)
