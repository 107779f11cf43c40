"""Multi-GPU sharding: one process per GPU, vertex- or pair-range shards, NCCL gather.

Every workload on the hot path partitions into independent units (query
vertices, reference x vertex pairs, vertex pairs -- SURVEY.md 8(e)), so each
rank computes a contiguous range on its own GPU with no exchange during
compute; the only collectives are the result assembly (an all-gather of equal,
padded shards -- NCCL over NVLink on the GPU box, gloo in the CPU tests) and,
for the V-sliced ground-truth field, one broadcast of the reference's member
vector (8 KB at M = 1000).

| path   | shard                    | resident per rank                   | collective      |
|----------------------|--------------------------|-------------------------------------|-----------------|
| NDF query (c1)       | vertex range             | model (weights, latent grid)        | all-gather      |
| multi-ref cube (c3)  | vertex range, all refs   | model                               | all-gather cube |
| GT Pearson / KSG     | vertex range             | its V-slice of X (+ sampling halo)  | bcast + gather  |
| bulk pairs (c4)      | pair range               | the whole variable (pairs roam)     | all-gather      |

The reference's only parallelism is a ProcessPoolExecutor over 4096-point
chunks for the MI ground truth (measures.py:303-310), bit-identical for any
``workers``; here too results do not depend on the number of ranks.  The local
compute of each path is a parameter (``_local``) so the CPU tests can drive the
same bookkeeping with an oracle stand-in over gloo (tests/test_dist.py).
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


def _rank_world(group):
    import torch.distributed as dist
    return dist.get_rank(group), dist.get_world_size(group)


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


def gather_columns(local, n_total: int, group=None):
    """All-gather a (rows, cols_r) block per rank split along its columns (the fp16
    cube of config 3: every rank holds all references x its vertex range) into the
    (rows, n_total) whole on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    shard = shard_size(n_total, world)
    rows = local.shape[0]
    pad = torch.zeros((rows, shard), dtype=local.dtype, device=local.device)
    pad[:, : local.shape[1]] = local
    out = torch.empty((world * rows, shard), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return out.view(world, rows, shard).permute(1, 0, 2).reshape(rows, world * shard)[:, :n_total]


def sampling_halo(dims) -> int:
    """Columns past a vertex range that trilinear sampling at a lattice cell whose lower
    corner lies in the range can touch: one z-plane, one x-row and one node."""
    nx, ny, _ = dims
    return nx * ny + nx + 1


def lower_corner(pos, dims) -> int:
    """Flat index of the lower lattice corner sample_many uses at ``pos``: the host twin
    of the device frac_index (ensemble.py:115-127, same fp64 operations)."""
    idx = []
    for p, n in zip(np.asarray(pos, dtype=np.float64).reshape(3), dims):
        u = (min(max(p, -1.0), 1.0) + 1.0) * 0.5 * (n - 1)
        idx.append(min(max(int(np.floor(u)), 0), n - 2))
    nx, ny, _ = dims
    return idx[0] + nx * (idx[1] + ny * idx[2])


def window_for_rank(V: int, dims, rank: int, world: int) -> tuple:
    """(v0, v1, c0, c1): the rank's vertex range and the column window it uploads
    (range + sampling halo, clipped to the grid)."""
    v0, v1 = shard_range(V, rank, world)
    c0 = min(v0, V - 1)                       # an empty tail rank keeps one column
    return v0, v1, c0, max(c0 + 1, min(V, v1 + sampling_halo(dims)))


def ref_owner(V: int, dims, pos, world: int) -> int:
    """The rank whose window holds all 8 lattice corners of ``pos``."""
    c = lower_corner(pos, dims)
    for r in range(world):
        v0, v1, c0, c1 = window_for_rank(V, dims, r, world)
        if c0 <= c < c1 and c + sampling_halo(dims) < c1:
            return r
    return world - 1


# ---------------------------------------------------------------------------
# the four sharded paths


def reconstruct_field_sharded(model, ref, role, dims, group=None, _local=None):
    """reconstruct_field split over the ranks of ``group`` (one GPU each).

    Returns the full float32 field on every rank; per-vertex arithmetic is
    independent of the split, so it equals the 1-GPU result bitwise."""
    V = int(np.prod(dims))
    rank, world = _rank_world(group)
    v0, v1 = shard_range(V, rank, world)
    if _local is None:
        from .service import reconstruct_field_device

        def _local(v0, v1):
            return reconstruct_field_device(model, ref, role, dims, v0, v1)
    return gather_shards(_local(v0, v1), V, group)


def reconstruct_multi_sharded(model, refs, role, dims, group=None, _local=None):
    """Config 3: the (n_ref, V) fp16 dependence cube, query vertices split over the
    ranks (every rank evaluates all references on its vertex range), assembled by one
    all-gather.  Rows equal the 1-GPU cube bitwise."""
    V = int(np.prod(dims))
    rank, world = _rank_world(group)
    v0, v1 = shard_range(V, rank, world)
    if _local is None:
        from .service import reconstruct_multi_device

        def _local(v0, v1):
            return reconstruct_multi_device(model, refs, role, dims, v0, v1)
    return gather_columns(_local(v0, v1), V, group)


def ground_truth_field_sharded(field_obj, measure, var_mu, var_nu, ref, dims, group=None,
                               _local=None, _ref_vec=None):
    """ground_truth_field_device split over the ranks of ``group``.

    Node-aligned fields of a host ensemble (this package's EnsembleField or the
    reference's) are V-sliced: each rank uploads only its vertex range of member
    columns plus the sampling halo (DeviceEnsemble.window: 0.88 GB instead of 7 GB
    per GPU for config 1 at 8 ranks), the rank whose window holds the reference's
    lattice corners samples its member vector and broadcasts it (fp64, M values), and
    every rank computes its range.  Other grids (sampling anywhere) or an ensemble
    already on the device run replicated over the same vertex split."""
    import torch
    import torch.distributed as dist
    V = int(np.prod(dims))
    rank, world = _rank_world(group)
    v0, v1, c0, c1 = window_for_rank(V, dims, rank, world)
    if _local is None:
        _local, _ref_vec = _gt_local_gpu(field_obj, measure, var_mu, var_nu, ref, dims, c0, c1)
    if _ref_vec is None:                      # replicated: every rank samples its own
        return gather_shards(_local(v0, v1, None), V, group)
    owner = ref_owner(V, dims, ref, world)
    vec = _ref_vec() if rank == owner else None
    if vec is None:
        M = _ref_vec(shape_only=True)
        vec = torch.empty(M, dtype=torch.float64, device=_local.device)
    src = dist.get_global_rank(group, owner) if group is not None else owner
    dist.broadcast(vec, src=src, group=group)
    return gather_shards(_local(v0, v1, vec), V, group)


def _gt_local_gpu(field_obj, measure, var_mu, var_nu, ref, dims, c0, c1):
    from .ensemble import DeviceEnsemble
    from .measures import ground_truth_field_device
    from . import _native as N
    node_aligned = (hasattr(field_obj, "domain") and hasattr(field_obj, "member_grids")
                    and tuple(dims) == (field_obj.domain.nx, field_obj.domain.ny,
                                        field_obj.domain.nz) and var_mu == var_nu)
    dev = N.require_cuda()
    if not node_aligned:
        def local(v0, v1, vec):
            return ground_truth_field_device(field_obj, measure, var_mu, var_nu, ref, dims, v0, v1)
        local.device = dev
        return local, None
    win = DeviceEnsemble.window(field_obj.member_grids(var_nu), c0, c1, dev)

    def local(v0, v1, vec):
        return ground_truth_field_device(win, measure, var_mu, var_nu, ref, dims, v0, v1,
                                         ref_vec=vec)
    local.device = dev

    def ref_vec(shape_only=False):
        if shape_only:
            return win.member_count
        return win.sample_many(np.asarray(ref, dtype=np.float64).reshape(1, 3))[0].contiguous()
    return local, ref_vec


def pair_estimators_sharded(field_obj, variable, pa, pb, k=8, measures=("pearson", "ksg_mi"),
                            group=None, _local=None):
    """Config 4: the pair list split into contiguous ranges over the ranks (the
    ensemble replicated on each -- pairs touch arbitrary vertices), each estimator's
    values all-gathered into the full (n,) fp64 result on every rank."""
    pa = np.asarray(pa, dtype=np.int64)
    pb = np.asarray(pb, dtype=np.int64)
    n = int(pa.size)
    rank, world = _rank_world(group)
    p0, p1 = shard_range(n, rank, world)
    if _local is None:
        from .measures import pair_estimators_device

        def _local(p0, p1):
            return pair_estimators_device(field_obj, variable, pa[p0:p1], pb[p0:p1], k, measures)
    res = _local(p0, p1)
    return {name: gather_shards(res[name], n, group) for name in measures}
