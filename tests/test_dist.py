"""Multi-process (world_size 2, gloo, CPU) tests of the sharding + gather logic."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_02203_b200.parallel import gather_shards, shard_range, shard_size


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 5, 1760000, 1760001):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a0, a1), (b0, b1) in zip(ranges[:-1], ranges[1:]):
                assert a1 == b0 and a0 <= a1
            assert max(b - a for a, b in ranges) <= shard_size(n, world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = np.arange(n, dtype=np.float32) * 0.5 - 3.0          # "the field"
        v0, v1 = shard_range(n, rank, world)
        local = torch.from_numpy(full[v0:v1].copy())
        got = gather_shards(local, n)
        # 2-D payload (fp16 cube rows) too
        cube = np.stack([full, -full]).T.astype(np.float16)
        got2 = gather_shards(torch.from_numpy(cube[v0:v1].copy()), n)
        out_q.put((rank, bool(np.array_equal(got.numpy(), full)),
                   bool(np.array_equal(got2.numpy(), cube))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 1000, 4097])
def test_gather_world2_gloo(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok1 and ok2 for _, ok1, ok2 in res)


# ---------------------------------------------------------------------------
# the four sharded paths of parallel.py, world size 2 over gloo, with the oracle
# standing in for each rank's GPU compute (the bookkeeping -- ranges, V-slice windows
# and their sampling halo, the reference owner + broadcast, the cube column gather, the
# pair split -- is the code under test; every rank's window is the ONLY data its local
# compute may read)


def _paths_worker(rank, world, port, seed, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import ndf_oracle as O
    from paper_2307_02203_b200 import parallel as P
    from paper_2307_02203_b200 import workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        w = W.Workload("small", (11, 9, 5), 40, (3, 3, 1), 4, "fp32", "pearson",
                       ref_vertex=(5, 4, 2), seed=seed)
        f = W.generate_host(w)
        X = f.member_grids("v")                      # (M, nz, ny, nx)
        V = w.n_vertices
        model = W.build_model(w, seed=seed, grid_init=1.0)
        om = O.OracleModel(6, model.grid_mu, model.grid_nu, model.weights, model.biases,
                           model.spec.merge, model.spec.activation, model.spec.head_kind)
        ref = np.array([0.31, -0.77, 0.2])
        # (1) vertex-sharded query
        full = O.reconstruct_field(om, ref, w.dims)
        got = P.reconstruct_field_sharded(None, ref, "reference-is-mu", w.dims, _local=lambda a, b: (
            torch.from_numpy(O.reconstruct_field(om, ref, w.dims, vertices=np.arange(a, b)))))
        res["query"] = bool(np.array_equal(got.numpy(), full))
        # (2) multi-reference cube, columns gathered
        refs = np.random.default_rng(seed).uniform(-1, 1, (3, 3))
        cube = np.stack([O.reconstruct_field(om, r, w.dims) for r in refs]).astype(np.float16)
        got = P.reconstruct_multi_sharded(None, refs, "reference-is-mu", w.dims, _local=lambda a, b: (
            torch.from_numpy(np.stack([O.reconstruct_field(om, r, w.dims, vertices=np.arange(a, b))
                                       for r in refs]).astype(np.float16))))
        res["cube"] = bool(np.array_equal(got.numpy(), cube))
        # (3) V-sliced ground truth: the local compute sees only its window
        v0, v1, c0, c1 = P.window_for_rank(V, w.dims, rank, world)
        flat = X.reshape(X.shape[0], -1)
        masked = np.full_like(flat, np.nan)
        masked[:, c0:c1] = flat[:, c0:c1]
        masked = masked.reshape(X.shape)

        def local(a, b, vec):
            assert c0 <= a <= b <= c1
            r = O.pearson_against(vec.numpy(), flat[:, a:b].T.astype(np.float64))
            return torch.from_numpy(r.astype(np.float32))
        local.device = torch.device("cpu")

        def ref_vec(shape_only=False):
            if shape_only:
                return X.shape[0]
            v = O.sample_many(masked, ref.reshape(1, 3))[0]
            assert np.isfinite(v).all(), "reference corners outside the owner's window"
            return torch.from_numpy(v)
        want = O.pearson_against(O.sample_many(X, ref.reshape(1, 3))[0],
                                 flat.T.astype(np.float64)).astype(np.float32)
        got = P.ground_truth_field_sharded(None, None, "v", "v", ref, w.dims, _local=local,
                                           _ref_vec=ref_vec)
        res["gt"] = bool(np.array_equal(got.numpy(), want, equal_nan=True))
        res["owner"] = P.ref_owner(V, w.dims, ref, world)
        # (4) pair ranges
        pa, pb = W.pair_list(w, count=301, seed=seed)
        A = flat[:, pa].T.astype(np.float64)
        B = flat[:, pb].T.astype(np.float64)
        got = P.pair_estimators_sharded(None, "v", pa, pb, measures=("pearson",), _local=lambda a, b: {
            "pearson": torch.from_numpy(O.pearson_rowwise(A[a:b], B[a:b]))})
        res["pairs"] = bool(np.array_equal(got["pearson"].numpy(), O.pearson_rowwise(A, B),
                                           equal_nan=True))
        out_q.put((rank, res))
    except Exception as exc:          # report, do not hang the peer
        out_q.put((rank, {"error": repr(exc)}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed", [1, 7])
def test_sharded_paths_world2_gloo(seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_paths_worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert "error" not in res[r], res[r]
        assert all(res[r][k] for k in ("query", "cube", "gt", "pairs")), res[r]
    assert res[0]["owner"] == res[1]["owner"]


def test_window_halo_covers_every_lattice_cell():
    """For every lattice cell of a grid, the owner of its lower corner holds all 8 corners."""
    from paper_2307_02203_b200 import parallel as P
    dims = (7, 5, 4)
    V = 7 * 5 * 4
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 8):
        for pos in rng.uniform(-1.2, 1.2, (200, 3)):
            owner = P.ref_owner(V, dims, pos, world)
            _, _, c0, c1 = P.window_for_rank(V, dims, owner, world)
            c = P.lower_corner(pos, dims)
            corners = [c + dx + dims[0] * (dy + dims[1] * dz)
                       for dx in (0, 1) for dy in (0, 1) for dz in (0, 1)]
            assert c0 <= min(corners) and max(corners) < c1, (world, pos)
