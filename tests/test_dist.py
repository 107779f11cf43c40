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
