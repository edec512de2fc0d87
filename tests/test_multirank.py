"""World-size-2 CPU (gloo) tests of the N>1 host path: batch sharding and the
max/sum reduction bench.py uses (replicas, no data collective)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1311_5614_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = D.shard(11, rank, world)
    # per-rank "work": each rank solves its own problems (here: a deterministic stand-in)
    times = [1.0 + rank, float(len(mine)), float(sum(mine))]
    tmax, tsum, tmin = D.reduce_stats(times)
    q.put((rank, mine, tmax.tolist(), tsum.tolist(), tmin.tolist()))
    dist.destroy_process_group()


def test_shard_is_a_partition():
    for P in (1, 2, 3, 8):
        got = sorted(i for r in range(P) for i in D.shard(512, r, P))
        assert got == list(range(512))
        sizes = [len(D.shard(512, r, P)) for r in range(P)]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.shard(4, 2, 2)


def test_gloo_world2_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, m0, mx0, s0, n0), (r1, m1, mx1, s1, n1) = out
    assert sorted(m0 + m1) == list(range(11)) and not set(m0) & set(m1)
    assert mx0 == mx1 == [2.0, 6.0, 30.0]
    assert s0 == s1 == [3.0, 11.0, 55.0]
    assert n0 == n1 == [1.0, 5.0, 25.0]
