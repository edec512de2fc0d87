"""Host-side slab plan of the partitioned solve, no GPU needed:
ibmg_slab_plan is the function every slab context uses to pick its rows and the
agglomeration level.  World-size-2 gloo test: each rank takes its own plan and
the ranks' rows tile every distributed level exactly (the N>1 host path)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1311_5614_b200 import ibmg


def check_plan(N, P, la, rows):
    nlev = rows.shape[1]
    assert nlev == int(np.log2(N // 4)) + 1
    for l in range(nlev):
        n = N >> l
        if l < la or l == 0:
            spans = sorted(tuple(rows[r, l]) for r in range(P))
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0  # contiguous, disjoint
            if l < la:
                h = n // P
                assert h % 32 == 0 and h >= 24  # tile-row parity, halo fits
        else:
            assert all(tuple(rows[r, l]) == (0, n) for r in range(P))


@pytest.mark.parametrize("N", [64, 256, 1024, 8192])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_plan_partitions_levels(N, P):
    la, rows = ibmg.slab_plan(N, P, min_rows=64, min_cells=0)
    check_plan(N, P, la, rows)
    if P == 1:
        assert la == 0


def test_plan_agglomeration_threshold():
    # agglomerate below 2^16 cells or 64 rows per GPU
    assert ibmg.slab_plan(8192, 8)[0] == 4      # 8192..1024 distributed; 512 x 64 rows < 2^16 cells
    assert ibmg.slab_plan(8192, 2)[0] == 5      # down to n = 512 (256 rows x 512 = 2^17 cells)
    assert ibmg.slab_plan(256, 2)[0] == 0       # C2: 128 x 256 < 2^16 cells: all agglomerated
    assert ibmg.slab_plan(256, 2, min_cells=0)[0] == 2
    assert ibmg.slab_plan(256, 2, min_rows=128, min_cells=0)[0] == 1
    with pytest.raises(ValueError):
        ibmg.slab_plan(256, 9)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    la, rows = ibmg.slab_plan(1024, world, min_rows=64, min_cells=0)
    mine = torch.tensor(rows[rank], dtype=torch.int64)
    got = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(got, mine)
    q.put((rank, la, np.stack([g.numpy() for g in got]).tolist()))
    dist.destroy_process_group()


def test_gloo_world2_slab_rows_tile_the_grid():
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
    (_, la0, rows0), (_, la1, rows1) = out
    assert la0 == la1 == 4 and rows0 == rows1
    check_plan(1024, 2, la0, np.array(rows0))
