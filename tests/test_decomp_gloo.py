"""Multi-process (gloo, world_size 2, CPU) tests of the slab-decomposition
host logic: halo exchange planes and the wave-speed / count reduction."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1808_03788_b200.decomp import (combine_reduce, exchange_planes,
                                                  exchange_planes_start, exchange_planes_wait)

        n = 7
        send_lo = torch.full((n,), 100.0 * rank + 1.0, dtype=torch.float64)
        send_hi = torch.full((n,), 100.0 * rank + 2.0, dtype=torch.float64)
        recv_lo = torch.empty(n, dtype=torch.float64)
        recv_hi = torch.empty(n, dtype=torch.float64)
        exchange_planes(send_lo, send_hi, recv_lo, recv_hi)
        left, right = (rank - 1) % world, (rank + 1) % world
        ok_x = bool(torch.all(recv_lo == 100.0 * left + 2.0)) and \
            bool(torch.all(recv_hi == 100.0 * right + 1.0))
        # split form (SlabSimulation._predict_exchange): post, work, wait
        works = exchange_planes_start(send_lo * 3, send_hi * 3, recv_lo, recv_hi)
        busy = torch.arange(1000, dtype=torch.float64).sum()   # "interior" work
        exchange_planes_wait(works)
        ok_x = ok_x and float(busy) == 499500.0 and \
            bool(torch.all(recv_lo == 3 * (100.0 * left + 2.0))) and \
            bool(torch.all(recv_hi == 3 * (100.0 * right + 1.0)))
        # adg_reduce record: lam bits MAX, counts SUM
        lam = np.array([0.5 + rank, 3.0 - rank, 1.25], dtype=np.float64)
        red = torch.zeros(8, dtype=torch.int64)
        red[0:3] = torch.from_numpy(lam.view(np.int64).copy())
        red[3] = 10 + rank
        red[4] = rank
        combine_reduce(red)
        got = red[0:3].numpy().view(np.float64)
        ok_r = bool(np.all(got == np.array([0.5 + world - 1, 3.0, 1.25]))) and \
            int(red[3]) == sum(10 + r for r in range(world)) and \
            int(red[4]) == sum(range(world))
        q.put((rank, ok_x, ok_r))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slab_exchange_and_reduce_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(ok_x and ok_r for _, ok_x, ok_r in res), res


def test_slab_geometry():
    from paper_1808_03788_b200 import CartesianMesh
    from paper_1808_03788_b200.decomp import local_mesh, slab_bounds

    g = CartesianMesh([(0.0, 4.0), (0.0, 1.0), (0.0, 1.0)], (8, 2, 2))
    assert slab_bounds(8, 4, 2) == (4, 6)
    m = local_mesh(g, 4, 3)
    assert m.cells == (2, 2, 2) and m.extents[0] == (3.0, 4.0)
    assert m.spacings == g.spacings
    with pytest.raises(ValueError):
        slab_bounds(7, 2, 0)
