"""decomp.SlabSimulation end to end with two real processes (world_size 2)
sharing one GPU over the gloo backend: the device trace planes travel
host-staged (decomp.exchange_planes_start), the wave-speed / count / totals
all-reduces run on device tensors.  No kernel of one rank waits on the other
(gloo is host-mediated), so two ranks on one device are safe.  Covers the
boundary-layer / interior predictor schedule that overlaps the halo swap
(SlabSimulation._predict_exchange) and the whole-slab schedule; the
assembled state and dt history must equal the single-domain run bitwise."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup(cells, degree):
    import paper_1808_03788_b200 as pkg

    d = len(cells)
    gmesh = pkg.CartesianMesh([(0.0, 2.0)] + [(0.0, 1.0)] * (d - 1), cells)
    system = pkg.make_system("euler", d)
    cfl = 0.9 / (d * (2 * degree + 1))
    ic, _ = pkg.build_problem("density_wave", system, velocity=[1.0, -0.5, 0.3][:d])
    return pkg, gmesh, system, cfl, ic


def _worker(rank, world, port, cells, degree, steps, overlap, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1808_03788_b200.decomp import SlabSimulation

        pkg, gmesh, system, cfl, ic = _setup(cells, degree)
        glob = pkg.Simulation(gmesh, system, degree, cfl)
        glob.project_initial_condition(ic)
        k = cells[0] // world
        sim = SlabSimulation(gmesh, system, degree, cfl, device=0)
        sim.overlap_halos = overlap
        sim.set_state(glob.u[rank * k:(rank + 1) * k].clone())
        del glob
        parts = []
        orig = sim._predict_part

        def counted(dt_dev, b, c):
            parts.append((b, c))
            orig(dt_dev, b, c)

        sim._predict_part = counted
        sim.run(np.inf, max_steps=steps)
        u = sim.u.cpu()
        gathered = [torch.empty_like(u) for _ in range(world)]
        dist.all_gather(gathered, u)
        dts = [h["dt"] for h in sim.history]
        totals = sim.history[-1]["totals"]
        q.put((rank, torch.cat(gathered).numpy() if rank == 0 else None, dts,
               np.asarray(totals), len(parts), sim._range_ok))
    except Exception as exc:  # surface the worker's failure in the parent
        q.put((rank, repr(exc), None, None, None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [True, False], ids=["overlap", "whole"])
@pytest.mark.parametrize("cells,degree", [((6, 3, 2), 3), ((8, 4), 4)])
def test_slab_simulation_two_ranks_gloo(cells, degree, overlap):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import sys
    sys.path.insert(0, ROOT)
    world, steps = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, cells, degree, steps, overlap, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(60)
    for r in res:
        assert r[2] is not None, f"rank {r[0]} failed: {r[1]}"
    _, u_slabs, dts, totals, nparts, range_ok = res[0]
    assert range_ok
    # 3 range launches per step when overlapping, none otherwise
    assert nparts == (3 * steps if overlap else 0)
    assert res[1][2] == dts   # every rank computed the same (global) dt

    pkg, gmesh, system, cfl, ic = _setup(cells, degree)
    ref = pkg.Simulation(gmesh, system, degree, cfl)
    ref.project_initial_condition(ic)
    ref.run(np.inf, max_steps=steps)
    assert dts == [h["dt"] for h in ref.history]
    np.testing.assert_array_equal(u_slabs, ref.u.cpu().numpy())
    # totals: SUM all-reduce of the per-slab partials (summation order differs)
    np.testing.assert_allclose(totals, ref.history[-1]["totals"], rtol=1e-13, atol=1e-15)
