"""Slab decomposition on one GPU, sequentially (no cross-waiting kernels):
K slab Simulations exchange their x-trace planes by device copies and
combine their wave-speed records exactly as decomp.SlabSimulation does over
NCCL.  The assembled state must equal the single-domain run bitwise (same
per-element arithmetic, identical dt)."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _run_inprocess(pkg, gmesh, system, degree, cfl, u0, steps, nslabs, ranges=False):
    from paper_1808_03788_b200.decomp import local_mesh
    from paper_1808_03788_b200.driver import Simulation

    sims = []
    P = degree + 1
    for r in range(nslabs):
        mesh = local_mesh(gmesh, nslabs, r)
        blk = P ** mesh.dim * system.n_vars
        plane = int(np.prod(mesh.cells[1:])) * (blk + (blk & 1))
        ghost = {(0, 0): torch.empty(plane, dtype=torch.float64, device="cuda"),
                 (0, 1): torch.empty(plane, dtype=torch.float64, device="cuda")}
        sim = Simulation(mesh, system, degree, cfl, _ghost=ghost)
        k = mesh.cells[0]
        sim.set_state(u0[r * k:(r + 1) * k])   # the global projection, sliced
        sims.append(sim)
    m = system.n_vars
    dts = []
    for _ in range(steps):
        for sim in sims:
            if sim._red_cur is None:
                sim._wavespeed()
        reds = torch.stack([sim._buf.red[sim._red_cur] for sim in sims])
        comb = reds[0].clone()
        comb[0:3] = reds[:, 0:3].amax(dim=0)     # decomp.combine_reduce semantics
        comb[3:5] = reds[:, 3:5].sum(dim=0)
        rows = []
        for sim in sims:
            sim._buf.red[sim._red_cur].copy_(comb)
            row = torch.zeros(2 + m, dtype=torch.float64, device="cuda")
            st = torch.zeros(1, dtype=torch.int32, device="cuda")
            sim._timestep_into(row[0:1], st, math.inf)
            if ranges:
                # SlabSimulation._predict_exchange's overlap schedule: first and
                # last x-layer, then the interior (adg_predict_range)
                E = sim.mesh.n_elements
                layer = E // sim.mesh.cells[0]
                sim._predict_part(row[0:1], 0, layer)
                sim._predict_part(row[0:1], E - layer, layer)
                sim._predict_part(row[0:1], layer, E - 2 * layer)
            else:
                sim._predict(row[0:1])
            rows.append(row)
        for r, sim in enumerate(sims):
            n = sim._ghost[(0, 0)].numel()
            face = sim.mesh.n_elements * sim._buf.tb
            lo = sim._buf.traces[0:n]
            hi = sim._buf.traces[2 * face - n:2 * face]
            sims[(r - 1) % nslabs]._ghost[(0, 1)].copy_(lo)
            sims[(r + 1) % nslabs]._ghost[(0, 0)].copy_(hi)
        for sim, row in zip(sims, rows):
            sim._faces()
            nxt = sim._update(row[0:1], None)
            sim._u, sim._u_next = sim._u_next, sim._u
            sim._red_cur = nxt
        dts.append(float(rows[0][0].item()))
    return torch.cat([s.u for s in sims], dim=0), dts


@pytest.mark.parametrize("ranges", [False, True], ids=["whole", "ranges"])
@pytest.mark.parametrize("nslabs,cells,degree", [(2, (6, 3, 2), 3), (4, (12, 2, 2), 4),
                                                 (2, (6, 4), 5)])
def test_slabs_equal_single_domain(nslabs, cells, degree, ranges):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1808_03788_b200 as pkg

    d = len(cells)
    gmesh = pkg.CartesianMesh([(0.0, float(nslabs))] + [(0.0, 1.0)] * (d - 1), cells)
    system = pkg.make_system("euler", d)
    cfl = 0.9 / (d * (2 * degree + 1))
    ic, _ = pkg.build_problem("density_wave", system, velocity=[1.0, -0.5, 0.3][:d])
    ref = pkg.Simulation(gmesh, system, degree, cfl)
    ref.project_initial_condition(ic)
    u0 = ref.u.clone()
    ref.run(np.inf, max_steps=3)
    u, dts = _run_inprocess(pkg, gmesh, system, degree, cfl, u0, 3, nslabs, ranges)
    np.testing.assert_array_equal(dts, [h["dt"] for h in ref.history])
    assert torch.equal(u, ref.u)


@pytest.mark.parametrize("cells,degree,mode", [((5, 4, 3), 4, "conservative"),
                                               ((4, 3, 3), 2, "primitive"),
                                               ((7, 5), 3, "conservative"),
                                               ((9,), 5, "conservative")])
def test_predict_range_bitwise(cells, degree, mode):
    """adg_predict_range over a split of the elements == one adg_predict."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1808_03788_b200 as pkg

    d = len(cells)
    mesh = pkg.CartesianMesh([(0.0, 1.0)] * d, cells)
    system = pkg.make_system("euler", d)
    sim = pkg.Simulation(mesh, system, degree, 0.9 / (d * (2 * degree + 1)),
                         predictor_mode=mode)
    sim.project_initial_condition(pkg.build_problem("density_wave", system)[0])
    dt = torch.tensor([sim.max_timestep()], dtype=torch.float64, device=sim.device)
    sim._ensure_buffers()
    buf = sim._buf

    def poison():
        # a sentinel both runs start from (entries a range misses show up)
        for x in (buf.vol, buf.traces):
            x.fill_(12345.0)
        buf.pred_bad.fill_(7)
        buf.sweeps.fill_(-1)

    poison()
    sim._predict(dt)
    want = [x.clone() for x in (buf.vol, buf.traces, buf.pred_bad, buf.sweeps)]
    poison()
    E = mesh.n_elements
    cuts = [0, 1, E // 3, E // 3, E - 2, E]   # includes an empty range
    for b, c in zip(cuts[:-1], cuts[1:]):
        sim._predict_part(dt, b, c - b)
    got = [buf.vol, buf.traces, buf.pred_bad, buf.sweeps]
    # the trace blocks' padding double carries whatever the staged bulk copy
    # held: compare the P^d m values of every block
    blk = (degree + 1) ** d * (d + 2)
    want[1] = want[1].view(-1, buf.tb)[:, :blk]
    got[1] = got[1].view(-1, buf.tb)[:, :blk]
    for w, g in zip(want, got):
        assert torch.equal(w, g)


def test_predict_range_errors():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1808_03788_b200 as pkg

    mesh = pkg.CartesianMesh([(0.0, 1.0)] * 3, (2, 2, 2))
    system = pkg.make_system("euler", 3)
    sim = pkg.Simulation(mesh, system, 4, 0.9 / 27)
    sim.project_initial_condition(pkg.build_problem("density_wave", system)[0])
    dt = torch.tensor([1e-3], dtype=torch.float64, device=sim.device)
    sim._ensure_buffers()
    with pytest.raises(ValueError):
        sim._predict_part(dt, 4, 5)
    big = pkg.Simulation(mesh, system, 7, 0.9 / 45)   # 3-D N=7: slice-streaming kernel
    big.project_initial_condition(pkg.build_problem("density_wave", system)[0])
    big._ensure_buffers()
    with pytest.raises(NotImplementedError):
        big._predict_part(dt, 0, 8)


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("cells,degree,steps", [((8, 6, 5), 4, 4), ((6, 4, 4), 2, 3)])
def test_nccl_self_exchange_equals_single_domain(cells, degree, steps, overlap):
    """The C-ABI NCCL transport (adg_comm_init / adg_halo_exchange /
    adg_allreduce_reduce / adg_allreduce_sum) on a one-rank communicator: the
    x faces are cut and the rank swaps its own halo planes through NCCL
    (send to itself as the left and right neighbour), on a side stream when
    overlapped.  State, dt and totals equal the periodic single-domain run
    bitwise; the batched fast path replays CUDA graphs that contain the NCCL
    calls."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1808_03788_b200 as pkg
    from paper_1808_03788_b200.decomp import SlabSimulation

    gmesh = pkg.CartesianMesh([(0.0, 1.0)] * 3, cells)
    system = pkg.make_system("euler", 3)
    cfl = 0.9 / (3 * (2 * degree + 1))
    ic, _ = pkg.build_problem("density_wave", system, velocity=[1.0, -0.5, 0.3])
    ref = pkg.Simulation(gmesh, system, degree, cfl)
    ref.project_initial_condition(ic)
    ref.run(np.inf, max_steps=steps)
    sim = SlabSimulation(gmesh, system, degree, cfl, self_exchange=True)
    assert sim.transport == "adg" and sim._capturable
    sim.overlap_halos = overlap
    sim.project_initial_condition(ic)
    sim.run(np.inf, max_steps=steps)   # batched: graphs with the NCCL calls inside
    np.testing.assert_array_equal([h["dt"] for h in sim.history],
                                  [h["dt"] for h in ref.history])
    assert torch.equal(sim.u, ref.u)
    np.testing.assert_array_equal(np.array([h["totals"] for h in sim.history]),
                                  np.array([h["totals"] for h in ref.history]))
    sim.run(np.inf, max_steps=steps + 1, on_step=lambda s: None)   # eager path
    ref.run(np.inf, max_steps=steps + 1, on_step=lambda s: None)
    assert torch.equal(sim.u, ref.u)
