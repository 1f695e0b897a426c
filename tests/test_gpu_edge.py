"""GPU edge cases against the CPU oracle: ragged / minimal grids, degrees 0-2,
1-D, the explicit advance/max_timestep API, finite t_end, error conventions,
force_limit_all and the dt-halving restart path."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def rel_linf(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1808_03788_b200 as p

    return p


def _pair(pkg, ext, cells, degree, cfl=None, bc="periodic", limiter=False, vel=None):
    from oracle import problems as oprob
    from oracle.euler import EulerOracle
    from oracle.sim import OracleMesh, OracleSimulation

    d = len(cells)
    cfl = cfl if cfl is not None else 0.9 / (d * (2 * degree + 1))
    vel = vel if vel is not None else [1.0, -0.5, 0.3][:d]
    osim = OracleSimulation(OracleMesh(ext, cells), EulerOracle(d), degree, cfl, boundary=bc,
                            use_limiter=limiter, per_element_picard=True)
    osim.project_initial_condition(oprob.density_wave(vel=vel)[0])
    system = pkg.make_system("euler", d)
    sim = pkg.Simulation(pkg.CartesianMesh(ext, cells), system, degree, cfl, boundary=bc,
                         use_limiter=limiter)
    sim.project_initial_condition(pkg.build_problem("density_wave", system, velocity=vel)[0])
    return sim, osim


@pytest.mark.parametrize("cells,degree", [((7,), 2), ((5,), 0), ((3, 1), 1), ((1, 1, 1), 3),
                                          ((3, 2, 1), 1), ((2, 3), 0), ((1, 2, 3), 2),
                                          ((5, 3, 1), 4)])
def test_small_and_ragged_grids(pkg, cells, degree):
    ext = [(0.0, 1.0)] * len(cells)
    sim, osim = _pair(pkg, ext, cells, degree)
    osim.run(np.inf, max_steps=3)
    sim.run(np.inf, max_steps=3)
    assert rel_linf(sim.u, osim.u) <= 1e-10
    np.testing.assert_allclose([h["dt"] for h in sim.history],
                               [h["dt"] for h in osim.history], rtol=1e-13)


@pytest.mark.parametrize("bc", ["outflow", "wall"])
def test_nonperiodic_unlimited(pkg, bc):
    sim, osim = _pair(pkg, [(0.0, 1.0), (0.0, 1.0)], (4, 3), 3, bc=bc, vel=[0.3, -0.2])
    osim.run(np.inf, max_steps=3)
    sim.run(np.inf, max_steps=3)
    assert rel_linf(sim.u, osim.u) <= 1e-10


def test_explicit_advance_and_finite_t_end(pkg):
    from oracle import dg

    sim, osim = _pair(pkg, [(0.0, 1.0)] * 3, (3, 3, 2), 3)
    dt_g = sim.max_timestep()
    dt_o = dg.compute_timestep(osim.u, osim.phys, osim.mesh.spacings, osim.cfl, 3)
    assert abs(dt_g - dt_o) <= 1e-14 * dt_o
    assert sim.advance(0.5 * dt_g) == 0.5 * dt_g
    osim.advance(0.5 * dt_o)
    assert rel_linf(sim.u, osim.u) <= 1e-10
    t_end = sim.t + 2.5 * dt_g
    sim.run(t_end)
    osim.run(t_end)
    assert sim.step_count == osim.step_count
    assert abs(sim.t - t_end) <= 1e-12 and abs(sim.history[-1]["dt"] -
                                                osim.history[-1]["dt"]) <= 1e-15
    assert rel_linf(sim.u, osim.u) <= 1e-10


def test_error_conventions(pkg):
    system = pkg.make_system("euler", 2)
    mesh = pkg.CartesianMesh([(0, 1), (0, 1)], (2, 2))
    sim = pkg.Simulation(mesh, system, 2, 0.05)
    with pytest.raises(RuntimeError):
        sim.run(1.0)                       # no initial state (driver.py:188-189)
    with pytest.raises(ValueError):
        sim.project_initial_condition(lambda x: np.ones(x.shape[:-1] + (3,)))
    bad = np.zeros((2, 2, 3, 3, 4))
    bad[..., 0] = -1.0                     # no admissible state (corrector.py:44-45)
    bad[..., 3] = 1.0
    sim.set_state(bad)
    with pytest.raises(RuntimeError, match="no admissible"):
        sim.max_timestep()
    ok = np.zeros((2, 2, 3, 3, 4))
    ok[..., 0] = 1.0
    ok[..., 3] = 2.5
    ok[0, 0, 1, 1, 1] = np.nan             # non-finite state (driver.py:197-199)
    sim.set_state(ok)
    with pytest.raises(RuntimeError):
        sim.run(np.inf, max_steps=2)


def test_force_limit_all_matches_oracle_and_conserves(pkg):
    sim, osim = _pair(pkg, [(0.0, 1.0), (0.0, 1.0)], (6, 5), 2, limiter=True, vel=[0.5, 0.25])
    sim.force_limit_all = True
    osim.force_limit_all = True
    t0 = sim.conserved_totals()
    for s in range(3):
        sim.run(np.inf, max_steps=s + 1)
        osim.run(np.inf, max_steps=s + 1)
        assert bool(sim.last_troubled.all())
        assert sim.last_limited_fraction == 1.0
    assert rel_linf(sim.u, osim.u) <= 1e-10
    t1 = sim.conserved_totals()
    assert np.max(np.abs(t1 - t0) / np.abs(t0)) <= 1e-11


def test_restart_halves_dt(pkg, monkeypatch):
    """A failed rescue restarts the step at dt/2 (driver.py:166-184); fault
    injection as in the reference's test_mesh_driver.py:216-237."""
    sim, _ = _pair(pkg, [(0.0, 1.0), (0.0, 1.0)], (4, 4), 2, limiter=True)
    real = sim._attempt_limited
    calls = []

    def flaky(row, trial):
        calls.append(trial)
        if len(calls) == 1:
            return False, 0.0, None
        return real(row, trial)

    monkeypatch.setattr(sim, "_attempt_limited", flaky)
    dt = sim.max_timestep()
    used = sim.advance(dt)
    assert used == 0.5 * dt and calls == [dt, 0.5 * dt]

    def hopeless(row, trial):
        return False, 0.0, None

    monkeypatch.setattr(sim, "_attempt_limited", hopeless)
    with pytest.raises(RuntimeError, match="halvings"):
        sim.advance(dt)


@pytest.mark.parametrize("degree", [1, 2, 3, 4, 5, 7, 9])
def test_limiter_3d_matches_oracle(pkg, degree):
    """3-D limited runs (every cell forced through the MUSCL-Hancock rescue,
    then natural detection) against the oracle, periodic and outflow faces:
    the subcell windows grow as (2N+5)^3, so from N = 3 on the rescue and
    screening kernels run with L2-resident global scratch."""
    cells = (3, 2, 2)
    for bc in ("periodic", "outflow"):
        sim, osim = _pair(pkg, [(0.0, 1.0)] * 3, cells, degree, bc=bc, limiter=True,
                          vel=[0.5, 0.25, -0.3])
        sim.force_limit_all = True
        osim.force_limit_all = True
        sim.run(np.inf, max_steps=1)
        osim.run(np.inf, max_steps=1)
        assert bool(sim.last_troubled.all())
        sim.force_limit_all = False
        osim.force_limit_all = False
        sim.run(np.inf, max_steps=3)
        osim.run(np.inf, max_steps=3)
        np.testing.assert_array_equal(sim.last_troubled.cpu().numpy(),
                                      np.asarray(osim.last_troubled))
        assert rel_linf(sim.u, osim.u) <= 1e-10


@pytest.mark.parametrize("unroll,steps", [(8, 21), (4, 7), (16, 40)])
def test_graph_unroll_bitwise(pkg, unroll, steps):
    """Batched runs replaying an unrolled CUDA graph (plus the two-step tail
    and a single eager step) match the two-step graph bit for bit."""
    out = []
    for n in (2, unroll):
        system = pkg.make_system("euler", 2)
        sim = pkg.Simulation(pkg.CartesianMesh([(0.0, 10.0), (0.0, 10.0)], (12, 10)), system, 3,
                             0.9 / 14)
        sim.graph_steps = n
        sim.project_initial_condition(pkg.build_problem("vortex", system)[0])
        sim.run(np.inf, max_steps=steps)
        rows = np.array([[h["dt"], h["time"], *h["totals"]] for h in sim.history])
        out.append((rows, sim.u.cpu().numpy(), sim.step_count))
    assert out[0][2] == out[1][2] == steps
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("dim,cells,degree", [(3, (5, 4, 3), 4), (2, (9, 7), 3), (1, (17,), 5),
                                              (3, (3, 3, 2), 6)])
def test_folded_state_update_matches_plain(pkg, monkeypatch, dim, cells, degree):
    """ADG_GRID_FOLD_STATE (the predictor leaves u^n + vol / mass, adg_update
    reads one array less) against the plain volume-integral path
    (ADG_NO_FOLD=1): the reference's u + (vol - faces) / mass
    (corrector.py:199-205) re-associated, so equal to rounding."""
    system = pkg.make_system("euler", dim)
    name = "density_wave" if dim > 1 else "density_wave"
    ic = pkg.build_problem(name, system)[0]

    def run(no_fold):
        if no_fold:
            monkeypatch.setenv("ADG_NO_FOLD", "1")
        else:
            monkeypatch.delenv("ADG_NO_FOLD", raising=False)
        sim = pkg.Simulation(pkg.CartesianMesh([(0.0, 1.0)] * dim, cells), system, degree,
                             0.9 / (dim * (2 * degree + 1)))
        sim.project_initial_condition(ic)
        sim.run(np.inf, max_steps=5)
        return sim

    a, b = run(False), run(True)
    assert a._grid.flags == 1 and b._grid.flags == 0
    np.testing.assert_allclose([h["dt"] for h in a.history], [h["dt"] for h in b.history],
                               rtol=1e-13)
    err = float((a.u - b.u).abs().max() / b.u.abs().max())
    assert err <= 1e-13
    # unsupported grids refuse the flag instead of ignoring it
    from paper_1808_03788_b200 import _lib
    g = _lib.Grid.from_buffer_copy(a._grid)
    g.mode = _lib.MODE_CODES["primitive"]
    assert _lib.load().adg_fold_supported(_lib.ctypes.byref(g)) == 0
