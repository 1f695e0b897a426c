""""exact" faces on the device: exterior space-time
traces evaluated from exact_solution per step (driver.py:250-261) and
exterior subcell slabs for the limiter (driver.py:317-340), against the
reference's golden runs and the oracle.  Bar: rel. L-inf <= 1e-10,
identical troubled-cell flags."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = 1e-10


def rel_linf(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1808_03788_b200 as p
    from paper_1808_03788_b200 import _lib

    _lib.load()
    return p


def test_exact_wave2d_golden(pkg, golden):
    from oracle import problems as oprob

    g = golden("exact_wave2d")
    ic, ex = oprob.density_wave(vel=(1.0, 0.5))
    mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
    sim = pkg.Simulation(mesh, pkg.make_system("euler", 2), int(g["degree"]), float(g["cfl"]),
                         boundary="exact", exact_solution=ex)
    sim.project_initial_condition(ic)
    assert rel_linf(sim.u, g["u0"]) <= 1e-14
    sim.run(np.inf, max_steps=len(g["dts"]))
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-12)
    assert rel_linf(sim.u, g["u"]) <= TOL


@pytest.mark.parametrize("mode", ["conservative", "primitive"])
def test_exact_explosion_limited(pkg, golden, mode):
    from oracle import problems as oprob
    from oracle.euler import EulerOracle
    from oracle.sim import OracleMesh, OracleSimulation

    g = golden("exact_explosion")
    ic = oprob.explosion()[0]
    bnd = {0: ("exact", "outflow"), 1: ("wall", "exact")}
    ext = [tuple(e) for e in g["extents"]]
    cells = tuple(int(c) for c in g["cells"])
    mesh = pkg.CartesianMesh(ext, cells)
    sim = pkg.Simulation(mesh, pkg.make_system("euler", 2), int(g["degree"]), float(g["cfl"]),
                         boundary=bnd, use_limiter=True, predictor_mode=mode,
                         exact_solution=lambda x, t: ic(x))
    sim.project_initial_condition(ic)
    if mode == "conservative":
        ref_flags, ref_u, ref_dts = g["troubled"], g["u"], g["dts"]
        for s in range(len(ref_dts)):
            sim.run(np.inf, max_steps=s + 1)
            np.testing.assert_array_equal(sim.last_troubled.cpu().numpy(), ref_flags[s],
                                          err_msg=f"step {s + 1}")
    else:
        osim = OracleSimulation(OracleMesh(ext, cells), EulerOracle(2), int(g["degree"]),
                                float(g["cfl"]), boundary=bnd, use_limiter=True,
                                exact_solution=lambda x, t: ic(x), per_element_picard=True,
                                predictor_mode="primitive")
        osim.project_initial_condition(ic)
        for s in range(6):
            osim.run(np.inf, max_steps=s + 1)
            sim.run(np.inf, max_steps=s + 1)
            np.testing.assert_array_equal(sim.last_troubled.cpu().numpy(), osim.last_troubled,
                                          err_msg=f"step {s + 1}")
        ref_u, ref_dts = osim.u, [h["dt"] for h in osim.history]
    np.testing.assert_allclose([h["dt"] for h in sim.history], ref_dts, rtol=1e-12)
    assert rel_linf(sim.u, ref_u) <= TOL


def test_exact_wave3d_vs_oracle(pkg):
    """3-D: exact faces on all six sides exercise the three trace-block
    orders (x [j][k][t], y [k][t][i], z [t][i][j])."""
    from oracle import problems as oprob
    from oracle.euler import EulerOracle
    from oracle.sim import OracleMesh, OracleSimulation

    ic, ex = oprob.density_wave(vel=(1.0, 0.5, -0.7))
    ext, cells, n, cfl = [(0.0, 1.0)] * 3, (4, 3, 5), 2, 0.9 / 15.0
    osim = OracleSimulation(OracleMesh(ext, cells), EulerOracle(3), n, cfl, boundary="exact",
                            exact_solution=ex, per_element_picard=True)
    osim.project_initial_condition(ic)
    osim.run(np.inf, max_steps=3)
    sim = pkg.Simulation(pkg.CartesianMesh(ext, cells), pkg.make_system("euler", 3), n, cfl,
                         boundary="exact", exact_solution=ex)
    sim.project_initial_condition(ic)
    sim.run(np.inf, max_steps=3)
    assert rel_linf(sim.u, osim.u) <= TOL
    err = sim.error_norms()
    assert err["linf"].max() < 5e-3


def test_exact_sod_1d_vs_oracle(pkg):
    """1-D Sod, static exact data on the left, outflow on the right, limited."""
    from oracle import problems as oprob
    from oracle.euler import EulerOracle
    from oracle.sim import OracleMesh, OracleSimulation

    ic = oprob.sod()[0]
    bnd = {0: ("exact", "outflow")}
    ext, cells, n, cfl = [(0.0, 1.0)], (30,), 3, 0.09
    osim = OracleSimulation(OracleMesh(ext, cells), EulerOracle(1), n, cfl, boundary=bnd,
                            use_limiter=True, exact_solution=lambda x, t: ic(x),
                            per_element_picard=True)
    osim.project_initial_condition(ic)
    sim = pkg.Simulation(pkg.CartesianMesh(ext, cells), pkg.make_system("euler", 1), n, cfl,
                         boundary=bnd, use_limiter=True, exact_solution=lambda x, t: ic(x))
    sim.project_initial_condition(ic)
    for s in range(10):
        osim.run(np.inf, max_steps=s + 1)
        sim.run(np.inf, max_steps=s + 1)
        np.testing.assert_array_equal(sim.last_troubled.cpu().numpy(), osim.last_troubled)
    assert rel_linf(sim.u, osim.u) <= TOL


def _exact_wave_sim(pkg, exact, limiter, **kw):
    system = pkg.make_system("euler", 2)
    ic, _ = pkg.build_problem("density_wave", system, velocity=(1.0, 0.5))
    mesh = pkg.CartesianMesh([(0.0, 1.0), (0.0, 0.8)], (6, 5))
    sim = pkg.Simulation(mesh, system, 3, 0.9 / (2 * 7), boundary="exact",
                         exact_solution=exact, use_limiter=limiter, **kw)
    sim.project_initial_condition(ic)
    return sim


@pytest.mark.parametrize("limiter", [False, True])
def test_exact_device_resident_matches_host_evaluation(pkg, limiter):
    """A `device_capable` exact_solution (the package's closed-form cases) is
    evaluated on the device from the device clock: boundary traces and the
    limiter's subcell slabs without host evaluation or upload, the batched /
    limited device loops stay on.  Same run with the same function hidden
    behind a plain lambda (host evaluation, driver.py:250-261, :317-340)."""
    system = pkg.make_system("euler", 2)
    _, ex = pkg.build_problem("density_wave", system, velocity=(1.0, 0.5))
    assert getattr(ex, "device_capable", False)
    a = _exact_wave_sim(pkg, ex, limiter)
    b = _exact_wave_sim(pkg, lambda x, t: ex(x, t), limiter)
    assert a._exact_dev and not b._exact_dev
    a.run(np.inf, max_steps=6)
    b.run(np.inf, max_steps=6)
    assert a.step_count == b.step_count == 6
    np.testing.assert_allclose([h["dt"] for h in a.history], [h["dt"] for h in b.history],
                               rtol=1e-13)
    assert rel_linf(a.u, b.u.cpu().numpy()) <= 1e-12
    if limiter:
        assert torch.equal(a.last_troubled, b.last_troubled)


def test_exact_device_resident_batched_equals_stepwise(pkg):
    """Unlimited run with device-resident exact faces: the batched (CUDA graph)
    loop against the step-by-step loop (an on_step callback forces it)."""
    system = pkg.make_system("euler", 2)
    _, ex = pkg.build_problem("density_wave", system, velocity=(1.0, 0.5))
    a = _exact_wave_sim(pkg, ex, False)
    b = _exact_wave_sim(pkg, ex, False)
    a.run(np.inf, max_steps=7)
    b.run(np.inf, max_steps=7, on_step=lambda s: None)
    np.testing.assert_allclose([h["dt"] for h in a.history], [h["dt"] for h in b.history],
                               rtol=1e-14)
    assert rel_linf(a.u, b.u.cpu().numpy()) <= 1e-13
    # and against the exact solution itself: boundary data consistent in time
    err = a.error_norms()
    assert err["linf"].max() < 5e-3
