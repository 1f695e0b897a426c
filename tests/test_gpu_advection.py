"""LinearAdvection on the device (reference
systems.py:77-109 with the registry's sine / pulse / step problems,
problems.py:54-93) against golden runs of the reference
(tests/golden/make_golden.py gen_advection).  Bar: fp64 relative L-inf <=
1e-10, dt to 1e-12, totals to 1e-11."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

CASES = {
    "adv_sine_2d": ([1.0, 0.5], "sine", "periodic"),
    "adv_sine_3d": ([1.0, -0.5, 0.3], "sine", "periodic"),
    "adv_sine_3d_N5": ([0.6, 0.8, -0.4], "sine", "periodic"),
    "adv_sine_2d_N9": ([1.0, -0.7], "sine", "periodic"),
    "adv_pulse_1d": ([1.0], "pulse", "outflow"),
    "adv_step_wall_2d": ([0.7, -0.4], "step", "wall"),
}


def rel_linf(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1808_03788_b200 as p

    return p


@pytest.mark.parametrize("name", sorted(CASES))
def test_advection_matches_reference(pkg, golden, name):
    vel, prob, bc = CASES[name]
    g = golden(name)
    mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
    system = pkg.make_system("advection", mesh.dim, velocity=vel)
    sim = pkg.Simulation(mesh, system, int(g["degree"]), float(g["cfl"]), boundary=bc)
    ic, _ = pkg.build_problem(prob, system)
    sim.project_initial_condition(ic)
    assert rel_linf(sim.u, g["u0"]) <= 1e-14
    n = len(g["dts"])
    sim.run(np.inf, max_steps=n)
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-12)
    assert rel_linf(sim.u, g["u"]) <= 1e-10
    np.testing.assert_allclose(np.array([h["totals"] for h in sim.history]), g["totals"],
                               rtol=1e-11, atol=1e-13)
    assert max(sim.sweep_log) <= max(int(x) for x in g["iters"])


def test_advection_nilpotent_fixed_point(pkg):
    """Linear advection reaches the Picard fixed point after N+1 sweeps from
    the startup (test_predictor.py:30-45): a run with min_picard_iter = N+1
    agrees with the converged run to the tolerance."""
    mesh = pkg.CartesianMesh([(0.0, 1.0), (0.0, 1.0)], (5, 4))
    system = pkg.make_system("advection", 2, velocity=[0.8, -0.3])
    out = []
    for mi in (1, 4):
        sim = pkg.Simulation(mesh, system, 3, 0.9 / 14.0, min_picard_iter=mi)
        sim.project_initial_condition(pkg.build_problem("sine", system)[0])
        sim.run(np.inf, max_steps=3)
        out.append(sim.u.clone())
    assert rel_linf(out[0], out[1].cpu().numpy()) <= 1e-12


LIMITED = {
    "adv_lim_step_1d": ([1.0], "step", "periodic", "conservative", False),
    "adv_lim_sine_forced": ([1.0], "sine", "periodic", "conservative", True),
    "adv_lim_step_wall_2d": ([0.7, -0.4], "step", "wall", "conservative", False),
    "adv_lim_step_prim_2d": ([0.6, 0.5], "step", "periodic", "primitive", False),
    "adv_lim_pulse_exact_1d": ([1.0], "pulse", {0: ("exact", "outflow")}, "conservative",
                               False),
    "adv_lim_step_3d": ([1.0, 0.5, -0.3], "step", "periodic", "conservative", False),
}


@pytest.mark.parametrize("name", sorted(LIMITED))
def test_advection_limited_matches_reference(pkg, golden, name):
    """The subcell limiter on the advection plugin (the limiter kernels'
    advection policy: admissible = finite, F = a q, |lambda| = |a_j|,
    identity reflection), primitive mode (identity primitives) and exact
    faces, against the reference's runs (make_golden.py
    gen_advection_limited; the reference's own limiter-in-driver cases,
    test_mesh_driver.py:396-432): troubled flags identical every step."""
    vel, prob, bc, mode, force = LIMITED[name]
    g = golden(name)
    mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
    system = pkg.make_system("advection", mesh.dim, velocity=vel)
    ic, ex = pkg.build_problem(prob, system)
    sim = pkg.Simulation(mesh, system, int(g["degree"]), float(g["cfl"]), boundary=bc,
                         use_limiter=True, predictor_mode=mode,
                         exact_solution=ex if name.endswith("exact_1d") else None)
    sim.force_limit_all = force
    sim.project_initial_condition(ic)
    assert rel_linf(sim.u, g["u0"]) <= 1e-14
    flags = []
    for _ in range(len(g["dts"])):
        sim.run(np.inf, max_steps=sim.step_count + 1)
        flags.append(sim.last_troubled.cpu().numpy())
    np.testing.assert_array_equal(np.stack(flags), g["troubled"])
    np.testing.assert_allclose([h["limited_fraction"] for h in sim.history], g["fracs"])
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-12)
    assert rel_linf(sim.u, g["u"]) <= 1e-10
    np.testing.assert_allclose(np.array([h["totals"] for h in sim.history]), g["totals"],
                               rtol=1e-11, atol=1e-13)


def test_advection_limited_device_loop(pkg, golden):
    """The one-sync-per-step limited run loop (run(t_end)) on the advection
    plugin equals step-by-step advancing."""
    g = golden("adv_lim_step_1d")
    mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
    system = pkg.make_system("advection", 1, velocity=[1.0])
    ic, _ = pkg.build_problem("step", system)
    sim = pkg.Simulation(mesh, system, int(g["degree"]), float(g["cfl"]), use_limiter=True)
    sim.project_initial_condition(ic)
    sim.run(np.inf, max_steps=len(g["dts"]))
    assert rel_linf(sim.u, g["u"]) <= 1e-10
