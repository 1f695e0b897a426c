"""Diffuse-interface elasticity on the device (the
NCP / path-conservative machinery; reference systems.py:237-345,
corrector.py:65-129, predictor.py:74-91 NCP branch, problems.py:135-192)
against golden runs of the reference (tests/golden/make_golden.py
gen_elasticity).  Bar: fp64 relative L-inf <= 1e-10 on the whole state and
on the dynamic fields (stresses, alpha-velocities) against their own scale,
dt to 1e-12, totals to 1e-11."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

CASES = {
    "el_pwave": ("pwave", "outflow"),
    "el_pwave_N5": ("pwave", "outflow"),
    "el_pwave_wall": ("pwave", "wall"),
    "el_constant": ("constant", "periodic"),
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
def test_elasticity_matches_reference(pkg, golden, name):
    prob, bc = CASES[name]
    g = golden(name)
    mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
    system = pkg.make_system("elasticity-di", 2)
    sim = pkg.Simulation(mesh, system, int(g["degree"]), float(g["cfl"]), boundary=bc)
    ic, _ = pkg.build_problem(prob, system)
    sim.project_initial_condition(ic)
    assert rel_linf(sim.u, g["u0"]) <= 1e-14
    n = len(g["dts"])
    sim.run(np.inf, max_steps=n)
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-12)
    got = sim.u.cpu().numpy()
    assert rel_linf(got, g["u"]) <= 1e-10
    dyn = np.max(np.abs(g["u"][..., :5]))
    if dyn > 0:
        assert float(np.max(np.abs(got[..., :5] - g["u"][..., :5]))) / dyn <= 1e-10
    np.testing.assert_allclose(np.array([h["totals"] for h in sim.history]), g["totals"],
                               rtol=1e-11, atol=1e-15)
    assert max(sim.sweep_log) <= max(int(x) for x in g["iters"])


def test_elasticity_constant_state_is_exact(pkg):
    """A uniform state is a fixed point of the whole step (free stream): no
    gradients, zero jumps, so every step returns u^n bitwise up to the
    update's rounding."""
    mesh = pkg.CartesianMesh([(0.0, 1.0), (0.0, 1.0)], (6, 5))
    system = pkg.make_system("elasticity-di", 2)
    sim = pkg.Simulation(mesh, system, 4, 0.9 / 18)
    ic, _ = pkg.build_problem("constant", system)
    sim.project_initial_condition(ic)
    u0 = sim.u.clone()
    sim.run(np.inf, max_steps=4)
    assert rel_linf(sim.u, u0.cpu().numpy()) <= 1e-14


def test_elasticity_unsupported_paths_fail_loudly(pkg):
    mesh = pkg.CartesianMesh([(0.0, 1.0), (0.0, 1.0)], (4, 4))
    system = pkg.make_system("elasticity-di", 2)
    with pytest.raises(NotImplementedError):
        pkg.Simulation(mesh, system, 3, 0.05, use_limiter=True)


def test_elasticity_primitive_mode_is_the_conservative_step(pkg):
    """The reference's elasticity plugin has identity primitives
    (systems.py:58-63) and primitive_rhs = -ncp(v, grad v) (systems.py:333-334),
    the conservative rate: predictor_mode="primitive" is the same step."""
    mesh = pkg.CartesianMesh([(0.0, 1.0), (0.0, 1.0)], (6, 5))
    system = pkg.make_system("elasticity-di", 2)
    ic, _ = pkg.build_problem("pwave", system)
    out = []
    for mode in ("conservative", "primitive"):
        sim = pkg.Simulation(mesh, system, 3, 0.05, boundary="outflow", predictor_mode=mode)
        sim.project_initial_condition(ic)
        sim.run(np.inf, max_steps=3)
        out.append(sim.u.cpu().numpy())
    assert np.array_equal(out[0], out[1])
