"""predictor_mode="primitive" on the device:
primitive-variable space-time predictor (predictor.py:94-96, :109-112,
:165-189) and primitive MUSCL-Hancock half step in the limiter
(limiter.py:124-202), against the reference's golden runs and the oracle.
Bar: fp64 relative L-inf <= 1e-10, identical troubled-cell flags.
"""

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


@pytest.mark.parametrize("name,problem,bc,limited", [
    ("prim_vortex", "vortex", "periodic", False),
    ("prim_wave3d", "density_wave", "periodic", False),
    ("prim_sod", "sod", "outflow", True),
    ("prim_blast", "blast", "wall", True)])
def test_primitive_golden(pkg, golden, name, problem, bc, limited):
    g = golden(name)
    mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
    system = pkg.make_system("euler", mesh.dim)
    sim = pkg.Simulation(mesh, system, int(g["degree"]), float(g["cfl"]), boundary=bc,
                         use_limiter=limited, predictor_mode="primitive")
    sim.project_initial_condition(pkg.build_problem(problem, system)[0])
    assert rel_linf(sim.u, g["u0"]) <= 1e-14
    for s in range(len(g["dts"])):
        sim.run(np.inf, max_steps=s + 1)
        if limited:
            np.testing.assert_array_equal(sim.last_troubled.cpu().numpy(), g["troubled"][s],
                                          err_msg=f"step {s + 1}")
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-12)
    assert max(sim.sweep_log) <= max(int(x) for x in g["iters"])
    assert rel_linf(sim.u, g["u"]) <= TOL


@pytest.mark.parametrize("d,n,cells", [(1, 3, (7,)), (1, 9, (3,)), (2, 3, (3, 4)),
                                       (2, 6, (2, 3)), (3, 2, (3, 2, 2)), (3, 4, (2, 2, 3)),
                                       (3, 5, (2, 2, 2)), (3, 6, (2, 1, 2))])
def test_primitive_predictor_vs_oracle(pkg, d, n, cells):
    """Fused primitive predictor vs the oracle's per-element Picard on seeded
    smooth states; covers the register (d<=2), shared 3-tile, single-buffer
    (3-D N=5) and L2-slab (3-D N>=6) kernel variants."""
    from oracle import dg
    from oracle.basis import oracle_tables
    from oracle.euler import EulerOracle
    from paper_1808_03788_b200.predictor import run_predictor

    rng = np.random.default_rng(10 * d + n)
    P = n + 1
    x = rng.uniform(0, 1, cells + (P,) * d)
    rho = 1.0 + 0.3 * np.sin(2 * np.pi * x)
    vel = (0.7, -0.4, 0.2)[:d]
    u = np.empty(cells + (P,) * d + (d + 2,))
    u[..., 0] = rho
    for j in range(d):
        u[..., 1 + j] = rho * vel[j]
    u[..., -1] = 2.5 * (1.0 + 0.1 * np.cos(2 * np.pi * x)) + 0.5 * rho * sum(v * v for v in vel)
    sp = (0.1, 0.2, 0.15)[:d]
    dt = 2e-3
    ref = dg.picard_solve(u, EulerOracle(d), sp, dt, oracle_tables(n), per_element=True,
                          mode="primitive")
    res, good = run_predictor(torch.as_tensor(u).cuda(), pkg.make_system("euler", d), sp, dt,
                              pkg.basis_tables(n), mode="primitive")
    assert rel_linf(res.q, ref.q) <= 1e-12
    np.testing.assert_array_equal(res.sweeps.cpu().numpy(), ref.sweeps)
    np.testing.assert_array_equal(good.cpu().numpy(), ref.converged & ref.admissible)


def test_primitive_explosion_vs_oracle(pkg):
    """Circular explosion (C4 shape at 32^2, N=3), primitive mode with the
    limiter: identical flags each step, states within 1e-10."""
    from oracle import problems as oprob
    from oracle.euler import EulerOracle
    from oracle.sim import OracleMesh, OracleSimulation

    ext, cells, n, cfl = [(-1.0, 1.0), (-1.0, 1.0)], (32, 32), 3, 0.9 / 14.0
    osim = OracleSimulation(OracleMesh(ext, cells), EulerOracle(2), n, cfl, boundary="outflow",
                            use_limiter=True, per_element_picard=True,
                            predictor_mode="primitive")
    osim.project_initial_condition(oprob.explosion()[0])
    mesh = pkg.CartesianMesh(ext, cells)
    system = pkg.make_system("euler", 2)
    sim = pkg.Simulation(mesh, system, n, cfl, boundary="outflow", use_limiter=True,
                         predictor_mode="primitive")
    sim.project_initial_condition(pkg.build_problem("explosion", system)[0])
    for s in range(4):
        osim.run(np.inf, max_steps=s + 1)
        sim.run(np.inf, max_steps=s + 1)
        np.testing.assert_array_equal(sim.last_troubled.cpu().numpy(), osim.last_troubled,
                                      err_msg=f"step {s + 1}")
    assert osim.last_limited_fraction > 0.0
    assert rel_linf(sim.u, osim.u) <= TOL


def test_primitive_free_stream(pkg):
    """A constant state is a fixed point in primitive mode too."""
    mesh = pkg.CartesianMesh([(0, 1)] * 3, (4, 3, 5))
    system = pkg.make_system("euler", 3)
    sim = pkg.Simulation(mesh, system, 3, 0.9 / 21.0, predictor_mode="primitive")
    u0 = sim.project_initial_condition(pkg.build_problem("constant", system)[0]).clone()
    sim.run(np.inf, max_steps=3)
    assert rel_linf(sim.u, u0.cpu().numpy()) <= 1e-12
