"""Pin the CPU oracle against golden vectors produced by the reference.

The fixtures come from `tests/golden/make_golden.py`, which imports and runs
`/root/reference/pkg/src/aderdg`.  The hand values below are the reference's
own known-answer tests (file:line cited).
"""

import numpy as np
import pytest

from oracle import dg, limiter as lim, problems
from oracle.basis import oracle_tables
from oracle.euler import EulerOracle
from oracle.sim import OracleMesh, OracleSimulation


@pytest.mark.parametrize("n", range(10))
def test_tables_match_reference(golden, n):
    g = golden("tables")
    t = oracle_tables(n)
    pairs = [("nodes", t.nodes), ("weights", t.weights), ("diff", t.diff),
             ("left", t.left_vals), ("right", t.right_vals),
             ("sub_project", t.sub_project), ("sub_recover", t.sub_recover),
             ("k1", t.k1), ("k1_inv", t.k1_inv), ("g0", t.g0), ("gw", t.gw),
             ("k1_opnorm", t.k1_opnorm)]
    for key, val in pairs:
        ref = g[f"N{n}_{key}"]
        scale = max(1.0, float(np.max(np.abs(ref))))
        assert np.max(np.abs(np.asarray(val) - ref)) <= 1e-13 * scale, key


def test_table_hand_values():
    # test_basis.py:79-83 (D rows +-sqrt(3) at N=1), :135-140 (P_sub thirds)
    t = oracle_tables(1)
    np.testing.assert_allclose(np.abs(t.diff), np.sqrt(3.0), rtol=1e-14)
    u = 2.0 * t.nodes - 1.0
    np.testing.assert_allclose(t.sub_project @ u, [-2 / 3, 0.0, 2 / 3], atol=1e-14)
    for n in range(10):
        tt = oracle_tables(n)
        np.testing.assert_allclose(tt.sub_recover @ tt.sub_project, np.eye(n + 1),
                                   atol=1e-11)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_pointwise_euler(golden, d):
    g = golden("pointwise")
    e = EulerOracle(d)
    qa = g[f"d{d}_q"]
    q = qa[:256]
    np.testing.assert_array_equal(e.flux(q), g[f"d{d}_flux"])
    np.testing.assert_array_equal(e.pressure(q), g[f"d{d}_pressure"])
    np.testing.assert_array_equal(e.admissible(qa), g[f"d{d}_admissible"])
    for j in range(d):
        np.testing.assert_array_equal(e.max_abs_eigenvalue_axis(q, j), g[f"d{d}_lam{j}"])
        lo, hi = dg.face_fluxes(q[:128], q[128:], j, e)
        np.testing.assert_array_equal(lo, g[f"d{d}_dlow{j}"])
        np.testing.assert_array_equal(hi, g[f"d{d}_dhigh{j}"])
        # d_low + d_high == 0 bitwise (test_corrector.py:168-173)
        assert np.all(lo + hi == 0.0)


def test_flux_hand_values():
    # test_systems.py:59-84: p = 1 at rest, x-flux (1, 2, 0, 0, 4)
    e = EulerOracle(3)
    q = np.array([1.0, 1.0, 0.0, 0.0, 1.0 / 0.4 + 0.5])
    f = e.flux(q)
    np.testing.assert_allclose(e.pressure(q), 1.0, rtol=1e-15)
    np.testing.assert_allclose(f[0], [1.0, 2.0, 0.0, 0.0, 4.0], rtol=1e-15)


@pytest.mark.parametrize("key", ["d3_N1", "d3_N2", "d3_N3", "d3_N4", "d3_N5",
                                 "d2_N3", "d2_N5"])
def test_predictor_pieces(golden, key):
    g = golden("predictor")
    d = int(key[1])
    n = int(key.split("N")[1])
    t = oracle_tables(n)
    e = EulerOracle(d)
    u = g[key + "_u"]
    dt = float(g[key + "_dt"])
    cells = u.shape[:d]
    sp = tuple(1.0 / c for c in cells)
    pr = dg.picard_solve(u, e, sp, dt, t)
    assert pr.iterations == int(g[key + "_iters"])
    np.testing.assert_array_equal(pr.converged, g[key + "_converged"])
    np.testing.assert_array_equal(pr.admissible, g[key + "_admissible"])
    qref = g[key + "_q"]
    assert np.max(np.abs(pr.q - qref)) <= 1e-13 * np.max(np.abs(qref))
    vol = dg.volume_integral(pr.q, e, sp, dt, t)
    vref = g[key + "_vol"]
    assert np.max(np.abs(vol - vref)) <= 1e-12 * np.max(np.abs(vref))
    tr = dg.extract_traces(pr.q, t, d)
    for (j, s), arr in tr.items():
        ref = g[key + f"_tr{j}{s}"]
        assert np.max(np.abs(arr - ref)) <= 1e-13 * np.max(np.abs(ref))
    defect = dg.weak_form_defect(pr.q, u, e, sp, dt, t)
    assert defect.max() <= 1e-11


def test_relaxed_bounds_hand_values():
    # test_limiter.py:118-131
    vals = np.array([[0.0, 0.0, 0.0], [1.0, 2.0, 3.0], [4.0, 5.0, 6.0],
                     [7.0, 8.0, 9.0], [10.0, 10.0, 10.0]])[..., None]
    lo, hi = lim.relaxed_bounds(vals, 1)
    np.testing.assert_allclose(lo[:, 0], [-0.006, 0.992, 3.994], atol=1e-15)
    np.testing.assert_allclose(hi[:, 0], [6.006, 9.008, 10.006], atol=1e-15)
    # minmod hand cases (test_limiter.py:109-114)
    a = np.array([1.0, 2.0, -1.0, 1.0, 0.0, -2.0])
    b = np.array([2.0, 1.0, -3.0, -1.0, 5.0, -2.0])
    np.testing.assert_array_equal(lim.minmod(a, b), [1.0, 1.0, -1.0, 0.0, 0.0, -2.0])


def test_muscl_constant_and_mixed_batch():
    # test_limiter.py:204-210 and :272-286
    e = EulerOracle(1)
    q0 = np.array([1.0, 0.1, 1.0])
    win = np.broadcast_to(q0, (2, 7, 3)).copy()
    new, failed = lim.muscl_step(win, e, (0.1,), 0.02)
    assert not failed.any()
    np.testing.assert_array_equal(new, win[:, 2:-2])
    healthy = np.broadcast_to(q0, (7, 3))
    mom = np.linspace(-5.0, 5.0, 7)
    hopeless = np.stack([np.full(7, 0.01), mom, 2000.0 + 0.5 * mom ** 2 / 0.01], axis=-1)
    new, failed = lim.muscl_step(np.stack([healthy, hopeless]), e, (0.01,), 0.05)
    np.testing.assert_array_equal(failed, [False, True])
    np.testing.assert_array_equal(new[0], healthy[2:-2])


def _mesh_from(g):
    return OracleMesh([tuple(e) for e in g["extents"]], tuple(int(c) for c in g["cells"]))


def _run_case(g, ic, boundary="periodic", use_limiter=False, steps=None,
              mode="conservative"):
    mesh = _mesh_from(g)
    e = EulerOracle(mesh.dim)
    sim = OracleSimulation(mesh, e, int(g["degree"]), float(g["cfl"]), boundary=boundary,
                           use_limiter=use_limiter, predictor_mode=mode)
    u0 = sim.project_initial_condition(ic)
    np.testing.assert_allclose(u0, g["u0"], rtol=0, atol=1e-14)
    n = len(g["dts"]) if steps is None else steps
    flags = []
    for _ in range(n):
        sim.run(np.inf, max_steps=sim.step_count + 1)
        if use_limiter:
            flags.append(sim.last_troubled.copy())
    return sim, flags


def _rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def test_case_c1_vortex(golden):
    g = golden("c1_vortex")
    ic, _ = problems.vortex()
    sim, _ = _run_case(g, ic)
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-13)
    assert sim.sweep_log == list(g["iters"])
    assert _rel(sim.u, g["u"]) <= 1e-12


@pytest.mark.parametrize("name", ["c2_wave_4", "c3_wave_N2", "c3_wave_N5", "c3_wave_N9",
                                  "c5_wave_ext"])
def test_case_density_wave(golden, name):
    g = golden(name)
    ic, _ = problems.density_wave()
    sim, _ = _run_case(g, ic)
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-13)
    assert sim.sweep_log == list(g["iters"])
    assert _rel(sim.u, g["u"]) <= 1e-12
    np.testing.assert_allclose(np.array([h["totals"] for h in sim.history]), g["totals"],
                               rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("name,icname,bc", [("c4_explosion_16", "explosion", "outflow"),
                                            ("sod_1d", "sod", "outflow"),
                                            ("blast_wall", "blast", "wall")])
def test_case_limiter(golden, name, icname, bc):
    g = golden(name)
    ic = {"explosion": problems.explosion,
          "sod": problems.sod,
          "blast": lambda: problems.blast(p_ambient=1e-2)}[icname]()[0]
    sim, flags = _run_case(g, ic, boundary=bc, use_limiter=True)
    np.testing.assert_array_equal(np.stack(flags), g["troubled"])
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-13)
    assert _rel(sim.u, g["u"]) <= 1e-12


@pytest.mark.parametrize("name,icname,bc,limited", [
    ("prim_vortex", "vortex", "periodic", False), ("prim_wave3d", "wave", "periodic", False),
    ("prim_sod", "sod", "outflow", True), ("prim_blast", "blast", "wall", True)])
def test_case_primitive_mode(golden, name, icname, bc, limited):
    """predictor_mode="primitive" (predictor.py:94-96, :165-189; limiter.py:127-177)."""
    g = golden(name)
    ic = {"vortex": problems.vortex, "wave": problems.density_wave, "sod": problems.sod,
          "blast": problems.blast}[icname]()[0]
    sim, flags = _run_case(g, ic, boundary=bc, use_limiter=limited, mode="primitive")
    if limited:
        np.testing.assert_array_equal(np.stack(flags), g["troubled"])
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-13)
    assert sim.sweep_log == list(g["iters"])
    assert _rel(sim.u, g["u"]) <= 1e-12


def test_case_exact_faces(golden):
    """"exact" faces (driver.py:250-261, :317-340): translating density wave
    with its exact solution on every face, unlimited."""
    g = golden("exact_wave2d")
    ic, ex = problems.density_wave(vel=(1.0, 0.5))
    mesh = _mesh_from(g)
    sim = OracleSimulation(mesh, EulerOracle(2), int(g["degree"]), float(g["cfl"]),
                           boundary="exact", exact_solution=ex)
    sim.project_initial_condition(ic)
    np.testing.assert_allclose(sim.u, g["u0"], rtol=0, atol=1e-14)
    sim.run(np.inf, max_steps=len(g["dts"]))
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-13)
    assert _rel(sim.u, g["u"]) <= 1e-12


def test_case_exact_faces_limited(golden):
    """Limited explosion with static Dirichlet ("exact") data mixed with
    outflow / wall faces: exact ghost subcells incl. corners."""
    g = golden("exact_explosion")
    ic, _ = problems.explosion()
    mesh = _mesh_from(g)
    sim = OracleSimulation(mesh, EulerOracle(2), int(g["degree"]), float(g["cfl"]),
                           boundary={0: ("exact", "outflow"), 1: ("wall", "exact")},
                           use_limiter=True, exact_solution=lambda x, t: ic(x))
    sim.project_initial_condition(ic)
    flags = []
    for _ in range(len(g["dts"])):
        sim.run(np.inf, max_steps=sim.step_count + 1)
        flags.append(sim.last_troubled.copy())
    np.testing.assert_array_equal(np.stack(flags), g["troubled"])
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-13)
    assert _rel(sim.u, g["u"]) <= 1e-12
