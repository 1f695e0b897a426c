"""The reference's module-level predictor / corrector contract, exercised on
the drop-in's device functions (predictor.py:99-230, corrector.py:30-205).
The cases restate the properties the reference's own test_predictor.py and
test_corrector.py check (nilpotent sweeps from a given starting iterate, exact
space-time solutions, flags, traces, time-step sizing, Riemann terms), plus
pins against the reference's golden predictor outputs (predictor.npz).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1808_03788_b200 import _lib, corrector, predictor, systems
    from paper_1808_03788_b200.basis import basis_tables

    _lib.load()
    return predictor, corrector, systems, basis_tables


def host(t):
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


def flat_start(u, degree):
    return np.repeat(np.asarray(u)[..., None, :], degree + 1, axis=-2)


# ------------------------------------------------------------------ predictor

@pytest.mark.parametrize("deg", range(6))
def test_advection_sweeps_nilpotent_from_flat_start(api, deg):
    """A linear homogeneous sweep map is nilpotent: from a constant-in-time
    start, N+1 sweeps reach the fixed point (weak-form defect at rounding)."""
    predictor, _, systems, tabs = api
    t = tabs(deg)
    u = np.random.default_rng(deg).uniform(-1, 1, (4, deg + 1, 1))
    adv = systems.LinearAdvection(1, velocity=[1.0])
    dt = 0.4 / (2 * deg + 1)
    res = predictor.picard_solve(u, adv, [1.0], dt, t, tol=0.0, max_iter=deg + 1,
                                 initial=flat_start(u, deg))
    assert res.iterations == deg + 1
    defect = predictor.weak_form_defect(res.q, u, adv, [1.0], dt, t)
    assert float(defect.max()) <= 1e-12


@pytest.mark.parametrize("deg", [2, 3, 4, 5])
def test_advection_two_sweeps_short_keeps_defect(api, deg):
    predictor, _, systems, tabs = api
    t = tabs(deg)
    u = np.random.default_rng(100 + deg).uniform(-1, 1, (4, deg + 1, 1))
    adv = systems.LinearAdvection(1, velocity=[1.0])
    dt = 0.4 / (2 * deg + 1)
    res = predictor.picard_solve(u, adv, [1.0], dt, t, tol=0.0, max_iter=deg - 1,
                                 initial=flat_start(u, deg))
    defect = predictor.weak_form_defect(res.q, u, adv, [1.0], dt, t)
    assert float(defect.max()) > 1e-12


def test_exact_linear_space_time_solution(api):
    """u0(x) = x at unit speed stays in the space-time basis."""
    predictor, _, systems, tabs = api
    deg = 3
    t = tabs(deg)
    adv = systems.LinearAdvection(1, velocity=[1.0])
    u = t.nodes.reshape(1, deg + 1, 1).copy()
    dt = 0.05
    res = predictor.picard_solve(u, adv, [1.0], dt, t)
    exact = t.nodes[None, :, None, None] - dt * t.nodes[None, None, :, None]
    np.testing.assert_allclose(host(res.q), exact, atol=1e-13)
    assert bool(res.converged.all()) and bool(res.admissible.all())
    tr = predictor.extract_traces(res.q, t, 1)
    np.testing.assert_allclose(host(tr[(0, 1)])[0, :, 0], 1.0 - dt * t.nodes, atol=1e-12)
    np.testing.assert_allclose(host(tr[(0, 0)])[0, :, 0], -dt * t.nodes, atol=1e-12)


def test_time_integral_consistency(api):
    """q(tau = 1) = u + dt * quadrature of dq/dt over the step."""
    predictor, _, systems, tabs = api
    deg = 3
    t = tabs(deg)
    adv = systems.LinearAdvection(1, velocity=[1.0])
    u = np.random.default_rng(5).uniform(-1, 1, (6, deg + 1, 1))
    dt = 0.03
    q = host(predictor.picard_solve(u, adv, [1.0], dt, t).q)
    qdot = np.einsum("kl,xnlv->xnkv", t.diff / dt, q)
    q_end = np.einsum("l,xnlv->xnv", t.right_vals, q)
    rebuilt = u + dt * np.einsum("t,xntv->xnv", t.weights, qdot)
    assert np.abs(rebuilt - q_end).max() <= 1e-11


def test_third_order_startup_converges_fast(api):
    predictor, _, systems, tabs = api
    deg = 3
    t = tabs(deg)
    e1 = systems.CompressibleEuler(1)
    h = 1.0 / 8
    x = (np.arange(8) * h)[:, None] + h * t.nodes[None, :]
    prim = np.stack([1.0 + 0.2 * np.sin(2 * np.pi * x), 0.5 * np.ones_like(x),
                     np.ones_like(x)], axis=-1)
    u = e1.prim_to_cons(prim)
    res = predictor.picard_solve(u, e1, [h], 0.1 * h / (2 * deg + 1), t)
    assert bool(res.converged.all())
    assert res.iterations <= deg + 2


def test_constant_state_fixed_point(api):
    predictor, _, systems, tabs = api
    deg = 3
    t = tabs(deg)
    const = np.array([1.0, 0.5, -0.25, 3.0])
    u = np.tile(const, (5, deg + 1, deg + 1, 1))
    res = predictor.picard_solve(u, systems.CompressibleEuler(2), [0.1, 0.1], 0.01, t)
    np.testing.assert_allclose(host(res.q), np.tile(const, (5, deg + 1, deg + 1, deg + 1, 1)),
                               rtol=0, atol=5e-14)
    assert bool(res.converged.all())


def test_primitive_equals_conservative_for_advection(api):
    predictor, _, systems, tabs = api
    deg = 2
    t = tabs(deg)
    adv = systems.LinearAdvection(1, velocity=[1.3])
    u = np.random.default_rng(11).uniform(-1, 1, (4, deg + 1, 1))
    cons = predictor.picard_solve(u, adv, [0.5], 0.02, t)
    prim = predictor.picard_solve(u, adv, [0.5], 0.02, t, mode="primitive")
    np.testing.assert_allclose(host(prim.q), host(cons.q), atol=1e-13)


def test_primitive_consistent_with_conservative_for_euler(api):
    predictor, _, systems, tabs = api
    deg = 3
    t = tabs(deg)
    e1 = systems.CompressibleEuler(1)
    h = 1.0 / 16
    x = (np.arange(16) * h)[:, None] + h * t.nodes[None, :]
    prim = np.stack([1.0 + 0.1 * np.sin(2 * np.pi * x), 0.3 * np.ones_like(x),
                     1.0 + 0.05 * np.cos(2 * np.pi * x)], axis=-1)
    u = e1.prim_to_cons(prim)
    dt = 0.2 * h / (2 * deg + 1)
    cons = predictor.picard_solve(u, e1, [h], dt, t)
    primr = predictor.picard_solve(u, e1, [h], dt, t, mode="primitive")
    assert bool(cons.converged.all()) and bool(primr.converged.all())
    np.testing.assert_allclose(host(primr.q), host(cons.q), atol=2e-9)


def test_inadmissible_flagged_separately(api):
    predictor, _, systems, tabs = api
    deg = 2
    t = tabs(deg)
    u = np.tile(np.array([1.0, 0.0, 2.0]), (3, deg + 1, 1))
    u[1, 0, -1] = 0.01
    u[2, 1, 1] = 5.0        # negative pressure at one node
    res = predictor.picard_solve(u, systems.CompressibleEuler(1), [0.1], 0.001, t)
    adm = host(res.admissible)
    assert adm[0] and not adm[2]


def test_elasticity_material_interface_at_rest(api):
    predictor, _, systems, tabs = api
    deg = 2
    t = tabs(deg)
    el = systems.DiffuseInterfaceElasticity()
    u = np.zeros((4, deg + 1, deg + 1, 9))
    u[..., el.ALPHA] = 1.0
    u[2:, ..., el.ALPHA] = 1e-3
    u[..., el.LAM], u[..., el.MU], u[..., el.RHO] = 2.0, 1.0, 1.0
    res = predictor.picard_solve(u, el, [0.1, 0.1], 0.005, t)
    assert bool(res.converged.all())
    assert np.abs(host(res.q)[..., :3]).max() <= 1e-13


def test_traces_of_raw_q_any_quantity_count(api):
    predictor, _, _, tabs = api
    deg = 2
    t = tabs(deg)
    q = np.random.default_rng(3).uniform(-1, 1, (5, deg + 1, deg + 1, deg + 1, 2))
    tr = predictor.extract_traces(q, t, dim=2)
    assert set(tr) == {(0, 0), (0, 1), (1, 0), (1, 1)}
    assert tuple(tr[(0, 0)].shape) == (5, deg + 1, deg + 1, 2)
    np.testing.assert_allclose(host(tr[(1, 1)]), np.tensordot(t.right_vals, q, axes=(0, 2)),
                               rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(host(tr[(0, 0)]), np.tensordot(t.left_vals, q, axes=(0, 1)),
                               rtol=1e-15, atol=1e-15)


@pytest.mark.parametrize("key", ["d3_N1", "d3_N2", "d3_N3", "d3_N4", "d3_N5", "d2_N3",
                                 "d2_N5"])
def test_global_sweep_rule_matches_reference(api, golden, key):
    """picard_solve's default (reference) sweep rule: the reference's global
    iteration count, q, both flags, raw-q traces and the weak-form defect of
    the reference's q."""
    predictor, _, systems, tabs = api
    g = golden("predictor")
    d, n = int(key[1]), int(key.split("N")[1])
    u = g[key + "_u"]
    sp = tuple(1.0 / c for c in u.shape[:d])
    e = systems.CompressibleEuler(d)
    t = tabs(n)
    dt = float(g[key + "_dt"])
    res = predictor.picard_solve(u, e, sp, dt, t)
    assert res.iterations == int(g[key + "_iters"])
    np.testing.assert_array_equal(host(res.converged), g[key + "_converged"])
    np.testing.assert_array_equal(host(res.admissible), g[key + "_admissible"])
    q = g[key + "_q"]
    assert np.abs(host(res.q) - q).max() / np.abs(q).max() <= 1e-13
    tr = predictor.extract_traces(q, t, d)
    for j in range(d):
        for s in (0, 1):
            ref = g[key + f"_tr{j}{s}"]
            assert np.abs(host(tr[(j, s)]) - ref).max() <= 1e-13 * np.abs(ref).max()
    defect = host(predictor.weak_form_defect(q, u, e, sp, dt, t))
    np.testing.assert_allclose(defect, g[key + "_defect"], rtol=1e-3, atol=1e-15)


def test_startup_guess_matches_oracle(api):
    from oracle import dg
    from oracle.basis import oracle_tables
    from oracle.euler import EulerOracle

    predictor, _, systems, tabs = api
    rng = np.random.default_rng(4)
    for d, n, mode in ((3, 4, "conservative"), (2, 3, "primitive"), (1, 1, "conservative")):
        P = n + 1
        cells = (2,) * d
        x = rng.uniform(0, 1, cells + (P,) * d)
        u = np.zeros(cells + (P,) * d + (d + 2,))
        u[..., 0] = 1.0 + 0.2 * np.sin(2 * np.pi * x)
        for j in range(d):
            u[..., 1 + j] = u[..., 0] * (0.3 - 0.2 * j)
        u[..., -1] = 2.0 + 0.1 * x
        sp = tuple(0.1 + 0.05 * j for j in range(d))
        got = host(predictor.startup_guess(u, systems.CompressibleEuler(d), sp, 1e-3, tabs(n),
                                           mode=mode))
        ref = dg.startup_guess(u, EulerOracle(d), sp, 1e-3, oracle_tables(n), mode=mode)
        assert np.abs(got - ref).max() / np.abs(ref).max() <= 1e-13


# ------------------------------------------------------------------ corrector

def test_timestep_sizing(api):
    _, corrector, systems, _ = api
    adv3 = systems.LinearAdvection(3, velocity=[1.0, 1.0, 1.0])
    dt = corrector.compute_timestep(np.ones((2, 4, 4, 4, 1)), adv3, [0.1] * 3, 0.1, degree=3)
    assert dt == pytest.approx(1.0 / 300.0, rel=1e-14)
    adv1 = systems.LinearAdvection(1, velocity=[2.0])
    assert corrector.compute_timestep(np.ones((5, 3, 1)), adv1, [0.5], 0.2,
                                      degree=1) == pytest.approx(0.05, rel=1e-14)
    with pytest.raises(ValueError):
        corrector.compute_timestep(np.ones((2, 4, 1)), adv1, [0.5], 0.5, degree=3)
    zero = systems.LinearAdvection(2, velocity=[0.0, 0.0])
    assert np.isinf(corrector.compute_timestep(np.ones((2, 3, 3, 1)), zero, [0.1, 0.1], 0.1,
                                               degree=2))
    e1 = systems.CompressibleEuler(1)
    u = np.tile(np.array([1.0, 0.0, 2.5]), (4, 3, 1))
    u[2, 1] = [1.0, 10.0, 0.1]   # inadmissible; must not dominate the scan
    clean = corrector.compute_timestep(u[:2], e1, [0.1], 0.1, degree=2)
    assert corrector.compute_timestep(u, e1, [0.1], 0.1, degree=2) == pytest.approx(
        clean, rel=1e-14)
    with pytest.raises(RuntimeError):
        corrector.compute_timestep(np.tile(np.array([-1.0, 0.0, 2.5]), (2, 3, 1)), e1, [0.1],
                                   0.1, degree=2)


def _euler_states(d, count, seed):
    rng = np.random.default_rng(seed)
    q = np.empty((count, d + 2))
    rho = rng.uniform(0.1, 3.0, count)
    vel = rng.uniform(-2.0, 2.0, (count, d))
    p = rng.uniform(0.05, 5.0, count)
    q[:, 0] = rho
    q[:, 1:-1] = rho[:, None] * vel
    q[:, -1] = p / 0.4 + 0.5 * rho * np.sum(vel * vel, axis=1)
    return q


def test_riemann_terms(api):
    _, corrector, systems, _ = api
    e3 = systems.CompressibleEuler(3)
    s = _euler_states(3, 1000, 1)
    n = np.random.default_rng(2).normal(size=3)
    n /= np.linalg.norm(n)
    d = host(corrector.riemann_dminus(s, s, n, e3))
    want = np.einsum("kjv,j->kv", e3.flux(s), n)
    assert np.abs(d - want).max() <= 1e-14 * max(1.0, np.abs(want).max())
    adv = systems.LinearAdvection(1, velocity=[1.0])
    up = host(corrector.riemann_dminus(np.array([[1.0]]), np.array([[0.0]]), [1.0], adv))
    assert up[0, 0] == pytest.approx(1.0, abs=1e-15)
    e2 = systems.CompressibleEuler(2)
    qm, qp = _euler_states(2, 50, 8), _euler_states(2, 50, 9)
    lo, hi = corrector.face_fluxes(qm, qp, 0, e2)
    nn = np.array([1.0, 0.0])
    np.testing.assert_allclose(host(lo), host(corrector.riemann_dminus(qm, qp, nn, e2)),
                               rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(host(hi), host(corrector.riemann_dminus(qp, qm, -nn, e2)),
                               rtol=1e-13, atol=1e-13)
    qm, qp = _euler_states(3, 100, 10), _euler_states(3, 100, 11)
    lo, hi = corrector.face_fluxes(qm, qp, 1, e3)
    np.testing.assert_array_equal(host(lo) + host(hi), 0.0)
    assert not np.any(host(corrector.path_integral_B(qm, qp, [0.0, 1.0, 0.0], e3)))
    # advection pair telescopes too
    qa, qb = np.random.default_rng(3).uniform(-1, 1, (2, 40, 1))
    lo, hi = corrector.face_fluxes(qa, qb, 0, systems.LinearAdvection(2, velocity=[0.7, -1]))
    np.testing.assert_array_equal(host(lo) + host(hi), 0.0)


def _elastic_states(count, seed):
    rng = np.random.default_rng(seed)
    q = rng.uniform(-1, 1, (count, 9))
    q[:, 5] = rng.uniform(0.0, 1.0, count)
    q[:, 6] = rng.uniform(1.0, 3.0, count)
    q[:, 7] = rng.uniform(0.5, 2.0, count)
    q[:, 8] = rng.uniform(0.5, 2.0, count)
    return q


def test_elasticity_path_terms(api):
    _, corrector, systems, _ = api
    el = systems.DiffuseInterfaceElasticity()
    qm, qp = _elastic_states(10, 5), _elastic_states(10, 6)
    n = np.array([0.0, 1.0])
    fwd = host(corrector.path_integral_B(qm, qp, n, el))
    bwd = host(corrector.path_integral_B(qp, qm, n, el))
    np.testing.assert_allclose(fwd, bwd, atol=1e-13)
    # against the host contract: 3-point Gauss rule of ncp_matrix
    r = np.sqrt(0.6)
    want = sum(w * el.ncp_matrix(qm + s * (qp - qm), n)
               for s, w in zip((0.5 - 0.5 * r, 0.5, 0.5 + 0.5 * r), (5 / 18, 8 / 18, 5 / 18)))
    np.testing.assert_allclose(fwd, want, rtol=1e-13, atol=1e-14)
    qm, qp = _elastic_states(30, 12), _elastic_states(30, 13)
    lo, hi = corrector.face_fluxes(qm, qp, 0, el)
    b = host(corrector.path_integral_B(qm, qp, np.array([1.0, 0.0]), el))
    np.testing.assert_allclose(host(lo) + host(hi), np.einsum("kab,kb->ka", b, qp - qm),
                               rtol=1e-13, atol=1e-14)


def test_update_and_face_integral_any_quantity_count(api):
    _, corrector, _, tabs = api
    t = tabs(3)
    vol = 0.25 * t.weights.reshape(1, -1, 1) * np.ones((2, 4, 1))
    out = corrector.element_update(np.zeros((2, 4, 1)), vol, [], [0.25], t, 1)
    np.testing.assert_allclose(host(out), 1.0, rtol=1e-14)
    t2 = tabs(2)
    acc = corrector.face_integral(np.ones((4, 3, 3, 1)), 0, 1, [0.5, 0.25], 0.1, t2, 2)
    assert tuple(acc.shape) == (4, 3, 3, 1)
    want = 0.1 * 0.25 * np.multiply.outer(t2.right_vals, t2.weights)
    np.testing.assert_allclose(host(acc)[0, :, :, 0], want, rtol=1e-13)


def test_constant_state_element_is_steady(api):
    predictor, corrector, systems, tabs = api
    deg, dim = 3, 2
    t = tabs(deg)
    e2 = systems.CompressibleEuler(2)
    const = np.array([1.0, 0.4, -0.3, 2.8])
    u = np.tile(const, (1, deg + 1, deg + 1, 1))
    sp, dt = [0.2, 0.3], 0.01
    res = predictor.picard_solve(u, e2, sp, dt, t)
    tr = predictor.extract_traces(res.q, t, dim)
    vol = corrector.volume_integral(res.q, e2, sp, dt, t)
    accs = []
    for j in range(dim):
        lo, hi = corrector.face_fluxes(tr[(j, 1)], tr[(j, 0)], j, e2)
        accs.append(corrector.face_integral(lo, j, 1, sp, dt, t, dim))
        accs.append(corrector.face_integral(hi, j, 0, sp, dt, t, dim))
    out = corrector.element_update(u, vol, accs, sp, t, dim)
    assert np.abs(host(out) - u).max() <= 1e-13
