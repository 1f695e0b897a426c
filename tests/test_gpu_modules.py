"""Module-level corrector / limiter functions on the device (SURVEY.md §8(b)
"module functions"): the reference's corrector.py / limiter.py call
signatures backed by the library's kernels, against the golden vectors
(pointwise Rusanov pairs, predictor-piece volume integrals) and the oracle
on seeded states (random_euler_states distribution, test_systems.py:15-25)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1808_03788_b200 import _lib, corrector, limiter, make_system

    _lib.load()
    return corrector, limiter, make_system


def host(t):
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


def rel(a, b):
    a, b = host(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def states(d, n, seed, gamma=1.4):
    rng = np.random.default_rng(seed)
    q = np.empty((n, d + 2))
    rho = rng.uniform(0.1, 3.0, n)
    vel = rng.uniform(-2.0, 2.0, (n, d))
    p = rng.uniform(0.05, 5.0, n)
    q[:, 0] = rho
    q[:, 1:1 + d] = rho[:, None] * vel
    q[:, -1] = p / (gamma - 1.0) + 0.5 * rho * np.sum(vel * vel, axis=1)
    return q


@pytest.mark.parametrize("d", [1, 2, 3])
def test_face_fluxes_golden(mods, golden, d):
    corrector, _, make_system = mods
    g = golden("pointwise")
    q = g[f"d{d}_q"][:256]
    for j in range(d):
        lo, hi = corrector.face_fluxes(q[:128], q[128:], j, make_system("euler", d))
        assert rel(lo, g[f"d{d}_dlow{j}"]) <= 1e-14
        assert rel(hi, g[f"d{d}_dhigh{j}"]) <= 1e-14
        assert torch.all(lo + hi == 0.0)   # telescoping (test_corrector.py:168-173)


@pytest.mark.parametrize("key", ["d3_N2", "d3_N4", "d3_N5", "d2_N3", "d2_N5"])
def test_volume_integral_golden(mods, golden, key):
    corrector, _, make_system = mods
    from paper_1808_03788_b200 import basis_tables

    g = golden("predictor")
    d, n = int(key[1]), int(key.split("N")[1])
    cells = g[key + "_u"].shape[:d]
    sp = tuple(1.0 / c for c in cells)
    vol = corrector.volume_integral(g[key + "_q"], make_system("euler", d), sp,
                                    float(g[key + "_dt"]), basis_tables(n))
    assert rel(vol, g[key + "_vol"]) <= 1e-12


def test_compute_timestep_and_errors(mods):
    corrector, _, make_system = mods
    from oracle import dg
    from oracle.euler import EulerOracle

    e3 = make_system("euler", 3)
    u = states(3, 4 * 27, 3).reshape(4, 3, 3, 3, 5)
    sp = (0.1, 0.2, 0.3)
    dt = corrector.compute_timestep(u, e3, sp, 0.1, 2)
    assert dt == pytest.approx(dg.compute_timestep(u, EulerOracle(3), sp, 0.1, 2), rel=1e-14)
    with pytest.raises(ValueError):
        corrector.compute_timestep(u, e3, sp, 0.5, 2)
    bad = u.copy()
    bad[..., 0] = -1.0
    with pytest.raises(RuntimeError):
        corrector.compute_timestep(bad, e3, sp, 0.1, 2)


@pytest.mark.parametrize("d,n", [(1, 3), (2, 2), (3, 4)])
def test_face_integral_and_update(mods, d, n):
    corrector, _, make_system = mods
    from oracle import dg
    from oracle.basis import oracle_tables
    from paper_1808_03788_b200 import basis_tables

    rng = np.random.default_rng(10 * d + n)
    P, m = n + 1, d + 2
    cells = (3, 2, 2)[:d]
    sp = (0.3, 0.2, 0.1)[:d]
    dt = 0.01
    tab, otab = basis_tables(n), oracle_tables(n)
    u = rng.uniform(0.5, 2.0, cells + (P,) * d + (m,))
    vol = rng.standard_normal(u.shape)
    accs, oaccs = [], []
    for axis in range(d):
        for side in (0, 1):
            dv = rng.standard_normal(cells + (P,) * (d - 1) + (P, m))
            a = corrector.face_integral(dv, axis, side, sp, dt, tab, d)
            o = dg.face_integral(dv, axis, side, sp, dt, otab, d)
            assert rel(a, o) <= 1e-14
            accs.append(a)
            oaccs.append(o)
    new = corrector.element_update(u, vol, accs, sp, tab, d)
    assert rel(new, dg.element_update(u, vol, oaccs, sp, otab, d)) <= 1e-14


@pytest.mark.parametrize("d,n", [(1, 4), (2, 3), (3, 2)])
def test_subcell_projection_recovery_flatten(mods, d, n):
    _, limiter, make_system = mods
    from oracle import limiter as olim
    from oracle.basis import oracle_tables
    from oracle.euler import EulerOracle
    from paper_1808_03788_b200 import basis_tables

    P, m = n + 1, d + 2
    E = 6
    u = states(d, E * P ** d, 7 + d).reshape((E,) + (P,) * d + (m,))
    tab, otab = basis_tables(n), oracle_tables(n)
    sub = limiter.project_to_subcells(u, tab, d)
    assert rel(sub, olim.to_subcells(u, otab, d)) <= 1e-13
    rec = limiter.recover_from_subcells(sub, tab, d)
    assert rel(rec, olim.from_subcells(host(sub), otab, d)) <= 1e-13
    bad = u.copy()
    bad[1, ..., 0] *= -1.0          # cell 1: negative density everywhere
    nodal, nflat = limiter.flatten_inadmissible(bad, host(sub), make_system("euler", d), tab, d)
    onod, oflat = olim.flatten(bad.copy(), host(sub), EulerOracle(d), otab, d)
    assert nflat == oflat >= 1
    assert rel(nodal, onod) <= 1e-14


def test_bounds_detect_windows_minmod(mods):
    _, limiter, make_system = mods
    from oracle import limiter as olim
    from oracle.euler import EulerOracle

    # hand values of test_limiter.py:109-131
    a = np.array([1.0, 2.0, -1.0, 1.0, 0.0, -2.0])
    b = np.array([2.0, 1.0, -3.0, -1.0, 5.0, -2.0])
    np.testing.assert_array_equal(host(limiter.minmod(a, b)), [1.0, 1.0, -1.0, 0.0, 0.0, -2.0])
    vals = np.array([[0.0, 0.0, 0.0], [1.0, 2.0, 3.0], [4.0, 5.0, 6.0],
                     [7.0, 8.0, 9.0], [10.0, 10.0, 10.0]])[..., None]
    lo, hi = limiter.relaxed_bounds(vals, 1)
    np.testing.assert_allclose(host(lo)[:, 0], [-0.006, 0.992, 3.994], atol=1e-15)
    np.testing.assert_allclose(host(hi)[:, 0], [6.006, 9.008, 10.006], atol=1e-15)
    rng = np.random.default_rng(5)
    d, S = 2, 5
    padded = rng.uniform(0.5, 2.0, (6, 7, S, S, 4))
    blo, bhi = limiter.relaxed_bounds(padded, d)
    olo, ohi = olim.relaxed_bounds(padded, d)
    assert rel(blo, olo) == 0.0 and rel(bhi, ohi) == 0.0
    cand = rng.uniform(0.5, 2.0, (4, 5, 3, 3, 4))
    csub = rng.uniform(0.4, 2.1, (4, 5, S, S, 4))
    flags = limiter.detect_troubled(cand, csub, (blo, bhi), make_system("euler", 2), d)
    np.testing.assert_array_equal(host(flags),
                                  olim.detect(cand, csub, (olo, ohi), EulerOracle(2), d))
    field = rng.standard_normal((20, 22, 4))
    starts = np.array([[0, 0], [5, 3], [11, 13]])
    np.testing.assert_array_equal(host(limiter.gather_windows(field, starts, 9, 2)),
                                  olim.windows(field, starts, 9, 2))


@pytest.mark.parametrize("mode", ["conservative", "primitive"])
def test_muscl_subcell_step(mods, mode):
    _, limiter, make_system = mods
    from oracle import limiter as olim
    from oracle.euler import EulerOracle

    e1 = make_system("euler", 1)
    # test_limiter.py:204-210 / :272-286: constant windows are fixed points,
    # a hopeless window fails while a healthy one in the same batch does not
    q0 = np.array([1.0, 0.1, 1.0])
    win = np.broadcast_to(q0, (2, 7, 3)).copy()
    new, failed = limiter.muscl_subcell_step(win, e1, (0.1,), 0.02, mode=mode)
    assert not host(failed).any()
    np.testing.assert_allclose(host(new), win[:, 2:-2], rtol=0, atol=1e-15)
    healthy = np.broadcast_to(q0, (7, 3))
    mom = np.linspace(-5.0, 5.0, 7)
    hopeless = np.stack([np.full(7, 0.01), mom, 2000.0 + 0.5 * mom ** 2 / 0.01], axis=-1)
    new, failed = limiter.muscl_subcell_step(np.stack([healthy, hopeless]), e1, (0.01,), 0.05,
                                             mode=mode)
    onew, ofailed = olim.muscl_step(np.stack([healthy, hopeless]), EulerOracle(1), (0.01,),
                                    0.05, mode=mode)
    np.testing.assert_array_equal(host(failed), ofailed)
    np.testing.assert_allclose(host(new)[0], healthy[2:-2], rtol=0, atol=1e-15)
    # seeded 2-D windows against the oracle
    e2 = make_system("euler", 2)
    S = 5
    wins = states(2, 6 * (S + 4) ** 2, 11).reshape(6, S + 4, S + 4, 4)
    new, failed = limiter.muscl_subcell_step(wins, e2, (0.02, 0.03), 1e-3, mode=mode)
    onew, ofailed = olim.muscl_step(wins, EulerOracle(2), (0.02, 0.03), 1e-3, mode=mode)
    np.testing.assert_array_equal(host(failed), ofailed)
    assert rel(new, onew) <= 1e-12


def test_rusanov_theta_and_screen_edge_cases(mods):
    """rusanov_theta (corrector.py:58-62) and the limiter helpers as library
    kernels against plain torch expressions of the same ops: general normals,
    the advection plugin, NaN propagation, inadmissible states."""
    corrector, limiter, make_system = mods
    for d in (1, 2, 3):
        e = make_system("euler", d)
        qm, qp = states(d, 257, 3 + d), states(d, 257, 30 + d)
        nrm = np.random.default_rng(d).standard_normal(d)
        nrm /= np.linalg.norm(nrm)
        got = corrector.rusanov_theta(qm, qp, nrm, e)
        tm, tp = torch.as_tensor(qm).cuda(), torch.as_tensor(qp).cuda()
        nt = torch.as_tensor(nrm).cuda()
        ref = torch.maximum(e.max_abs_eigenvalue(tm, nt), e.max_abs_eigenvalue(tp, nt))
        assert got.shape == ref.shape
        assert rel(got, host(ref)) <= 1e-14
    adv = make_system("advection", 2)
    q = np.random.default_rng(0).standard_normal((5, 7, 1))
    got = corrector.rusanov_theta(q, 2 * q, (0.6, 0.8), adv)
    assert got.shape == (5, 7)
    np.testing.assert_allclose(host(got), abs(0.6 * adv.velocity[0] + 0.8 * adv.velocity[1]),
                               rtol=1e-15)
    # screen: a NaN subcell, a negative density node and a negative pressure
    # subcell are troubled; cells inside their bounds are not
    e2 = make_system("euler", 2)
    S, P = 3, 2
    cand = np.broadcast_to(np.array([1.0, 0.1, 0.2, 2.5]), (4, P, P, 4)).copy()
    csub = np.broadcast_to(np.array([1.0, 0.1, 0.2, 2.5]), (4, S, S, 4)).copy()
    lo = np.broadcast_to(np.array([0.9, 0.0, 0.1, 2.4]), (4, 4)).copy()
    hi = np.broadcast_to(np.array([1.1, 0.2, 0.3, 2.6]), (4, 4)).copy()
    csub[1, 2, 1, 2] = np.nan
    cand[2, 0, 1, 0] = -1.0
    csub[3, 0, 0, 3] = 0.001          # p < 0 at this subcell, inside no bound either
    flags = host(limiter.detect_troubled(cand, csub, (lo, hi), e2, 2))
    np.testing.assert_array_equal(flags, [False, True, True, True])
    # finite-only screen of the advection plugin, 1-D
    a1 = make_system("advection", 1)
    c1 = np.zeros((3, 2, 1))
    s1 = np.zeros((3, 3, 1))
    s1[1, 2, 0] = 0.5
    c1[2, 1, 0] = np.inf
    f1 = host(limiter.detect_troubled(c1, s1, (np.full((3, 1), -0.1), np.full((3, 1), 0.1)),
                                      a1, 1))
    np.testing.assert_array_equal(f1, [False, True, True])
    # minmod broadcasting and the bounds' NaN propagation like the torch ops
    a = torch.tensor([[1.0, -2.0, 3.0]], dtype=torch.float64).cuda()
    b = torch.tensor([[2.0], [-1.0]], dtype=torch.float64).cuda()
    pick = torch.where(a.abs() <= b.abs(), a, b)
    ref = torch.where(a * b > 0.0, pick, torch.zeros_like(pick))
    assert torch.equal(limiter.minmod(a, b), ref)
    pad = np.random.default_rng(2).uniform(0.5, 2.0, (5, 3, 1))
    pad[2, 1, 0] = np.nan
    lo2, hi2 = limiter.relaxed_bounds(pad, 1)
    assert np.isnan(host(lo2)).all() and np.isnan(host(hi2)).all()
