"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (the reference does not exist on the GPU
box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes small .npz fixtures next to this file.  They pin the oracle
(`oracle/`) and, through it, the CUDA path.  Nothing here is copied from
the reference sources: the reference package is imported and executed.
The two BASELINE initial conditions missing from the reference registry
(3-D density wave, circular explosion) are passed as callables through
`Simulation.project_initial_condition`, exactly as SURVEY.md §0 prescribes.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import aderdg  # noqa: E402  (reference, from PYTHONPATH)
from aderdg import corrector, limiter, predictor  # noqa: E402
from aderdg.basis import basis_tables  # noqa: E402
from aderdg.systems import CompressibleEuler  # noqa: E402

from oracle import problems  # noqa: E402  (pure IC formulas)

GAMMA = 1.4


def euler_states(dim, count, seed):
    """Seeded states with the distribution of the reference's
    random_euler_states (pkg/tests/test_systems.py:15-25)."""
    rng = np.random.default_rng(seed)
    q = np.empty((count, dim + 2))
    rho = rng.uniform(0.1, 3.0, count)
    vel = rng.uniform(-2.0, 2.0, (count, dim))
    p = rng.uniform(0.05, 5.0, count)
    q[:, 0] = rho
    for j in range(dim):
        q[:, 1 + j] = rho * vel[:, j]
    q[:, -1] = p / (GAMMA - 1.0) + 0.5 * rho * np.sum(vel * vel, axis=1)
    return q


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def gen_tables():
    out = {}
    for n in range(10):
        t = basis_tables(n)
        ops = predictor.time_operators(n)
        for key, val in (("nodes", t.nodes), ("weights", t.weights), ("diff", t.diff),
                         ("left", t.left_vals), ("right", t.right_vals),
                         ("sub_project", t.sub_project), ("sub_recover", t.sub_recover),
                         ("k1", ops.k1), ("k1_inv", ops.k1_inv), ("g0", ops.g0),
                         ("gw", ops.gw), ("k1_opnorm", np.array(ops.k1_opnorm))):
            out[f"N{n}_{key}"] = np.asarray(val)
    save("tables", **out)


def gen_pointwise():
    out = {}
    for d in (1, 2, 3):
        sysd = CompressibleEuler(d, gamma=GAMMA)
        q = euler_states(d, 256, seed=10 + d)
        # a few inadmissible probes: negative density, negative pressure, nan
        bad = q[:4].copy()
        bad[0, 0] = -0.5
        bad[1, -1] = 0.0
        bad[2, 1] = np.nan
        bad[3, -1] = 1e-3
        qa = np.concatenate([q, bad])
        out[f"d{d}_q"] = qa
        out[f"d{d}_flux"] = sysd.flux(q)
        out[f"d{d}_pressure"] = sysd.pressure(q)
        out[f"d{d}_admissible"] = sysd.admissible(qa)
        for j in range(d):
            out[f"d{d}_lam{j}"] = sysd.max_abs_eigenvalue(q, np.eye(d)[j])
        # Rusanov terms across axis 0 between shifted states
        qm, qp = q[:128], q[128:]
        for j in range(d):
            lo, hi = corrector.face_fluxes(qm, qp, j, sysd)
            out[f"d{d}_dlow{j}"] = lo
            out[f"d{d}_dhigh{j}"] = hi
    save("pointwise", **out)


def wave_mesh(cells, extent_x=1.0):
    d = len(cells)
    ext = [(0.0, extent_x)] + [(0.0, 1.0)] * (d - 1)
    return aderdg.CartesianMesh(ext, cells)


def gen_predictor():
    """Element-local predictor + corrector pieces on small 3-D / 2-D grids."""
    out = {}
    for d, cells, degrees in ((3, (2, 2, 2), (1, 2, 3, 4, 5)), (2, (3, 3), (3, 5))):
        sysd = CompressibleEuler(d, gamma=GAMMA)
        for n in degrees:
            mesh = wave_mesh(cells)
            cfl = 0.9 / (d * (2 * n + 1))
            sim = aderdg.Simulation(mesh, sysd, n, cfl)
            ic, _ = problems.density_wave(vel=(1.0, 0.5, -0.7)[:d])
            u = sim.project_initial_condition(ic)
            rng = np.random.default_rng(n)
            u = u * (1.0 + 0.01 * rng.uniform(-1, 1, u.shape))
            t = basis_tables(n)
            dt = corrector.compute_timestep(u, sysd, mesh.spacings, cfl, n)
            res = predictor.picard_solve(u, sysd, mesh.spacings, dt, t)
            tr = predictor.extract_traces(res.q, t, d)
            vol = corrector.volume_integral(res.q, sysd, mesh.spacings, dt, t)
            key = f"d{d}_N{n}"
            out[key + "_u"] = u
            out[key + "_dt"] = np.array(dt)
            out[key + "_q"] = res.q
            out[key + "_iters"] = np.array(res.iterations)
            out[key + "_converged"] = res.converged
            out[key + "_admissible"] = res.admissible
            out[key + "_vol"] = vol
            out[key + "_defect"] = predictor.weak_form_defect(res.q, u, sysd, mesh.spacings,
                                                               dt, t)
            for (j, s), arr in tr.items():
                out[key + f"_tr{j}{s}"] = arr
    save("predictor", **out)


def run_case(name, mesh, sysd, degree, cfl, ic, steps, boundary="periodic",
             use_limiter=False, store_first=False, predictor_mode="conservative",
             force_limit_all=False, exact_solution=None):
    sim = aderdg.Simulation(mesh, sysd, degree, cfl, boundary=boundary,
                            use_limiter=use_limiter, predictor_mode=predictor_mode,
                            exact_solution=exact_solution)
    sim.force_limit_all = force_limit_all
    u0 = sim.project_initial_condition(ic).copy()
    dts, iters, flags, fracs, lam = [], [], [], [], []
    orig = predictor.picard_solve

    def spy(*a, **k):
        r = orig(*a, **k)
        iters.append(r.iterations)
        return r

    predictor.picard_solve = spy
    first = None
    try:
        for _ in range(steps):
            lam.append([float(np.max(sysd.max_abs_eigenvalue(
                sim.u.reshape(-1, sysd.n_vars)[sysd.admissible(sim.u.reshape(-1, sysd.n_vars))],
                np.eye(mesh.dim)[j]))) for j in range(mesh.dim)])
            sim.run(np.inf, max_steps=sim.step_count + 1)
            dts.append(sim.history[-1]["dt"])
            fracs.append(sim.last_limited_fraction)
            if use_limiter:
                flags.append(np.asarray(sim.last_troubled, dtype=bool))
            if store_first and first is None:
                first = sim.u.copy()
    finally:
        predictor.picard_solve = orig
    arrays = dict(u0=u0, u=sim.u, dts=np.array(dts), iters=np.array(iters),
                  fracs=np.array(fracs), lam=np.array(lam),
                  totals=np.array([h["totals"] for h in sim.history]),
                  degree=np.array(degree), cfl=np.array(cfl),
                  cells=np.array(mesh.cells),
                  extents=np.array(mesh.extents))
    if use_limiter:
        arrays["troubled"] = np.stack(flags)
    if first is not None:
        arrays["u1"] = first
    save(name, **arrays)


def gen_cases():
    e2 = CompressibleEuler(2, gamma=GAMMA)
    e3 = CompressibleEuler(3, gamma=GAMMA)
    e1 = CompressibleEuler(1, gamma=GAMMA)
    # C1: full config (2-D vortex, 32^2, N=3, cfl 0.9/(2*7), 10 steps)
    ic, _ = problems.vortex()
    run_case("c1_vortex", aderdg.CartesianMesh([(0, 10), (0, 10)], (32, 32)), e2, 3,
             0.9 / 14.0, ic, 10, store_first=True)
    # C2 shape at oracle size: density wave N=4, 4^3, cfl 1/30, 3 steps
    ic, _ = problems.density_wave()
    run_case("c2_wave_4", wave_mesh((4, 4, 4)), e3, 4, 0.9 / 27.0, ic, 3,
             store_first=True)
    # C3 degree sweep at oracle size
    for n in range(2, 10):
        cells = (3, 3, 3) if n <= 5 else (2, 2, 2)
        run_case(f"c3_wave_N{n}", wave_mesh(cells), e3, n, 0.9 / (3 * (2 * n + 1)), ic, 2)
    # C4 shape at oracle size: circular explosion, N=5, limiter, outflow
    ic4, _ = problems.explosion()
    run_case("c4_explosion_16", aderdg.CartesianMesh([(-1, 1), (-1, 1)], (16, 16)), e2, 5,
             0.9 / 22.0, ic4, 6, boundary="outflow", use_limiter=True)
    # C5 weak-scaling domain: x extended to [0, 2], 4x2x2 cells (2 slabs of 2x2x2)
    run_case("c5_wave_ext", wave_mesh((4, 2, 2), extent_x=2.0), e3, 4, 0.9 / 27.0, ic, 2)
    # limiter in 1-D (Sod, outflow) and 2-D walls (blast) for rescue coverage
    ics, _ = problems.sod()
    run_case("sod_1d", aderdg.CartesianMesh([(0, 1)], (40,)), e1, 3, 0.09, ics, 12,
             boundary="outflow", use_limiter=True)
    icb, _ = problems.blast(p_ambient=1e-2)
    run_case("blast_wall", aderdg.CartesianMesh([(-1, 1), (-1, 1)], (12, 12)), e2, 2,
             0.15, icb, 4, boundary="wall", use_limiter=True)


def gen_primitive():
    """predictor_mode="primitive" (predictor.py:94-96, :109-112, :165-189;
    limiter.py:127-177): smooth, limited and near-vacuum cases."""
    e2 = CompressibleEuler(2, gamma=GAMMA)
    e1 = CompressibleEuler(1, gamma=GAMMA)
    e3 = CompressibleEuler(3, gamma=GAMMA)
    ic, _ = problems.vortex()
    run_case("prim_vortex", aderdg.CartesianMesh([(0, 10), (0, 10)], (16, 16)), e2, 3,
             0.9 / 14.0, ic, 4, predictor_mode="primitive")
    ic3, _ = problems.density_wave()
    run_case("prim_wave3d", wave_mesh((3, 3, 3)), e3, 4, 0.9 / 27.0, ic3, 2,
             predictor_mode="primitive")
    ics, _ = problems.sod()
    run_case("prim_sod", aderdg.CartesianMesh([(0, 1)], (40,)), e1, 3, 0.09, ics, 10,
             boundary="outflow", use_limiter=True, predictor_mode="primitive")
    # the reference's near-vacuum blast (test_acceptance.py:164-197 setup)
    icb, _ = problems.blast()
    run_case("prim_blast", aderdg.CartesianMesh([(-1, 1), (-1, 1)], (16, 16)), e2, 2, 0.15,
             icb, 4, boundary="wall", use_limiter=True, predictor_mode="primitive")


def gen_output():
    """Diagnostics / snapshot text of the reference writers (output.py) for a
    small Sod run (the determinism acceptance case, test_acceptance.py:354-366,
    at fewer steps) and a 2-D vortex state: formatting parity fixtures."""
    from aderdg import output
    e1 = CompressibleEuler(1, gamma=GAMMA)
    ics, _ = problems.sod()
    sim = aderdg.Simulation(aderdg.CartesianMesh([(0, 1)], (50,)), e1, 2, 0.15,
                            boundary="outflow", use_limiter=True)
    sim.project_initial_condition(ics)
    sim.run(np.inf, max_steps=8)
    hist = sim.history
    arrays = dict(
        steps=np.array([h["step"] for h in hist]), times=np.array([h["time"] for h in hist]),
        dts=np.array([h["dt"] for h in hist]), totals=np.array([h["totals"] for h in hist]),
        fracs=np.array([h["limited_fraction"] for h in hist]),
        diag_csv=np.array(output.diagnostics_csv(hist, e1.quantity_names)),
        u=sim.u, t=np.array(sim.t), step_count=np.array(sim.step_count),
        fields_csv=np.array(output.fields_csv(sim)), fields_vtk=np.array(output.fields_vtk(sim)),
        names=np.array(e1.quantity_names))
    e2 = CompressibleEuler(2, gamma=GAMMA)
    ic, _ = problems.vortex()
    sim2 = aderdg.Simulation(aderdg.CartesianMesh([(0, 10), (0, 10)], (4, 3)), e2, 2, 0.1)
    sim2.project_initial_condition(ic)
    sim2.run(np.inf, max_steps=1)
    arrays.update(u2=sim2.u, t2=np.array(sim2.t), vtk2=np.array(output.fields_vtk(sim2)),
                  csv2=np.array(output.fields_csv(sim2)),
                  tdu=np.array(aderdg.kernels.throughput_per_dof(1.25, 4096, 20, 4, 3)))
    save("output_sod", **arrays)


def static_exact(ic):
    """A time-independent "exact" solution (Dirichlet data = the IC)."""
    return lambda x, t: ic(x)


def gen_exact():
    """"exact" faces (driver.py:250-261, :317-340): a 2-D density wave with
    its true translating solution on every face (unlimited), and a limited
    explosion whose Dirichlet data is the static IC, mixed with outflow and
    wall faces so ghost corners combine exact with other kinds."""
    e2 = CompressibleEuler(2, gamma=GAMMA)
    ic, ex = problems.density_wave(vel=(1.0, 0.5))
    sim = aderdg.Simulation(aderdg.CartesianMesh([(0, 1), (0, 1)], (8, 6)), e2, 3, 0.9 / 14.0,
                            boundary="exact", exact_solution=ex)
    u0 = sim.project_initial_condition(ic).copy()
    sim.run(np.inf, max_steps=5)
    save("exact_wave2d", u0=u0, u=sim.u, dts=np.array([h["dt"] for h in sim.history]),
         degree=np.array(3), cfl=np.array(0.9 / 14.0), cells=np.array(sim.mesh.cells),
         extents=np.array(sim.mesh.extents))
    ic4, _ = problems.explosion()
    bnd = {0: ("exact", "outflow"), 1: ("wall", "exact")}
    sim = aderdg.Simulation(aderdg.CartesianMesh([(-0.8, 0.8), (-0.8, 0.8)], (12, 12)), e2, 2,
                            0.15, boundary=bnd, use_limiter=True,
                            exact_solution=static_exact(ic4))
    u0 = sim.project_initial_condition(ic4).copy()
    flags = []
    for _ in range(8):
        sim.run(np.inf, max_steps=sim.step_count + 1)
        flags.append(np.asarray(sim.last_troubled, dtype=bool))
    save("exact_explosion", u0=u0, u=sim.u, dts=np.array([h["dt"] for h in sim.history]),
         troubled=np.stack(flags), degree=np.array(2), cfl=np.array(0.15),
         cells=np.array(sim.mesh.cells), extents=np.array(sim.mesh.extents))


def gen_advection():
    """LinearAdvection plugin (systems.py:77-109) with the registry's sine /
    pulse / step initial conditions (problems.py:54-93), periodic, outflow
    and wall faces, degrees 2..9, d = 1..3."""
    from aderdg.systems import LinearAdvection

    def case(name, ext, cells, vel, degree, prob, steps, boundary="periodic"):
        sysd = LinearAdvection(len(cells), velocity=vel)
        ic, _ = aderdg.build_problem(prob, sysd)
        cfl = 0.9 / (len(cells) * (2 * degree + 1))
        run_case(name, aderdg.CartesianMesh(ext, cells), sysd, degree, cfl, ic, steps,
                 boundary=boundary)

    case("adv_sine_2d", [(0, 1), (0, 1)], (8, 6), [1.0, 0.5], 3, "sine", 6)
    case("adv_sine_3d", [(0, 1)] * 3, (3, 3, 2), [1.0, -0.5, 0.3], 2, "sine", 4)
    case("adv_sine_3d_N5", [(0, 1)] * 3, (2, 2, 2), [0.6, 0.8, -0.4], 5, "sine", 2)
    case("adv_sine_2d_N9", [(0, 1), (0, 1)], (3, 2), [1.0, -0.7], 9, "sine", 3)
    case("adv_pulse_1d", [(0, 1)], (20,), [1.0], 5, "pulse", 8, boundary="outflow")
    case("adv_step_wall_2d", [(0, 1), (0, 1)], (6, 6), [0.7, -0.4], 4, "step", 4,
         boundary="wall")


def gen_advection_limited():
    """LinearAdvection with the subcell limiter, primitive mode and exact faces
    (the reference's own limiter-in-driver cases, test_mesh_driver.py:396-432,
    plus 2-D / wall / exact variants)."""
    from aderdg.driver import default_cfl
    from aderdg.systems import LinearAdvection

    def case(name, ext, cells, vel, degree, prob, steps, boundary="periodic", force=False,
             mode="conservative", exact=False):
        sysd = LinearAdvection(len(cells), velocity=vel)
        ic, ex = aderdg.build_problem(prob, sysd)
        run_case(name, aderdg.CartesianMesh(ext, cells), sysd, degree, default_cfl(degree), ic,
                 steps, boundary=boundary, use_limiter=True, force_limit_all=force,
                 predictor_mode=mode, exact_solution=ex if exact else None)

    case("adv_lim_step_1d", [(0, 1)], (50,), [1.0], 2, "step", 30)
    case("adv_lim_sine_forced", [(0, 1)], (16,), [1.0], 2, "sine", 5, force=True)
    case("adv_lim_step_wall_2d", [(0, 1), (0, 1)], (12, 10), [0.7, -0.4], 3, "step", 8,
         boundary="wall")
    case("adv_lim_step_prim_2d", [(0, 1), (0, 1)], (10, 8), [0.6, 0.5], 2, "step", 6,
         mode="primitive")
    case("adv_lim_pulse_exact_1d", [(0, 1)], (24,), [1.0], 4, "pulse", 12,
         boundary={0: ("exact", "outflow")}, exact=True)
    case("adv_lim_step_3d", [(0, 1)] * 3, (5, 4, 4), [1.0, 0.5, -0.3], 2, "step", 4)


def gen_elasticity():
    """DiffuseInterfaceElasticity plugin (systems.py:237-345): the registry's
    P-wave toward the diffuse free surface (problems.py:135-173) with
    outflow and wall faces, and a periodic constant state (problems.py:
    176-192), degrees 2..5 (the NCP /
    path-conservative machinery of corrector.py:65-129)."""
    from aderdg.systems import DiffuseInterfaceElasticity

    sysd = DiffuseInterfaceElasticity(2)

    def case(name, cells, degree, prob, steps, boundary, ext=((0.0, 1.0), (0.0, 0.25))):
        ic, _ = aderdg.build_problem(prob, sysd)
        cfl = 0.9 / (2 * (2 * degree + 1))
        run_case(name, aderdg.CartesianMesh([tuple(e) for e in ext], cells), sysd, degree, cfl,
                 ic, steps, boundary=boundary)

    case("el_pwave", (16, 4), 3, "pwave", 8, "outflow")
    case("el_pwave_N5", (8, 2), 5, "pwave", 4, "outflow")
    case("el_pwave_wall", (12, 3), 2, "pwave", 6, "wall")
    case("el_constant", (4, 4), 3, "constant", 3, "periodic", ext=((0.0, 1.0), (0.0, 1.0)))


def gen_plugins():
    """Plugin-contract methods (systems.py:16-74, :158-223, :269-318) on seeded
    states: Euler eigenvalues / cons_to_prim / prim_to_cons / primitive_rhs,
    advection eigenvalues / primitive_rhs, elasticity ncp / ncp_matrix."""
    from aderdg.systems import DiffuseInterfaceElasticity, HyperbolicSystem, LinearAdvection

    out = {}
    rng = np.random.default_rng(77)
    for d in (1, 2, 3):
        sysd = CompressibleEuler(d, gamma=GAMMA)
        q = euler_states(d, 64, seed=30 + d)
        grad = rng.uniform(-1, 1, (64, d, d + 2))
        normal = rng.uniform(-1, 1, d)
        out[f"e{d}_q"] = q
        out[f"e{d}_grad"] = grad
        out[f"e{d}_normal"] = normal
        out[f"e{d}_eig"] = sysd.eigenvalues(q, normal)
        out[f"e{d}_prim"] = sysd.cons_to_prim(q)
        out[f"e{d}_cons"] = sysd.prim_to_cons(sysd.cons_to_prim(q))
        out[f"e{d}_prim_rhs"] = sysd.primitive_rhs(sysd.cons_to_prim(q), grad)
        adv = LinearAdvection(d, velocity=rng.uniform(-1, 1, d))
        qa = rng.uniform(-1, 1, (16, 1))
        ga = rng.uniform(-1, 1, (16, d, 1))
        out[f"a{d}_vel"] = adv.velocity
        out[f"a{d}_q"] = qa
        out[f"a{d}_grad"] = ga
        out[f"a{d}_eig"] = adv.eigenvalues(qa, normal)
        out[f"a{d}_prim_rhs"] = adv.primitive_rhs(qa, ga)
    el = DiffuseInterfaceElasticity(2)
    qe = rng.uniform(0.2, 2.0, (64, 9))
    qe[:8, el.ALPHA] = rng.uniform(0.0, 2e-3, 8)   # below / around the floor
    ge = rng.uniform(-1, 1, (64, 2, 9))
    ne = np.array([0.6, -0.8])
    out["el_q"] = qe
    out["el_grad"] = ge
    out["el_normal"] = ne
    out["el_ncp"] = el.ncp(qe, ge)
    out["el_ncp_matrix"] = el.ncp_matrix(qe, ne)
    out["el_prim_rhs"] = el.primitive_rhs(qe, ge)
    out["el_eig"] = el.eigenvalues(qe, ne)
    base = HyperbolicSystem(2, 3, ("a", "b", "c"))
    out["base_flux"] = base.flux(qe[:4, :3])
    out["base_ncp_matrix"] = base.ncp_matrix(qe[:4, :3], ne)
    save("plugins", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tables", "pointwise", "predictor", "cases", "primitive", "output",
                             "exact", "advection", "elasticity", "plugins",
                             "advection_limited"]
    if "plugins" in which:
        gen_plugins()
    if "advection_limited" in which:
        gen_advection_limited()
    if "elasticity" in which:
        gen_elasticity()
    if "advection" in which:
        gen_advection()
    if "tables" in which:
        gen_tables()
    if "pointwise" in which:
        gen_pointwise()
    if "predictor" in which:
        gen_predictor()
    if "cases" in which:
        gen_cases()
    if "primitive" in which:
        gen_primitive()
    if "output" in which:
        gen_output()
    if "exact" in which:
        gen_exact()
