"""Diagnose troubled-flag mismatches of C4 at 512^2 against the reference
fixture: which step, which cells, and whether the Picard sweep rule matters."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1808_03788_b200 as pkg  # noqa: E402

g = dict(np.load("tests/golden/c4_explosion_512_2.npz"))
n = int(g["n_cells"])
ref = np.unpackbits(g["troubled_bits"], axis=1)[:, :n].astype(bool)
for mi in (() if len(sys.argv) > 1 else (1, 11)):
    mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
    system = pkg.make_system("euler", 2)
    sim = pkg.Simulation(mesh, system, 5, float(g["cfl"]), boundary="outflow", use_limiter=True,
                         min_picard_iter=mi)
    sim.project_initial_condition(pkg.build_problem("explosion", system)[0])
    for k in (1, 2):
        sim.run(np.inf, max_steps=k)
        f = sim.last_troubled.cpu().numpy().ravel()
        bad = np.flatnonzero(f != ref[k - 1])
        print(f"min_iter={mi} step {k}: ours {f.sum()} ref {ref[k-1].sum()} mismatches {bad.size}"
              f" cells {[(int(b) // 512, int(b) % 512, bool(f[b])) for b in bad[:12]]}"
              f" sweeps {sim.sweep_log[-1]} dt {sim.history[-1]['dt']!r} ref dt {g['dts'][k-1]!r}",
              flush=True)


def dmp_margin(pkg, sim, u_prev, cand, cells, delta0=1e-3, eps=1e-3):
    """Signed distance of each cell's candidate subcell averages to its relaxed
    DMP interval (limiter.py:51-86): min over subcells and quantities of
    min(c - (lo - delta), (hi + delta) - c); negative = troubled."""
    t = sim.tables
    Ps = np.asarray(t.sub_project)
    up = u_prev.cpu().numpy()
    cd = cand.cpu().numpy()
    nx, ny = up.shape[:2]
    out = []
    for (i, j) in cells:
        def sub(a, ii, jj):
            return np.einsum("ak,bl,klv->abv", Ps, Ps, a[ii, jj])
        nb = [(i, j)] + [(i + di, j + dj) for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1))]
        vals = np.concatenate([sub(up, *c).reshape(-1, up.shape[-1]) for c in nb
                               if 0 <= c[0] < nx and 0 <= c[1] < ny])
        lo, hi = vals.min(axis=0), vals.max(axis=0)
        d = np.maximum(delta0, eps * (hi - lo))
        c = sub(cd, i, j).reshape(-1, up.shape[-1])
        out.append(float(np.min(np.minimum(c - (lo - d), (hi + d) - c))))
    return out


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "margin":
    import math
    mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
    system = pkg.make_system("euler", 2)
    sim = pkg.Simulation(mesh, system, 5, float(g["cfl"]), boundary="outflow", use_limiter=True)
    sim.project_initial_condition(pkg.build_problem("explosion", system)[0])
    sim.run(np.inf, max_steps=1)
    u1 = sim.u.clone()
    row = torch.zeros(6, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    sim._timestep_into(row[0:1], st, math.inf)
    sim._attempt_limited_device(row)
    torch.cuda.synchronize()
    bad = [(157, 172), (157, 339), (172, 157), (172, 354), (339, 157), (339, 354), (354, 172),
           (354, 339)]
    print("margins of the mismatched cells:", dmp_margin(pkg, sim, u1, sim._u_next, bad))
    # troubled cells near them for scale
    f = sim._lim["troubled"].cpu().numpy()
    print("ours flags there:", [int(f[c]) for c in bad])


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "pred":
    import math

    from oracle import dg
    from oracle.basis import oracle_tables
    from oracle.euler import EulerOracle
    from paper_1808_03788_b200 import predictor as pr
    mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
    system = pkg.make_system("euler", 2)
    sim = pkg.Simulation(mesh, system, 5, float(g["cfl"]), boundary="outflow", use_limiter=True)
    sim.project_initial_condition(pkg.build_problem("explosion", system)[0])
    sim.run(np.inf, max_steps=1)
    dt2 = sim.max_timestep()
    bad = [(157, 172), (157, 339), (172, 157), (172, 354), (339, 157), (339, 354), (354, 172),
           (354, 339)]
    u = np.stack([sim.u[i, j].cpu().numpy() for i, j in bad])
    for mi in (1, 9, 12):
        res = pr.picard_solve(u, system, mesh.spacings, dt2, sim.tables, min_iter=mi,
                              sweep_rule="element")
        q = res.q.cpu().numpy()
        p = 0.4 * (q[..., 3] - 0.5 * (q[..., 1] ** 2 + q[..., 2] ** 2) / q[..., 0])
        print(f"ours min_iter={mi}: sweeps {res.sweeps.tolist()} conv {res.converged.tolist()} "
              f"adm {res.admissible.tolist()} min p {p.reshape(8, -1).min(axis=1)} "
              f"min rho {q[..., 0].reshape(8, -1).min(axis=1)}")
    ref = dg.picard_solve(u, EulerOracle(2), mesh.spacings, dt2, oracle_tables(5))
    qo = ref.q
    po = 0.4 * (qo[..., 3] - 0.5 * (qo[..., 1] ** 2 + qo[..., 2] ** 2) / qo[..., 0])
    print(f"oracle: iters {ref.iterations} conv {ref.converged.tolist()} adm "
          f"{ref.admissible.tolist()} min p {po.reshape(8, -1).min(axis=1)}")
    ref9 = dg.picard_solve(u, EulerOracle(2), mesh.spacings, dt2, oracle_tables(5), max_iter=9,
                           tol=0.0)
    print(f"oracle 9 sweeps: adm {ref9.admissible.tolist()}")
    print("rel diff ours vs oracle q:", np.abs(q - qo).max() / np.abs(qo).max())
