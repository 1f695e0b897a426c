"""Rounding sensitivity of C4 (64^2, N=5, outflow, limiter) to t = 0.25: two
runs of this implementation from initial states that differ by 1e-15
relative (seeded), compared every 50 steps.  Shows whether the end-state
difference against the reference (corner cells) is the amplification of
last-bit differences at the outflow corners rather than an implementation
difference."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1808_03788_b200 as pkg  # noqa: E402

g = dict(np.load("tests/golden/c4_explosion_64_full.npz"))
mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
system = pkg.make_system("euler", 2)


def make(eps):
    sim = pkg.Simulation(mesh, system, 5, float(g["cfl"]), boundary="outflow", use_limiter=True)
    sim.project_initial_condition(pkg.build_problem("explosion", system)[0])
    if eps:
        rng = np.random.default_rng(0)
        u = sim.u.cpu().numpy()
        sim.set_state(u * (1.0 + eps * rng.uniform(-1, 1, u.shape)))
    return sim


a, b = make(0.0), make(1e-15)
rows = []
t_marks = np.linspace(0.0, 0.25, 11)[1:]
for tm in t_marks:
    a.run(tm)
    b.run(tm)
    d = (a.u - b.u).abs().reshape(64, 64, -1).amax(dim=2).cpu().numpy()
    ur = g["u"] if abs(tm - 0.25) < 1e-15 else None
    row = {"t": float(tm), "steps": a.step_count, "max_diff": float(d.max()),
           "corner_diff": float(max(d[0, 0], d[0, 63], d[63, 0], d[63, 63])),
           "interior_diff": float(d[8:56, 8:56].max()),
           "corner_rho_dev": float(abs(a.u[0, 0, :, :, 0].mean().item() - 0.125))}
    if ur is not None:
        row["vs_reference_max"] = float(np.abs(a.u.cpu().numpy() - ur).max())
        row["vs_reference_interior"] = float(
            np.abs(a.u.cpu().numpy() - ur)[8:56, 8:56].max())
    rows.append(row)
    print(json.dumps(row), flush=True)
