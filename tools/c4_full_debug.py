"""Where does the C4 64^2 t=0.25 state differ from the reference fixture?"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1808_03788_b200 as pkg  # noqa: E402

g = dict(np.load("tests/golden/c4_explosion_64_full.npz"))
n = int(g["n_cells"])
ref_flags = np.unpackbits(g["troubled_bits"], axis=1)[:, :n].astype(bool)
mesh = pkg.CartesianMesh([tuple(e) for e in g["extents"]], [int(c) for c in g["cells"]])
system = pkg.make_system("euler", 2)
sim = pkg.Simulation(mesh, system, 5, float(g["cfl"]), boundary="outflow", use_limiter=True)
sim.project_initial_condition(pkg.build_problem("explosion", system)[0])
ever = np.zeros(n, bool)
def cb(s):
    ever[:] |= s.last_troubled.cpu().numpy().ravel()
sim.run(0.25, on_step=cb)
u = sim.u.cpu().numpy()
err = np.abs(u - g["u"]).reshape(64, 64, -1).max(axis=2)
order = np.argsort(err.ravel())[::-1][:15]
print("max err", err.max(), "scale", np.abs(g["u"]).max())
for k in order:
    i, j = divmod(int(k), 64)
    print(i, j, f"{err[i, j]:.3e}", "ever troubled" if ever[k] else "")
print("cells with err > 1e-10:", int((err > 1e-10).sum()), "of", n)
print("err rows (max over j):", np.array2string(err.max(axis=1), precision=1))
tot = np.array([h["totals"] for h in sim.history])
d = np.abs(tot - g["totals"]).max(axis=1)
first = np.flatnonzero(d > 1e-12)
print("first step with totals diff > 1e-12:", first[:5] + 1, d[first[:5]] if first.size else "")
dts = np.array([h["dt"] for h in sim.history])
rd = np.abs(dts - g["dts"]) / g["dts"]
print("dt rel diff first > 1e-13 at step", (np.flatnonzero(rd > 1e-13)[:5] + 1), rd.max())
