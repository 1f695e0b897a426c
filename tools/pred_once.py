#!/usr/bin/env python
"""Run the C2 shape (64^3, N=4 density wave, or AB_CELLS / AB_DEG) for a few
steps through the library selected by ADG_LIB (default: the in-tree build):
a short, deterministic command to put under ncu
(`-k regex:predict_kernel -s 2 -c 1`).  Development tool."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_03788_b200 as pkg  # noqa: E402

n = int(os.environ.get("AB_CELLS", "64"))
deg = int(os.environ.get("AB_DEG", "4"))
steps = int(os.environ.get("AB_STEPS", "3"))
system = pkg.make_system("euler", 3)
cfl = 0.9 / (3 * (2 * deg + 1))
sim = pkg.Simulation(pkg.CartesianMesh([(0, 1)] * 3, (n, n, n)), system, deg, cfl)
sim.project_initial_condition(pkg.build_problem("density_wave", system)[0])
sim.run(np.inf, max_steps=steps)
torch.cuda.synchronize()
print("ok", n, deg, steps, float(sim.t))
