#!/usr/bin/env python
"""A/B timing of library builds on the C2 shape (64^3, N=4): the fused
predictor alone and the full step.  Usage:

    python tools/pred_ab.py lib1.so lib2.so ...

Each library runs in its own process (ADG_LIB selects it); prints one JSON
line per library.  Development tool, not part of the bench contract.
"""

import json
import os
import subprocess
import sys

CHILD = r'''
import json, sys, os, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1808_03788_b200 as pkg
from paper_1808_03788_b200.predictor import run_predictor
n = int(os.environ.get("AB_CELLS", "64")); deg = int(os.environ.get("AB_DEG", "4"))
system = pkg.make_system("euler", 3)
cfl = 0.9 / (3 * (2 * deg + 1))
sim = pkg.Simulation(pkg.CartesianMesh([(0, 1)] * 3, (n, n, n)), system, deg, cfl)
sim.project_initial_condition(pkg.build_problem("density_wave", system)[0])
sim.run(np.inf, max_steps=2)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
K = 10
a.record(); sim.run(np.inf, max_steps=2 + K); b.record(); torch.cuda.synchronize()
step_ms = a.elapsed_time(b) / K
u = sim.u.contiguous()
dt = sim.history[-1]["dt"]
tabs = pkg.basis_tables(deg)
from paper_1808_03788_b200 import _lib
from paper_1808_03788_b200.predictor import _grid
h = _lib.Handle.get(u.device.index)
h.ensure_tables(tabs)
g = _grid(system, n ** 3, sim.mesh.spacings, deg)
E = n ** 3; pd = (deg + 1) ** 3; m = 5
tb = pd * m + ((pd * m) & 1)
f64 = dict(dtype=torch.float64, device=u.device)
vol = torch.empty(u.shape, **f64); tr = torch.empty(6, E, tb, **f64)
bad = torch.empty(E, dtype=torch.uint8, device=u.device)
sw = torch.empty(E, dtype=torch.int32, device=u.device)
dtd = torch.full((1,), float(dt), **f64)
def launch():
    h.call("adg_predict", _lib.ctypes.byref(g), u.data_ptr(), dtd.data_ptr(), 1e-12, 0, 1, None,
           vol.data_ptr(), tr.data_ptr(), bad.data_ptr(), sw.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    launch()
torch.cuda.synchronize()
ts = []
for _ in range(7):
    a.record(); launch(); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
chk = [float(vol.double().sum().item()), float(tr[:, :, :pd * m].sum().item()), int(sw.sum().item()), int(bad.sum().item())]
print(json.dumps({"lib": os.path.basename(os.environ["ADG_LIB"]), "chk": chk, "step_ms": step_ms, "pred_ms_min": min(ts),
                  "pred_ms_med": sorted(ts)[3], "cells": n, "degree": deg}))
'''

for lib in sys.argv[1:]:
    env = dict(os.environ, ADG_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    out = r.stdout.strip().splitlines()
    print(out[-1] if out else json.dumps({"lib": lib, "error": r.stderr[-800:]}), flush=True)
