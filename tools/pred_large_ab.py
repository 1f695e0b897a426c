#!/usr/bin/env python
"""A/B timing of the 3-D large-tile predictors (N = 7..9, 32^3 by default):
ADG_PREDICTOR unset (phase kernels) against ADG_PREDICTOR=stream (fused
slice-streaming kernel); predictor alone and the full step, plus output
checksums.  Development tool.  Usage: python tools/pred_large_ab.py [N ...]"""

import json
import os
import subprocess
import sys

CHILD = r'''
import json, sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1808_03788_b200 as pkg
n = int(os.environ.get("AB_CELLS", "32")); deg = int(os.environ["AB_DEG"])
system = pkg.make_system("euler", 3)
cfl = 0.9 / (3 * (2 * deg + 1))
sim = pkg.Simulation(pkg.CartesianMesh([(0, 1)] * 3, (n, n, n)), system, deg, cfl)
sim.project_initial_condition(pkg.build_problem("density_wave", system)[0])
sim.run(np.inf, max_steps=2)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
K = 4
a.record(); sim.run(np.inf, max_steps=2 + K); b.record(); torch.cuda.synchronize()
step_ms = a.elapsed_time(b) / K
u = sim.u.contiguous()
dt = sim.history[-1]["dt"]
tabs = pkg.basis_tables(deg)
from paper_1808_03788_b200 import _lib
from paper_1808_03788_b200.predictor import _grid
h = sim._h if hasattr(sim, "_h") else _lib.Handle.get(u.device.index)
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
for _ in range(5):
    a.record(); launch(); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
chk = [float(vol.sum().item()), float(tr[:, :, :pd * m].sum().item()), int(sw.sum().item()), int(bad.sum().item()),
       float(sim.u.sum().item())]
print(json.dumps({"predictor": os.environ.get("ADG_PREDICTOR", "phased"), "degree": deg, "cells": n,
                  "step_ms": step_ms, "pred_ms_min": min(ts), "chk": chk}))
'''

# usage: pred_large_ab.py [N ...] [-- variant ...]; a variant is "phased" or
# "stream" (ADG_PREDICTOR), optionally followed by ":path of a library build"
args = sys.argv[1:]
variants = ["phased", "stream"]
if "--" in args:
    k = args.index("--")
    args, variants = args[:k], args[k + 1:]
degs = [int(x) for x in args] or [7, 8, 9]
for deg in degs:
    for var in variants:
        env = dict(os.environ, AB_DEG=str(deg))
        env.pop("ADG_PREDICTOR", None)
        env.pop("ADG_LIB", None)
        # "phased" / "stream", optionally ":library path"
        kind, _, lib = var.partition(":")
        env["ADG_PREDICTOR"] = kind
        if lib:
            env["ADG_LIB"] = os.path.abspath(lib)
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        out = r.stdout.strip().splitlines()
        if out:
            d = json.loads(out[-1]); d["variant"] = os.path.basename(var)
            print(json.dumps(d), flush=True)
        else:
            print(json.dumps({"deg": deg, "variant": var, "error": r.stderr[-1500:]}), flush=True)
