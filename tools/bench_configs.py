#!/usr/bin/env python
"""Throughput of every BASELINE config shape on one B200 (supplement to
bench.py, whose single JSON line is C2).  Prints one JSON object per case:

  C1  2-D vortex 32^2, N=3, 10 steps
  C2  3-D density wave 64^3, N=4, 20 steps
  C3  3-D density wave 32^3, N=2..9, 10 steps each
  C4  2-D circular explosion 512^2, N=5, limiter, to the stated t = 0.25
      (--c4-steps K > 0: only the first K steps)

DOF-updates/s = E (N+1)^d steps / t, t from CUDA events around
Simulation.run (the bench-tdu scope, cli.py:79-91), after 3 warm-up steps.
nvidia-smi clocks and throttle reasons are sampled during every timed region
(bench.ClockSampler).  The roofline uses the mean Picard sweeps actually
executed; for the limited C4 run it is the unlimited-step
work model (the rescue of the troubled cells comes on top of it).
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1808_03788_b200 as pkg  # noqa: E402
from bench import ClockSampler, load_peaks  # noqa: E402
from paper_1808_03788_b200 import roofline  # noqa: E402

PEAKS = load_peaks()


def run_case(name, ext, cells, degree, cfl, problem, steps, boundary="periodic",
             limiter=False, warmup=3, t_end=np.inf):
    d = len(cells)
    system = pkg.make_system("euler", d)
    sim = pkg.Simulation(pkg.CartesianMesh(ext, cells), system, degree, cfl,
                         boundary=boundary, use_limiter=limiter)
    sim.project_initial_condition(pkg.build_problem(problem, system)[0])
    sim.run(t_end, max_steps=warmup)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        w0 = time.perf_counter()
        a.record()
        sim.run(t_end, max_steps=(warmup + steps) if steps else None)
        b.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    ms = a.elapsed_time(b)
    n = sim.step_count - warmup
    dofs = sim.mesh.n_elements * (degree + 1) ** d * n
    sweeps = [s for s in sim.sweep_log[warmup:] if s is not None]
    out = {"case": name, "cells": list(cells), "degree": degree, "steps": n,
           "ms_per_step": ms / n, "dof_per_s": dofs / (ms * 1e-3),
           "wall_dof_per_s": dofs / wall, "picard_sweeps_max": max(sweeps) if sweeps else None,
           "clocks": clocks.summary()}
    if limiter:
        fr = [h["limited_fraction"] for h in sim.history[warmup:]]
        out["limited_fraction_mean"] = float(np.mean(fr))
        out["t"] = sim.t
    s = float(np.mean(sweeps))
    fl = roofline.step_flops_per_dof(degree, d, s)
    by = roofline.step_bytes_per_dof(degree, d)
    out["picard_sweeps_mean"] = s
    out["flop_per_dof"] = fl
    out["flop_per_byte"] = fl / by
    out["step_roofline_dof_per_s"] = roofline.roofline_dofs(
        degree, d, s, PEAKS["fp64_dfma_tflops"] * 1e12, PEAKS["hbm_gbs"] * 1e9)
    out["step_roofline_frac"] = out["dof_per_s"] / out["step_roofline_dof_per_s"]
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4")
    ap.add_argument("--c4-steps", type=int, default=0, help="0: run to t = 0.25")
    ap.add_argument("--c3-cells", type=int, default=32)
    ap.add_argument("--c4-cells", type=int, default=512)
    ap.add_argument("--c3-degrees", default="2,3,4,5,6,7,8,9")
    args = ap.parse_args()
    which = set(args.only.split(","))
    if "C1" in which:
        run_case("C1", [(0.0, 10.0), (0.0, 10.0)], (32, 32), 3, 0.9 / 14.0, "vortex", 10)
    if "C2" in which:
        run_case("C2", [(0.0, 1.0)] * 3, (64, 64, 64), 4, 0.9 / 27.0, "density_wave", 20)
    if "C3" in which:
        n3 = args.c3_cells
        for n in [int(x) for x in args.c3_degrees.split(",")]:
            run_case(f"C3_N{n}", [(0.0, 1.0)] * 3, (n3,) * 3, n, 0.9 / (3 * (2 * n + 1)),
                     "density_wave", 10)
    if "C4" in which:
        n4 = args.c4_cells
        run_case("C4", [(-1.0, 1.0), (-1.0, 1.0)], (n4, n4), 5, 0.9 / 22.0, "explosion",
                 args.c4_steps, boundary="outflow", limiter=True, t_end=0.25)


if __name__ == "__main__":
    main()
