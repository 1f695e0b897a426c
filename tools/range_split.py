"""Cost of splitting the predictor into the slab schedule's three element
ranges (first x-layer, last x-layer, interior; SlabSimulation._predict_exchange)
vs one whole-grid launch, on one GPU.  Usage: python tools/range_split.py [n]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_03788_b200 as pkg  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    system = pkg.make_system("euler", 3)
    mesh = pkg.CartesianMesh([(0.0, 1.0)] * 3, (n, n, n))
    sim = pkg.Simulation(mesh, system, 4, 0.9 / 27)
    sim.project_initial_condition(pkg.build_problem("density_wave", system)[0])
    sim._ensure_buffers()
    dt = torch.tensor([sim.max_timestep()], dtype=torch.float64, device=sim.device)
    E = mesh.n_elements
    layer = E // n

    def whole():
        sim._predict(dt)

    def split():
        sim._predict_part(dt, 0, layer)
        sim._predict_part(dt, E - layer, layer)
        sim._predict_part(dt, layer, E - 2 * layer)

    out = {"cells": n}
    for name, fn in (("whole", whole), ("split", split), ("whole2", whole), ("split2", split)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            fn()
        b.record()
        torch.cuda.synchronize()
        out[name + "_ms"] = a.elapsed_time(b) / 5
    print(json.dumps(out))


if __name__ == "__main__":
    main()
