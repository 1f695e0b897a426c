"""C1 (2-D vortex 32^2, N=3) ms/step against the batched CUDA graph's unroll
length (Simulation.graph_steps); history rows must be bitwise equal."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_03788_b200 as pkg  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 192
ref = None
for n in (2, 4, 8, 16, 32, 64):
    system = pkg.make_system("euler", 2)
    sim = pkg.Simulation(pkg.CartesianMesh([(0.0, 10.0), (0.0, 10.0)], (32, 32)), system, 3,
                         0.9 / 14)
    sim.graph_steps = n
    sim.project_initial_condition(pkg.build_problem("vortex", system)[0])
    sim.run(np.inf, max_steps=2 * n)         # warm-up: captures both graphs
    torch.cuda.synchronize()
    best = []
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0 = sim.step_count
        a.record()
        sim.run(np.inf, max_steps=k0 + steps)
        b.record()
        torch.cuda.synchronize()
        best.append(a.elapsed_time(b) / (sim.step_count - k0))
    u = sim.state.cpu().numpy() if hasattr(sim, "state") else None
    rows = np.array([[h["dt"], h["time"], *h["totals"]] for h in sim.history])
    L = min(len(rows), len(ref)) if ref is not None else 0
    same = None if ref is None else bool(np.array_equal(rows[:L], ref[:L]))
    if ref is None:
        ref = rows
    print(json.dumps({"graph_steps": n, "ms_per_step": min(best), "all": best,
                      "history_bitwise_equal_to_2": same}), flush=True)
