import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1808_03788_b200 as pkg
system = pkg.make_system("euler", 2)
sim = pkg.Simulation(pkg.CartesianMesh([(0.0, 10.0), (0.0, 10.0)], (32, 32)), system, 3, 0.9/14)
sim.project_initial_condition(pkg.build_problem("vortex", system)[0])
sim.run(np.inf, max_steps=3)
torch.cuda.synchronize()
sim.run(np.inf, max_steps=13)
torch.cuda.synchronize()
print("ok")
