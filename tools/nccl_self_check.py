"""Step-by-step check of the C-ABI NCCL transport on a one-rank communicator."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1808_03788_b200 as pkg  # noqa: E402
from paper_1808_03788_b200.decomp import SlabSimulation  # noqa: E402


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


gmesh = pkg.CartesianMesh([(0.0, 1.0)] * 3, (8, 6, 5))
system = pkg.make_system("euler", 3)
cfl = 0.9 / 27
ic, _ = pkg.build_problem("density_wave", system, velocity=[1.0, -0.5, 0.3])
log("create")
sim = SlabSimulation(gmesh, system, 4, cfl, self_exchange=True)
log("comm ok", sim.transport)
sim.project_initial_condition(ic)
sim._ensure_buffers()
buf = sim._buf
red = buf.red[0]
sim._wavespeed()
sim._comm.allreduce_record(buf.red[0], sim._h.stream())
torch.cuda.synchronize()
log("allreduce_record ok", buf.red[0].tolist())
t = torch.ones(7, dtype=torch.float64, device="cuda")
sim._comm.allreduce_sum(t, sim._h.stream())
torch.cuda.synchronize()
log("allreduce_sum ok", t.tolist())
buf.traces.normal_()
sim._comm.halo_exchange(sim._gp(), buf.traces, sim._ghost[(0, 0)], sim._ghost[(0, 1)],
                        sim._h.stream())
torch.cuda.synchronize()
n = sim._ghost[(0, 0)].numel()
face = sim.mesh.n_elements * buf.tb
ok = (torch.equal(sim._ghost[(0, 1)], buf.traces[0:n]) and
      torch.equal(sim._ghost[(0, 0)], buf.traces[2 * face - n:2 * face]))
log("halo eager ok", ok)
sim.overlap_halos = False
sim.graphs_enabled = False
sim.run(np.inf, max_steps=2)
log("run eager no-overlap ok")
sim.overlap_halos = True
sim.run(np.inf, max_steps=4)
log("run eager overlap ok")
sim.graphs_enabled = True
sim.run(np.inf, max_steps=8)
log("run graphs ok")
sim.close(); log("closed")
