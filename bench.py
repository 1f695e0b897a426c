#!/usr/bin/env python
"""Benchmark: DOF-updates/s (1/TDU) of the 3-D Euler ADER-DG N=4 time step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 runs BASELINE config C2 (64^3 elements, N=4, smooth density wave,
periodic unit cube, cfl = 0.9/(3(2N+1)) = 1/30).  With N>1 (launched under
torchrun, or `--gpus N` alone: bench.py then starts the N ranks itself
through torch.distributed.run on 127.0.0.1) it runs BASELINE config C5:

* weak scaling (default): every rank owns 128^3 elements of the x-extended
  domain [0, N] x [0, 1]^2 (dx = 1/128 at every N);
* `--scaling strong`: the fixed 256^3 unit cube, x-slabs of 256/N layers
  (one slab Simulation needs ~107 GB at 128 x 256^2 elements, so N = 8 is
  the smallest feasible strong-scaling point; smaller N stop with a clear
  message instead of running out of memory);

x-slab decomposed with NCCL halo exchange and wave-speed all-reduce.

A "step" is one ADER-DG time step (dt reduction, predictor, face fluxes,
update) over the whole grid.  value = DOF-updates/s = E P^d K / t over all
ranks, t = max over ranks of the CUDA-event time of K steps.  u (1.31 GB per
GPU) is far larger than the 126 MB L2, so no flush is needed.

--impl reference times the reference algorithm's CPU implementation (the
numpy oracle port under oracle/, BLAS threads = all host cores) on a bounded
12^3 sample of the same workload; the reference package itself cannot be
shipped to the GPU box.
"""

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DOF updates/s (1/TDU) for 3D Euler ADER-DG N=4"
UNIT = "DOF/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cells", type=int, default=None,
                    help="elements per axis per GPU (weak; default 64 at N=1 (C2), 128 at N>1 "
                         "(C5)) or of the global cube (strong; default 256)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / domain check on CPU (gloo), no GPU work")
    ap.add_argument("--degree", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._loop, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.samples)}


def load_peaks():
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks.update(json.load(f))
    except Exception:
        peaks["hbm_gbs"] = 6650.0   # B200_PROFILING.md fallback
        peaks["hbm_source"] = "fallback"
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as f:
            peaks["fp64_dfma_tflops"] = json.load(f)["fp64_dfma_tflops"]
            peaks["fp64_source"] = "measured (tools/fp64_peak.cu, profiles/r01_fp64_peak.json)"
    except Exception:
        peaks["fp64_dfma_tflops"] = 37.0
        peaks["fp64_source"] = "spec fallback"
    return peaks


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "predictor_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


# ----------------------------------------------------------------------------
def cpu_oracle_dofs(cells, degree, steps, warmup=0):
    """Time the oracle port's Simulation.run (bench-tdu scope, cli.py:79-91)."""
    import numpy as np

    from oracle import problems as oprob
    from oracle.euler import EulerOracle
    from oracle.sim import OracleMesh, OracleSimulation

    d = 3
    cfl = 0.9 / (d * (2 * degree + 1))
    sim = OracleSimulation(OracleMesh([(0.0, 1.0)] * d, (cells,) * d), EulerOracle(d), degree,
                           cfl)
    sim.project_initial_condition(oprob.density_wave()[0])
    if warmup:
        sim.run(np.inf, max_steps=warmup)
    t0 = time.perf_counter()
    sim.run(np.inf, max_steps=sim.step_count + steps)
    wall = time.perf_counter() - t0
    dof = cells ** d * (degree + 1) ** d * steps
    return dof / wall, wall


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample(cells, degree, steps, threads, warmup=0):
    """oracle port timing in a fresh process with `threads` BLAS threads
    (OpenBLAS reads its thread count once, at load)."""
    env = dict(os.environ)
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        env[var] = str(threads)
    code = (f"import sys, json; sys.path.insert(0, {ROOT!r}); import bench; "
            f"v, w = bench.cpu_oracle_dofs({cells}, {degree}, {steps}, {warmup}); "
            f"print(json.dumps([v, w]))")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         check=True).stdout.strip().splitlines()[-1]
    v, w = json.loads(out)
    return v, w


def reference_arm(args, rank):
    if rank != 0:
        return
    n = os.cpu_count() or 1
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(var, str(n))
    cells = 12
    val, wall = cpu_oracle_dofs(cells, args.degree, args.steps, args.warmup)
    out = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (closed-form density-wave IC)",
        "config": {"workload": f"C2 sample: 3-D Euler density wave, {cells}^3 elements, "
                               f"N={args.degree}, periodic, cfl=1/30 (bounded CPU sample "
                               "of the 64^3 C2 grid; TDU is size independent)",
                   "degree": args.degree, "cells": [cells] * 3},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": n, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{cells}^3 elements x {args.steps} steps of oracle/ "
                                   "(numpy restatement of the reference, BLAS threads = "
                                   f"{n})"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------
class LaunchCounter:
    """Counts kernels launched through the C-ABI (calls -> kernels)."""

    KERNELS = {"adg_wavespeed": 2, "adg_timestep": 1, "adg_advance_time": 1,
               "adg_predict": 1, "adg_predict_range": 1, "adg_face_flux": 1, "adg_update": 2,
               "adg_totals_finalize": 1, "adg_totals": 3}

    def __init__(self, handle):
        self.h = handle
        self.count = 0
        self._orig = handle.call

        def call(name, *a):
            self.count += self.KERNELS.get(name, 1)
            return self._orig(name, *a)

        handle.call = call


def ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1808_03788_b200 as pkg
    from paper_1808_03788_b200 import roofline
    from paper_1808_03788_b200.decomp import SlabSimulation

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    N = args.degree
    d = 3
    P = N + 1
    cfl = 0.9 / (d * (2 * N + 1))
    strong = args.scaling == "strong"
    ext, gcells, slab_cells, workload = plan(args, world)
    gmesh = pkg.CartesianMesh(ext, gcells)
    # one slab Simulation: u, u_next, vol, 2d trace planes, face terms
    e_slab = slab_cells[0] * slab_cells[1] * slab_cells[2]
    need = e_slab * P ** d * (d + 2) * 8 * (3 + 2 * d) + e_slab * 2 * d * P ** (d - 1) * (d + 2) * 8
    free_b, _ = torch.cuda.mem_get_info(dev)
    if need > 0.97 * free_b:
        raise SystemExit(f"{slab_cells} elements per GPU need {need / 1e9:.0f} GB "
                         f"({free_b / 1e9:.0f} GB free): use more GPUs")
    system = pkg.make_system("euler", d)
    ic, _ = pkg.build_problem("density_wave", system)

    def make():
        s = SlabSimulation(gmesh, system, N, cfl, device=local_rank)
        s.project_initial_condition(ic)
        return s

    sim = make()
    E = sim.mesh.n_elements
    dofs_per_step_rank = E * P ** d

    # predictor launch timing on the launching stream (roofline)
    pred_events = []
    sweeps_total = []
    # (N > 1: the boundary-layer + interior predictor launches of a step with
    # the halo swap overlapped between them, SlabSimulation._predict_exchange)
    orig_predict = sim._predict_exchange

    def timed_predict(dt_dev):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        orig_predict(dt_dev)
        b.record()
        pred_events.append((a, b))
        sweeps_total.append(sim._buf.sweeps.sum(dtype=torch.int64))

    sim._predict_exchange = timed_predict
    # the step is GPU-bound at this size (launch overhead ~0.3 %), so the
    # 2-step CUDA graph replay of Simulation._run_batch is switched off to keep
    # the per-launch CUDA events and the launch count observable
    sim.graphs_enabled = False
    counter = LaunchCounter(sim._h)

    sim.run(np.inf, max_steps=args.warmup)
    pred_events.clear()
    sweeps_total.clear()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    counter.count = 0
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        start.record()
        sim.run(np.inf, max_steps=sim.step_count + args.steps)
        end.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = counter.count
    ms = start.elapsed_time(end)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = dofs_per_step_rank * world * args.steps / (ms_max * 1e-3)

    pred_ms = [a.elapsed_time(b) for a, b in pred_events]
    sw_tot = [int(x.item()) for x in sweeps_total]
    avg_pred_ms = sum(pred_ms) / len(pred_ms)
    avg_sweeps = sum(sw_tot) / len(sw_tot) / E
    flops = sum(roofline.predictor_flops(N, d, s, E) for s in sw_tot) / len(sw_tot)
    peaks = load_peaks()
    achieved = flops / (avg_pred_ms * 1e-3) / 1e12
    traffic = load_traffic()
    S_exec = max(sim.sweep_log[-args.steps:])
    step_roof = roofline.roofline_dofs(N, d, avg_sweeps, peaks["fp64_dfma_tflops"] * 1e12,
                                       peaks["hbm_gbs"] * 1e9) * world

    e2e = None
    local = sim.mesh
    tables = sim.tables
    del sim, counter, pred_events, sweeps_total, orig_predict
    torch.cuda.empty_cache()
    if not args.no_e2e:
        # end to end through the public API: pinned host IC -> device -> K steps ->
        # final state back to pinned host memory (the timed Simulation is freed
        # first and the IC is collocated on the host: one slab Simulation per GPU)
        host_u0 = torch.from_numpy(np.ascontiguousarray(
            ic(local.node_coords(tables)), dtype=np.float64)).pin_memory()
        host_out = torch.empty_like(host_u0).pin_memory()
        sim2 = SlabSimulation(gmesh, system, N, cfl, device=local_rank)
        sim2.set_state(host_u0)   # allocate workspaces outside the timed region
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s2 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        s2.record()
        sim2.set_state(host_u0)
        sim2.t = 0.0
        sim2.step_count = 0
        sim2.run(np.inf, max_steps=args.steps)
        host_out.copy_(sim2.u, non_blocking=True)
        e2.record()
        torch.cuda.synchronize()
        t2 = torch.tensor([s2.elapsed_time(e2)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        ub = host_u0.numel() * 8
        e2e = {"value": dofs_per_step_rank * world * args.steps / (float(t2.item()) * 1e-3),
               "unit": UNIT,
               "h2d_bytes_per_step": ub / args.steps,
               "d2h_bytes_per_step": (ub + args.steps * (4 + (d + 2)) * 8) / args.steps,
               "scope": "Simulation.set_state(pinned host u0) + run(max_steps=K) + final "
                        "state copied back to pinned host memory"}
        del sim2

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ncores = os.cpu_count() or 1
        # the reference arm's per-step sample (12^3 elements of the C2
        # workload), 2 steps with every host thread and 2 with one
        val, wall = cpu_sample(12, N, 2, ncores)
        val1, wall1 = cpu_sample(12, N, 2, 1)
        cpu = {"value": val, "unit": UNIT, "cores": ncores, "kind": "port",
               "value_1thread": val1, "cpu_model": cpu_model(),
               "sample": f"12^3 elements x 2 steps of the C2 workload (the reference arm's "
                         f"sample) through oracle/ (numpy restatement of the reference): "
                         f"{wall:.1f} s with {ncores} BLAS threads, {wall1:.1f} s with 1"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (closed-form density-wave IC, BASELINE C2/C5)",
            "config": {
                "workload": workload,
                "cells_per_gpu": list(slab_cells), "degree": N, "cfl": cfl,
                "l2": "inputs larger than L2 (u = %.2f GB per GPU)" % (
                    dofs_per_step_rank * (d + 2) * 8 / 1e9),
                "parallelism": "single GPU" if world == 1 else (
                    f"slab-x dp{world} ({dist.get_backend()} halos"
                    + (", all ranks on cuda:0: NOT a bench value)"
                       if os.environ.get("ADG_BENCH_ONE_DEVICE") == "1" else ")")),
                "picard_sweeps_max": S_exec, "picard_sweeps_mean": avg_sweeps},
            "roofline": {"kernel": "adg_predict (predict_kernel<3,5>)" if world == 1 else
                         "adg_predict_range x3 (predict_kernel<3,5>: boundary layers, "
                         "interior; halo swap overlapped)", "bound": "fp64",
                         "achieved": achieved, "peak": peaks["fp64_dfma_tflops"],
                         "unit": "TFLOP/s", "frac": achieved / peaks["fp64_dfma_tflops"],
                         # the ncu capture is of the C2 grid on one GPU
                         "traffic": (traffic.get("bytes_per_launch")
                                     if traffic and world == 1 and slab_cells == (64, 64, 64)
                                     and N == 4 else None),
                         "peak_source": peaks["fp64_source"],
                         "algorithmic_flops_per_launch": flops,
                         "avg_launch_ms": avg_pred_ms,
                         "share_of_step": avg_pred_ms / (ms_max / args.steps)},
            "step_roofline": {"dofs_per_s": step_roof, "frac": value / step_roof,
                              "model": "min(FP64 peak / flop_per_DOF, HBM / 560 B per DOF), "
                                       "SURVEY.md 8(d)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        print(json.dumps(out), flush=True)


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and relay rank 0's JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def plan(args, world):
    """Domain of this run: (global extents, global cells, cells per rank,
    workload text).  Weak: 128^3 per rank on [0, N] x [0, 1]^2 (C2's 64^3 at
    N = 1); strong: the fixed cube split into x-slabs."""
    if args.scaling == "strong":
        n = args.cells or 256
        if n % world:
            raise SystemExit(f"--scaling strong: {n} x-layers do not split over {world} ranks")
        return ([(0.0, 1.0)] * 3, (n, n, n), (n // world, n, n),
                f"C5 strong: {n}^3 unit cube, N={args.degree}, x-slabs of {n // world} layers "
                f"over {world} GPUs")
    n = args.cells or (64 if world == 1 else 128)
    work = ("C2: 3-D Euler smooth density wave, 64^3 elements, N=4, periodic unit cube, "
            "cfl=1/30" if world == 1 and n == 64 and args.degree == 4 else
            f"C5 weak: {n}^3 elements per GPU on [0,{world}]x[0,1]^2, N={args.degree}, "
            f"x-slab decomposition over {world} GPUs")
    return ([(0.0, float(world)), (0.0, 1.0), (0.0, 1.0)], (n * world, n, n), (n, n, n), work)


def dry_run(args, rank, world):
    """Launcher check without a GPU (CPU tests): every rank joins a gloo group,
    agrees on the plan, and rank 0 prints it as one JSON line."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    ext, cells, slab, work = plan(args, world)
    t = torch.tensor([float(slab[0])])
    if world > 1:
        dist.all_reduce(t)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": args.scaling,
                          "layers_total": float(t.item()),
                          "config": {"workload": work, "global_cells": list(cells),
                                     "cells_per_gpu": list(slab), "extents": ext}}),
              flush=True)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:
        dry_run(args, rank, world)
        return
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    # development check of the N > 1 code path on a one-GPU box:
    # ADG_BENCH_ONE_DEVICE=1 puts every rank on cuda:0 over gloo (host-staged
    # halos; ranks never wait on each other's kernels).  Its numbers are not
    # bench values; the driver's runs use NCCL with one GPU per rank.
    if os.environ.get("ADG_BENCH_ONE_DEVICE") == "1":
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if os.environ.get("ADG_BENCH_ONE_DEVICE") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
