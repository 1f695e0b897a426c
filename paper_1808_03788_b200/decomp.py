"""Slab domain decomposition across GPUs.

One process per GPU (torch.distributed, NCCL).  The global Cartesian grid is
split along x into equal slabs; rank r owns cells [r*n0/W, (r+1)*n0/W) of
axis 0.  Per step the only exchanges are

  * face-trace halos: after the predictor, each rank sends the low-x trace
    plane of its first element layer to rank r-1 and the high-x plane of
    its last layer to rank r+1 (the reference's ghost/periodic face states,
    driver.py:234-248, across the slab cut); received planes become the
    ADG_BC_GHOST exterior traces of adg_face_flux;
  * the CFL reduction: a MAX all-reduce of the per-axis wave-speed bits and
    a SUM of the admissible / non-finite counts (corrector.py:47-55 taken
    over the global grid -- exactly the reference's dt, not a min of
    per-rank dts);
  * conserved totals: a SUM all-reduce of the per-step totals rows, once per
    batch of steps.

No collective touches the element data itself.  Two transports carry them:

  * "adg" (default under NCCL, one GPU per rank): the library's own NCCL
    communicator behind the C-ABI (`adg_comm_init`, `adg_halo_exchange`,
    `adg_allreduce_reduce`, `adg_allreduce_sum`; csrc/adg_comm.cu) --
    stream-ordered calls on the Simulation's stream, so the step stays
    CUDA-graph capturable;
  * "torch": torch.distributed P2P / all-reduce, which works on any backend;
    the CPU test suite covers the exchange logic with gloo at world_size 2.
"""

import ctypes

import torch
import torch.distributed as dist

from . import _lib
from .driver import Simulation
from .mesh import CartesianMesh


def slab_bounds(n0, world, rank):
    if n0 % world:
        raise ValueError(f"{n0} cells along x do not split evenly over {world} ranks")
    k = n0 // world
    return rank * k, (rank + 1) * k


def local_mesh(global_mesh, world, rank):
    lo, hi = slab_bounds(global_mesh.cells[0], world, rank)
    x0, x1 = global_mesh.extents[0]
    dx = (x1 - x0) / global_mesh.cells[0]
    ext = [(x0 + lo * dx, x0 + hi * dx)] + list(global_mesh.extents[1:])
    mesh = CartesianMesh(ext, (hi - lo,) + tuple(global_mesh.cells[1:]))
    # the slab's element widths are the global ones bit for bit (recomputing
    # them from the slab extents can differ by an ulp)
    mesh.spacings = tuple(global_mesh.spacings)
    return mesh


def exchange_planes_start(send_lo, send_hi, recv_lo, recv_hi, group=None):
    """Post the periodic ring halo swap along x; returns the pending works.

    send_lo -> rank-1 (it becomes that rank's high ghost), send_hi -> rank+1
    (its low ghost); recv_lo <- rank-1's send_hi, recv_hi <- rank+1's send_lo.
    All four are contiguous tensors on this rank's device.  On NCCL the
    transfers are ordered after the work already on the current stream and
    run on NCCL's stream, so kernels launched before the works are waited
    on overlap them.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    left = (rank - 1) % world
    right = (rank + 1) % world
    if world == 1:
        recv_lo.copy_(send_hi)
        recv_hi.copy_(send_lo)
        return []
    g = lambda r: dist.get_global_rank(group, r) if group is not None else r  # noqa: E731
    staged = send_lo.is_cuda and dist.get_backend(group) != "nccl"
    if staged:
        # host-transport backends (gloo) move host memory only: stage the
        # device planes through host copies (the multi-process CPU/GPU tests)
        send_lo, send_hi = send_lo.cpu(), send_hi.cpu()
        dev_lo, dev_hi = recv_lo, recv_hi
        recv_lo, recv_hi = torch.empty_like(send_lo), torch.empty_like(send_hi)
    ops = [dist.P2POp(dist.isend, send_lo, g(left), group),
           dist.P2POp(dist.irecv, recv_hi, g(right), group),
           dist.P2POp(dist.isend, send_hi, g(right), group),
           dist.P2POp(dist.irecv, recv_lo, g(left), group)]
    works = dist.batch_isend_irecv(ops)
    if staged:
        works.append(_HostToDevice(((recv_lo, dev_lo), (recv_hi, dev_hi))))
    return works


class _StreamJoin:
    """Pending halo swap on a side stream: wait() joins it into the main one."""

    def __init__(self, side, main):
        self.side = side
        self.main = main

    def wait(self):
        self.main.wait_stream(self.side)


class _HostToDevice:
    """Pending copy of host-staged receive planes into their device buffers."""

    def __init__(self, pairs):
        self.pairs = pairs

    def wait(self):
        for host, dev in self.pairs:
            dev.copy_(host)


def exchange_planes_wait(works):
    """Complete exchange_planes_start (NCCL: the current stream waits)."""
    for req in works:
        req.wait()


def exchange_planes(send_lo, send_hi, recv_lo, recv_hi, group=None):
    """Periodic ring halo swap along x (exchange_planes_start + wait)."""
    exchange_planes_wait(exchange_planes_start(send_lo, send_hi, recv_lo, recv_hi, group))


class Communicator:
    """An adg_comm (NCCL) on this rank's device, its unique id shared through
    the torch.distributed group (broadcast from rank 0)."""

    def __init__(self, handle, group=None, world=None, rank=None):
        lib = _lib.load()
        self.lib = lib
        self.handle = handle
        self.world = dist.get_world_size(group) if world is None else world
        self.rank = dist.get_rank(group) if rank is None else rank
        uid = torch.zeros(_lib.COMM_ID_BYTES, dtype=torch.uint8)
        if self.rank == 0:
            buf = ctypes.create_string_buffer(_lib.COMM_ID_BYTES)
            rc = lib.adg_comm_unique_id(buf)
            if rc != _lib.ADG_OK:
                raise RuntimeError(f"adg_comm_unique_id failed (rc={rc})")
            uid.copy_(torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8))
        if self.world > 1:
            if dist.get_backend(group) == "nccl":
                dev = uid.to(torch.device("cuda", handle.device_index))
                dist.broadcast(dev, dist.get_global_rank(group, 0) if group else 0, group=group)
                uid = dev.cpu()
            else:
                dist.broadcast(uid, dist.get_global_rank(group, 0) if group else 0, group=group)
        raw = bytes(uid.numpy().tobytes())
        ptr = ctypes.c_void_p()
        handle.call("adg_comm_init", ctypes.c_char_p(raw), int(self.world), int(self.rank),
                    ctypes.byref(ptr))
        self.ptr = ptr

    def halo_exchange(self, grid_ref, traces, ghost_lo, ghost_hi, stream):
        self.handle.call("adg_halo_exchange", self.ptr, grid_ref, traces.data_ptr(),
                         ghost_lo.data_ptr(), ghost_hi.data_ptr(), stream)

    def allreduce_record(self, red, stream):
        self.handle.call("adg_allreduce_reduce", self.ptr, red.data_ptr(), stream)

    def allreduce_sum(self, buf, stream):
        self.handle.call("adg_allreduce_sum", self.ptr, buf.data_ptr(), buf.numel(), stream)

    def __del__(self):
        ptr, self.ptr = getattr(self, "ptr", None), None
        if ptr is not None and ptr.value:
            try:
                self.lib.adg_comm_destroy(ptr)
            except Exception:
                pass


def combine_reduce(red, group=None):
    """adg_reduce record: MAX of lam bit patterns (non-negative doubles order
    like integers), SUM of the admissible / non-finite counts."""
    dist.all_reduce(red[0:3], op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(red[3:5], op=dist.ReduceOp.SUM, group=group)


class SlabSimulation(Simulation):
    """Simulation of one x-slab of `global_mesh` on this rank's GPU.

    Only periodic x boundaries are supported across the cut (the C5 setup);
    y / z keep the requested boundary kinds.
    """

    def __init__(self, global_mesh, system, degree, cfl, boundary="periodic", group=None,
                 transport=None, self_exchange=False, **kw):
        """transport: "adg" (the C-ABI NCCL communicator), "torch"
        (torch.distributed; default unless the backend is NCCL).
        self_exchange: a one-rank run that still cuts the x faces and swaps
        its own halo planes over a one-rank communicator (an on-device check
        of the exchange path against the periodic single-domain run)."""
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.global_mesh = global_mesh
        mesh = local_mesh(global_mesh, self.world, self.rank)
        ghost = {}
        cut = self.world > 1 or self_exchange
        if transport is None:
            transport = ("adg" if self_exchange or (self.world > 1 and
                                                    dist.get_backend(group) == "nccl")
                         else "torch")
        if transport not in ("adg", "torch"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport
        if cut:
            if kw.get("use_limiter"):
                # the limiter's windows and DMP bounds would need a u^n ghost
                # layer across the cut; not part of C5
                raise NotImplementedError("slab decomposition: no subcell limiter across ranks")
            if boundary != "periodic":
                raise NotImplementedError("slab decomposition needs periodic x faces")
            P = degree + 1
            plane = 1
            for c in mesh.cells[1:]:
                plane *= c
            blk = P ** mesh.dim * system.n_vars
            n = plane * (blk + (blk & 1))   # trace blocks are padded (adg_trace_block)
            dev = kw.get("device")
            dev = torch.device("cuda", torch.cuda.current_device() if dev is None else int(dev))
            ghost = {(0, 0): torch.empty(n, dtype=torch.float64, device=dev),
                     (0, 1): torch.empty(n, dtype=torch.float64, device=dev)}
        super().__init__(mesh, system, degree, cfl, boundary=boundary, _ghost=ghost, **kw)
        self._comm = None
        if cut:
            self._exchange = SlabSimulation._swap_halos
            if transport == "adg":
                self._comm = Communicator(self._h, group,
                                          world=1 if self_exchange else None,
                                          rank=0 if self_exchange else None)
                # stream-ordered NCCL calls: the batched step graph-captures
                self._capturable = True
        self._cut = cut
        # boundary-layer predictor + halo swap overlapped with the interior
        self.overlap_halos = True
        self._range_ok = (cut and bool(_lib.load().adg_predict_range_supported(self._gp())))

    def _swap_halos(self, wait=True):
        buf = self._buf
        if self._comm is not None:
            # C-ABI NCCL transport: on a side stream when overlapped (the
            # caller joins it before the faces), else on the step's stream
            if wait:
                self._comm.halo_exchange(self._gp(), buf.traces, self._ghost[(0, 0)],
                                         self._ghost[(0, 1)], self._h.stream())
                return []
            main = torch.cuda.current_stream(self.device)
            side = self._side_stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self._comm.halo_exchange(self._gp(), buf.traces, self._ghost[(0, 0)],
                                         self._ghost[(0, 1)], side.cuda_stream)
            return [_StreamJoin(side, main)]
        n = self._ghost[(0, 0)].numel()
        face = self.mesh.n_elements * buf.tb
        lo_plane = buf.traces[0:n]                       # axis 0, side 0, first layer
        hi_plane = buf.traces[2 * face - n:2 * face]     # axis 0, side 1, last layer
        works = exchange_planes_start(lo_plane, hi_plane, self._ghost[(0, 0)],
                                      self._ghost[(0, 1)], self.group)
        if wait:
            exchange_planes_wait(works)
            return []
        return works

    def close(self):
        """Release the captured graphs (they hold the communicator's calls),
        then the communicator."""
        torch.cuda.synchronize(self.device)
        bb = getattr(self, "_bb", None)
        if bb is not None:
            bb["graphs"].clear()
        self._comm = None

    def __del__(self):
        try:
            if getattr(self, "_comm", None) is not None:
                self.close()
        except Exception:
            pass

    def _side_stream(self):
        s = getattr(self, "_side", None)
        if s is None:
            s = self._side = torch.cuda.Stream(self.device)
        return s

    def _predict_exchange(self, dt_dev):
        """Boundary layers first, their halo exchange overlapped with the
        interior predictor: predict the first and last x-layers
        of the slab, post the trace-plane swap, predict the interior, then
        make the stream wait for the swap before the face kernels."""
        if not self._cut:
            return super()._predict_exchange(dt_dev)
        nx = self.mesh.cells[0]
        E = self.mesh.n_elements
        layer = E // nx
        if not (self.overlap_halos and nx >= 3 and self._range_ok):
            self._predict(dt_dev)
            self._swap_halos()
            return
        self._predict_part(dt_dev, 0, layer)
        self._predict_part(dt_dev, E - layer, layer)
        works = self._swap_halos(wait=False)
        self._predict_part(dt_dev, layer, E - 2 * layer)
        exchange_planes_wait(works)

    def _timestep_into(self, dt_dst, status_dst, t_end):
        if self._red_cur is None:
            self._wavespeed()
        if self._comm is not None:
            self._comm.allreduce_record(self._buf.red[self._red_cur], self._h.stream())
        elif self.world > 1:
            combine_reduce(self._buf.red[self._red_cur], self.group)
        super()._timestep_into(dt_dst, status_dst, t_end)

    def _sum_ranks(self, t):
        if self._comm is not None:
            self._comm.allreduce_sum(t, self._h.stream())
        elif self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def _combine_rows(self, rows):
        if self.world > 1 or self._comm is not None:
            tot = rows[:, 2:].contiguous()   # collectives need dense tensors
            self._sum_ranks(tot)
            rows[:, 2:] = tot

    def _state_finite(self):
        if self.world > 1:
            red = self._buf.red[self._red_cur].clone()
            if self._comm is not None:
                self._comm.allreduce_record(red, self._h.stream())
            else:
                dist.all_reduce(red[4:5], op=dist.ReduceOp.SUM, group=self.group)
            return int(red[4].item()) == 0
        return super()._state_finite()

    def conserved_totals(self):
        tot = torch.as_tensor(super().conserved_totals(), device=self.device)
        if self.world > 1:
            self._sum_ranks(tot)
        return tot.cpu().numpy()
