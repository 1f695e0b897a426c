"""Single-grid time marching on a B200 (drop-in for reference driver.py).

`Simulation` keeps the reference constructor, attributes and methods
(driver.py:72-377); the state `u` is a CUDA fp64 torch tensor in the
reference layout (cells..., P..., m).  One accepted step is the kernel
sequence

    adg_timestep   dt = cfl / sum_j lambda_j / dx_j   (lambda from the previous
                   update's epilogue, or adg_wavespeed for a fresh state)
    adg_predict    startup + Picard + traces + volume integral, per element
    adg_face_flux  Rusanov face terms, one launch per axis
    adg_update     face integrals + element update + next-step wave speeds
                   + conserved-total partials
    [limiter]      adg_project_subcells / adg_detect / adg_rescue (C4)

all stream ordered with dt and t resident on the device, so
`run(max_steps=K)` without a limiter or callback issues K steps with no
host synchronisation; status words (no admissible state, non-finite
state) are checked once at the end and raised as the reference's
RuntimeErrors.
"""

import math
import os

import numpy as np
import torch

from . import _lib
from .basis import basis_tables, weight_tensor

BOUNDARY_KINDS = ("periodic", "outflow", "wall", "exact")

DMP_DELTA0 = 1e-3   # limiter.py:22
DMP_EPS = 1e-3      # limiter.py:23
GRAPH_MAX_DOFS = 1 << 21   # batched steps replay a CUDA graph below this size
MAX_HALVINGS = 3    # limiter.py:24

DEFAULT_CFL = {0: 0.9, 1: 0.30, 2: 0.15, 3: 0.09, 4: 0.062, 5: 0.044,
               6: 0.033, 7: 0.026, 8: 0.021, 9: 0.018}   # driver.py:27-28


def default_cfl(degree):
    return DEFAULT_CFL.get(degree, 0.4 / (2 * degree + 1))


def max_cfl_number(degree):
    return 1.0 / (2 * degree + 1)


def normalize_boundary(spec, dim):
    """{(axis, side): kind} from a kind, a per-axis mapping or a per-face dict
    (driver.py:36-69, same accepted forms and errors)."""
    table = {}
    if isinstance(spec, str):
        table = {(j, s): spec for j in range(dim) for s in (0, 1)}
    elif isinstance(spec, dict) and spec and all(isinstance(k, tuple) for k in spec):
        table = dict(spec)
    elif isinstance(spec, dict):
        for j in range(dim):
            kind = spec.get(j, "periodic")
            pair = (kind, kind) if isinstance(kind, str) else tuple(kind)
            table[(j, 0)], table[(j, 1)] = pair
    else:
        raise ValueError(f"unsupported boundary spec: {spec!r}")
    for j in range(dim):
        for s in (0, 1):
            kind = table.get((j, s))
            if kind not in BOUNDARY_KINDS:
                raise ValueError(f"unknown boundary kind {kind!r} on axis {j} side {s}")
        lo, hi = table[(j, 0)], table[(j, 1)]
        if "periodic" in (lo, hi) and lo != hi:
            raise ValueError(f"axis {j}: periodic must be set on both sides")
    return table


def _ptr(t):
    return None if t is None else t.data_ptr()


class StepBuffers:
    """Device workspaces of one grid (all torch CUDA tensors)."""

    def __init__(self, grid, n_elem, pd, m, dim, device, cells, limiter=False):
        f64 = dict(dtype=torch.float64, device=device)
        self.vol = torch.empty(n_elem * pd * m, **f64)
        # trace element blocks padded to a 16-byte multiple (adg_trace_block)
        self.tb = int(_lib.load().adg_trace_block(_lib.ctypes.byref(grid)))
        self.traces = torch.empty(2 * dim * n_elem * self.tb, **f64)
        # element-major face terms [E][dim][2 sides][P^(d-1)][m] (adg_face_flux)
        p = round(pd ** (1.0 / dim))
        self.fd = torch.empty(n_elem * 2 * dim * (pd // p) * m, **f64)
        self.pred_bad = torch.empty(n_elem, dtype=torch.uint8, device=device)
        self.sweeps = torch.empty(n_elem, dtype=torch.int32, device=device)
        self.red = torch.zeros(2, _lib.REDUCE_WORDS, dtype=torch.int64, device=device)
        self.nblocks = int(_lib.load().adg_update_blocks(_lib.ctypes.byref(grid)))
        self.partial = torch.empty(self.nblocks * m, **f64)
        self.t = torch.zeros(1, **f64)


class Simulation:
    """Owns the device state and marches it in time (driver.py:72-123).

    Extra keyword (not in the reference): `device` (CUDA device index or
    torch.device; default the current device), `min_picard_iter` (an element
    keeps sweeping until at least this many sweeps, default 1).
    """

    def __init__(self, mesh, system, degree, cfl, boundary="periodic",
                 use_limiter=False, predictor_mode="conservative",
                 exact_solution=None, dmp_delta0=DMP_DELTA0,
                 dmp_eps=DMP_EPS, batch_width=None, picard_tol=1e-12,
                 device=None, min_picard_iter=1, _ghost=None):
        if mesh.dim != system.dim:
            raise ValueError("mesh and system dimensions differ")
        if not 0.0 < cfl < max_cfl_number(degree):
            raise ValueError(
                f"cfl must lie in (0, {max_cfl_number(degree)}) "
                f"for degree {degree}, got {cfl}")
        name = getattr(system, "name", None)
        if name not in ("euler", "advection", "elasticity-di"):
            raise NotImplementedError(
                f"system '{getattr(system, 'name', system)}' has no B200 kernels "
                "(euler, advection, elasticity-di)")
        if predictor_mode not in ("conservative", "primitive"):
            raise ValueError(f"unknown predictor mode {predictor_mode!r}")
        if name in ("advection", "elasticity-di"):
            # both plugins have identity primitives (systems.py:60-64) and a
            # primitive_rhs equal to the conservative rate: predictor_mode
            # "primitive" iterates the same variables with the same rate
            self._iterate_mode = "conservative"
            if name == "elasticity-di":
                # the NCP plugin: unlimited step, periodic / outflow / wall faces
                if use_limiter:
                    raise NotImplementedError("elasticity-di on the device: no subcell limiter")
                kinds = normalize_boundary(boundary, mesh.dim).values()
                if "exact" in kinds:
                    raise NotImplementedError("elasticity-di on the device: no exact faces")
                if degree > 5:
                    raise NotImplementedError("elasticity-di on the device: degree <= 5")
        else:
            self._iterate_mode = predictor_mode
        self.mesh = mesh
        self.system = system
        self.tables = basis_tables(degree)
        self.cfl = float(cfl)
        self.boundary = normalize_boundary(boundary, mesh.dim)
        self.use_limiter = bool(use_limiter)
        self.predictor_mode = predictor_mode
        self.exact_solution = exact_solution
        self.dmp_delta0 = float(dmp_delta0)
        self.dmp_eps = float(dmp_eps)
        self.batch_width = batch_width
        self.picard_tol = float(picard_tol)
        self.min_picard_iter = int(min_picard_iter)
        if exact_solution is None and any(k == "exact" for k in self.boundary.values()):
            raise ValueError("exact boundaries need an exact_solution")
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1808_03788_b200 needs a CUDA device (B200); "
                               "there is no CPU fallback")
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", torch.device(device).index
                                   if isinstance(device, torch.device) else int(device))
        # a private handle: the predictor workspace belongs to this Simulation
        self._h = _lib.Handle(self.device.index)
        self._h.ensure_tables(self.tables)
        self._ghost = _ghost or {}
        # "exact" faces: exterior traces / subcell slabs evaluated from
        # exact_solution on the host each step (driver.py:250-261, :317-340)
        # and handed to the kernels as ADG_BC_GHOST data
        self._exact_faces = [k for k, v in self.boundary.items()
                             if v == "exact" and k not in self._ghost]
        self._exact_trace = {}
        # an exact_solution marked `device_capable` (the package's closed-form
        # cases; any callable that evaluates torch tensors) forms the boundary
        # data ON THE DEVICE from the device-resident t and dt: no host
        # evaluation or upload per step, and the batched / limited device
        # loops stay available (driver.py:250-261, :317-340)
        self._exact_dev = bool(self._exact_faces) and bool(
            getattr(exact_solution, "device_capable", False))
        self._exact_cache = {}
        d = mesh.dim
        self._P = degree + 1
        self._m = system.n_vars
        self._pd = self._P ** d
        self._shape = tuple(mesh.cells) + (self._P,) * d + (self._m,)
        self._grid = self._make_grid(mesh.cells, mesh.spacings)
        self._buf = None
        self._u = None
        self._u_next = None
        self._red_cur = None      # index into buf.red holding lambda of u (or None)
        self.t = 0.0
        self.step_count = 0
        self.force_limit_all = False
        self.last_limited_fraction = 0.0
        self.last_troubled = None
        self.last_sweeps = None
        self.history = []
        self.sweep_log = []

    # -- plumbing ------------------------------------------------------
    def _make_grid(self, cells, spacings):
        g = _lib.Grid()
        d = self.mesh.dim
        g.dim = d
        g.degree = self.tables.degree
        g.nvars = self.system.n_vars
        g.mode = _lib.MODE_CODES[self._iterate_mode]
        g.flags = 0
        for j in range(3):
            g.cells[j] = int(cells[j]) if j < d else 1
            g.dx[j] = float(spacings[j]) if j < d else 1.0
        _lib.fill_system(g, self.system)
        for j in range(d):
            for s in (0, 1):
                kind = self.boundary[(j, s)]
                if (j, s) in self._ghost:
                    kind = "ghost"
                g.bc[j][s] = _lib.BC_CODES[kind]
        # the predictor leaves u^n + vol / mass for the update where the
        # library supports it (one array less through HBM per step;
        # ADG_NO_FOLD=1: the plain volume integral, for A/B runs)
        if (os.environ.get("ADG_NO_FOLD") != "1"
                and _lib.load().adg_fold_supported(_lib.ctypes.byref(g))):
            g.flags |= _lib.GRID_FOLD_STATE
        return g

    def _gp(self):
        return _lib.ctypes.byref(self._grid)

    def _ensure_buffers(self):
        if self._buf is None:
            self._buf = StepBuffers(self._grid, self.mesh.n_elements, self._pd, self._m,
                                    self.mesh.dim, self.device, self.mesh.cells,
                                    self.use_limiter)
            self._u_next = torch.empty(self._shape, dtype=torch.float64, device=self.device)
        return self._buf

    # -- setup ---------------------------------------------------------
    def project_initial_condition(self, fn):
        """Collocate fn at the quadrature nodes (driver.py:127-154) and upload.
        With the limiter on, cells with an inadmissible nodal or subcell state
        are flattened to their weighted mean on the device (adg_flatten_ic)."""
        coords = self.mesh.node_coords(self.tables)
        u = np.asarray(fn(coords), dtype=float)
        if u.shape != self._shape:
            raise ValueError(f"initial condition returned shape {u.shape}, "
                             f"expected {self._shape}")
        self.set_state(u)
        if self.use_limiter:
            nflat = torch.zeros(1, dtype=torch.int32, device=self.device)
            self._h.call("adg_flatten_ic", self._gp(), _ptr(self._u), _ptr(nflat),
                         self._h.stream())
            self.ic_flattened = int(nflat.item())
            self._red_cur = None
        return self._u

    def set_state(self, u):
        """driver.py:156-157; accepts numpy arrays or tensors of the state shape."""
        if not isinstance(u, torch.Tensor):
            u = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64))
        if tuple(u.shape) != self._shape:
            raise ValueError(f"state shape {tuple(u.shape)} != {self._shape}")
        self._ensure_buffers()
        if self._u is None:
            self._u = torch.empty(self._shape, dtype=torch.float64, device=self.device)
        # pinned host tensors are copied asynchronously on the current stream
        self._u.copy_(u, non_blocking=u.device.type == "cpu" and u.is_pinned())
        self._red_cur = None

    @property
    def u(self):
        return self._u

    @u.setter
    def u(self, value):
        self.set_state(value)

    # -- device step pieces -------------------------------------------
    def _wavespeed(self):
        buf = self._ensure_buffers()
        red = buf.red[0]
        self._h.call("adg_wavespeed", self._gp(), _ptr(self._u), _ptr(red), self._h.stream())
        self._red_cur = 0

    def _timestep_into(self, dt_dst, status_dst, t_end):
        buf = self._buf
        if self._red_cur is None:
            self._wavespeed()
        red = buf.red[self._red_cur]
        self._h.call("adg_timestep", self._gp(), _ptr(red), self.cfl, _ptr(buf.t),
                     float(t_end), _ptr(dt_dst), _ptr(status_dst), self._h.stream())

    def _predict(self, dt_dev, q_out=None):
        buf = self._buf
        self._h.call("adg_predict", self._gp(), _ptr(self._u), _ptr(dt_dev), self.picard_tol,
                     0, self.min_picard_iter, _ptr(q_out), _ptr(buf.vol), _ptr(buf.traces),
                     _ptr(buf.pred_bad), _ptr(buf.sweeps), self._h.stream())

    # -- exact faces ----------------------------------------------------
    def _trace_strides(self, axis):
        """(tangential strides..., time stride) of a face trace block in units
        of m (the predictor's owner-role order, adg_predict)."""
        P = self._P
        d = self.mesh.dim
        if d == 3:
            return {0: ((P * P, P), 1), 1: ((1, P * P), P), 2: ((P, 1), P * P)}[axis]
        if d == 2:
            return {0: ((P,), 1), 1: ((1,), P)}[axis]
        return ((), 1)

    def _fill_exact_traces(self, dt):
        """Exterior space-time traces of the exact faces for a step of dt
        (driver._ghost_trace, driver.py:250-261), in trace-block layout."""
        if not self._exact_faces:
            return
        if self._exact_dev:
            return self._fill_exact_traces_device(self.t, dt)
        buf = self._buf
        P, m, d = self._P, self._m, self.mesh.dim
        for (axis, side) in self._exact_faces:
            pts = self.mesh.face_node_coords(self.tables, axis, side)
            vals = np.stack([np.asarray(self.exact_solution(pts, self.t + tau * dt), dtype=float)
                             for tau in self.tables.nodes], axis=-2)
            nplanes = self.mesh.n_elements // self.mesh.cells[axis]
            vals = vals.reshape((nplanes,) + (P,) * (d - 1) + (P, m))
            tang, st = self._trace_strides(axis)
            pos = np.zeros((P,) * (d - 1) + (P,), dtype=np.int64)
            for k, stride in enumerate(tang):
                sh = [1] * d
                sh[k] = P
                pos = pos + stride * np.arange(P).reshape(sh)
            sh = [1] * d
            sh[d - 1] = P
            pos = pos + st * np.arange(P).reshape(sh)
            block = np.zeros((nplanes, buf.tb))
            cols = (pos[..., None] * m + np.arange(m)).reshape(-1)
            block[:, cols] = vals.reshape(nplanes, -1)
            dst = self._exact_trace.get((axis, side))
            if dst is None:
                dst = torch.empty(nplanes * buf.tb, dtype=torch.float64, device=self.device)
                self._exact_trace[(axis, side)] = dst
            dst.copy_(torch.from_numpy(block.reshape(-1)))

    def _trace_cols(self, axis):
        """Positions (in doubles) of a face's [tangential.., time, m] values
        inside its trace block (the predictor's owner-role order)."""
        P, m, d = self._P, self._m, self.mesh.dim
        tang, st = self._trace_strides(axis)
        pos = np.zeros((P,) * (d - 1) + (P,), dtype=np.int64)
        for k, stride in enumerate(tang):
            sh = [1] * d
            sh[k] = P
            pos = pos + stride * np.arange(P).reshape(sh)
        sh = [1] * d
        sh[d - 1] = P
        pos = pos + st * np.arange(P).reshape(sh)
        return (pos[..., None] * m + np.arange(m)).reshape(-1)

    def _fill_exact_traces_device(self, t, dt):
        """_fill_exact_traces with exact_solution evaluated on the device; t
        and dt are floats or one-element device tensors (the batched loops
        pass the device clock and the step adg_timestep just formed)."""
        buf = self._buf
        f64 = dict(dtype=torch.float64, device=self.device)
        for (axis, side) in self._exact_faces:
            c = self._exact_cache.get(("tr", axis, side))
            if c is None:
                pts = torch.as_tensor(np.ascontiguousarray(
                    self.mesh.face_node_coords(self.tables, axis, side)), **f64)
                nplanes = self.mesh.n_elements // self.mesh.cells[axis]
                cols = torch.as_tensor(self._trace_cols(axis), device=self.device)
                dst = torch.zeros(nplanes * buf.tb, **f64)
                c = (pts, nplanes, cols, dst)
                self._exact_cache[("tr", axis, side)] = c
                self._exact_trace[(axis, side)] = dst
            pts, nplanes, cols, dst = c
            vals = torch.stack([self.exact_solution(pts, t + float(tau) * dt)
                                for tau in self.tables.nodes], dim=-2)
            dst.view(nplanes, buf.tb).index_copy_(1, cols, vals.reshape(nplanes, -1))

    def _exact_subcell_ghosts_device(self, t):
        """_exact_subcell_ghosts evaluated on the device at t (float or
        one-element device tensor) into persistent slabs."""
        c = self._exact_cache.get("gh")
        if c is None:
            d = self.mesh.dim
            S = self.tables.n_subcells
            L = max(S, 2)
            gh = _lib.SubcellGhosts()
            gh.layers = L
            slabs = []
            for (axis, side) in self._exact_faces:
                coords = []
                for i in range(d):
                    if i < axis:
                        coords.append(self.mesh.subcell_axis_coords(i, S, L))
                    elif i == axis:
                        full = self.mesh.subcell_axis_coords(i, S, L)
                        coords.append(full[:L] if side == 0 else full[-L:])
                    else:
                        coords.append(self.mesh.subcell_axis_coords(i, S, 0))
                pts = torch.as_tensor(np.ascontiguousarray(
                    np.stack(np.meshgrid(*coords, indexing="ij"), axis=-1)),
                    dtype=torch.float64, device=self.device)
                dev = torch.empty(pts.shape[:-1] + (self._m,), dtype=torch.float64,
                                  device=self.device)
                gh.slab[axis][side] = dev.data_ptr()
                slabs.append((pts, dev))
            c = (gh, slabs)
            self._exact_cache["gh"] = c
        gh, slabs = c
        for pts, dev in slabs:
            dev.copy_(self.exact_solution(pts, t))
        return gh

    def _exact_subcell_ghosts(self):
        """adg_subcell_ghosts for the exact faces at t_n (driver._boundary_slab,
        driver.py:317-340): slab (j, s) spans the axes padded before j with
        their ghost layers, its own `layers` ghost layers, and the interior of
        the later axes."""
        if not self._exact_faces:
            return None
        if self._exact_dev:
            return self._exact_subcell_ghosts_device(self.t)
        d = self.mesh.dim
        S = self.tables.n_subcells
        L = max(S, 2)
        gh = _lib.SubcellGhosts()
        gh.layers = L
        keep = []
        for (axis, side) in self._exact_faces:
            coords = []
            for i in range(d):
                if i < axis:
                    coords.append(self.mesh.subcell_axis_coords(i, S, L))
                elif i == axis:
                    full = self.mesh.subcell_axis_coords(i, S, L)
                    coords.append(full[:L] if side == 0 else full[-L:])
                else:
                    coords.append(self.mesh.subcell_axis_coords(i, S, 0))
            pts = np.stack(np.meshgrid(*coords, indexing="ij"), axis=-1)
            vals = np.ascontiguousarray(np.asarray(self.exact_solution(pts, self.t), dtype=float))
            dev = torch.from_numpy(vals.reshape(-1)).to(self.device)
            keep.append(dev)
            gh.slab[axis][side] = dev.data_ptr()
        self._exact_slabs = keep   # keep the device copies alive
        return gh

    def _faces(self):
        buf = self._buf
        for a in range(self.mesh.dim):
            glo = self._ghost.get((a, 0), self._exact_trace.get((a, 0)))
            ghi = self._ghost.get((a, 1), self._exact_trace.get((a, 1)))
            self._h.call("adg_face_flux", self._gp(), a, _ptr(buf.traces), _ptr(glo),
                         _ptr(ghi), _ptr(buf.fd), self._h.stream())

    def _update(self, dt_dev, totals_dst):
        buf = self._buf
        nxt = 1 - (self._red_cur or 0)
        self._h.call("adg_update", self._gp(), _ptr(self._u), _ptr(buf.vol), _ptr(buf.fd),
                     _ptr(dt_dev), _ptr(self._u_next), _ptr(buf.red[nxt]), _ptr(buf.partial),
                     self._h.stream())
        if totals_dst is not None:
            self._h.call("adg_totals_finalize", self._gp(), _ptr(buf.partial), buf.nblocks,
                         _ptr(totals_dst), self._h.stream())
        return nxt

    def _enqueue_unlimited(self, dt_dev, totals_dst, t_dst):
        """One unlimited step on the stream; commits u <- u_next."""
        buf = self._buf
        self._predict_exchange(dt_dev)
        self._faces()
        nxt = self._update(dt_dev, totals_dst)
        self._h.call("adg_advance_time", _ptr(buf.t), _ptr(dt_dev), _ptr(t_dst), self._h.stream())
        self._u, self._u_next = self._u_next, self._u
        self._red_cur = nxt

    def _predict_exchange(self, dt_dev):
        """Predictor, then (slab decomposition) the neighbour-rank face-trace
        halos into the ghost buffers; decomp.SlabSimulation overlaps the two."""
        self._predict(dt_dev)
        if self._exchange is not None:
            self._exchange(self)

    def _predict_part(self, dt_dev, e_begin, e_count):
        """The predictor on elements [e_begin, e_begin + e_count) of the
        whole-grid buffers (adg_predict_range)."""
        buf = self._buf
        self._h.call("adg_predict_range", self._gp(), int(e_begin), int(e_count),
                     _ptr(self._u), _ptr(dt_dev), self.picard_tol, 0, self.min_picard_iter,
                     None, _ptr(buf.vol), _ptr(buf.traces), _ptr(buf.pred_bad),
                     _ptr(buf.sweeps), self._h.stream())

    _exchange = None   # hook for slab decomposition (decomp.SlabSimulation)
    _capturable = False   # the exchange is stream ordered (C-ABI NCCL transport)

    # -- stepping ------------------------------------------------------
    def max_timestep(self):
        """corrector.compute_timestep on the device (corrector.py:30-55)."""
        if self._u is None:
            raise RuntimeError("no initial state set")
        self._ensure_buffers()
        out = torch.empty(1, dtype=torch.float64, device=self.device)
        status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._timestep_into(out, status, math.inf)
        st = int(status.item())
        if st & _lib.STATUS_NO_ADMISSIBLE:
            raise RuntimeError("no admissible state found while sizing the time step")
        return float(out.item())

    def advance(self, dt):
        """One step of (at most) dt with stability restarts (driver.py:166-184)."""
        if self._u is None:
            raise RuntimeError("no initial state set")
        self._ensure_buffers()
        trial = float(dt)
        m = self._m
        row = torch.empty(2 + m, dtype=torch.float64, device=self.device)
        for _ in range(MAX_HALVINGS + 1):
            row[0] = trial
            ok, fraction, troubled = self._attempt(row, trial)
            if ok:
                self.t += trial
                self.step_count += 1
                self.last_limited_fraction = fraction
                self.last_troubled = troubled
                self._combine_rows(row[None])
                host = row.cpu().numpy()
                self._record(trial, host[2:2 + m])
                return trial
            trial *= 0.5
        raise RuntimeError(f"step at t={self.t:.6g} failed after "
                           f"{MAX_HALVINGS} step halvings")

    def _attempt(self, row, trial):
        buf = self._buf
        dt_dev = row[0:1]
        self._fill_exact_traces(trial)
        if not self.use_limiter:
            self._enqueue_unlimited(dt_dev, row[2:], row[1:2])
            self.sweep_log.append(int(buf.sweeps.max().item()))
            return True, 0.0, None
        return self._attempt_limited(row, trial)

    def _limiter_buffers(self):
        lb = getattr(self, "_lim", None)
        if lb is None:
            E = self.mesh.n_elements
            S = self.tables.n_subcells
            m = self._m
            f64 = dict(dtype=torch.float64, device=self.device)
            # t^n subcell averages / extrema and the next step's, swapped on
            # acceptance (adg_detect + adg_rescue write the next ones)
            lb = {"sub": torch.empty(E * S ** self.mesh.dim * m, **f64),
                  "cmin": torch.empty(E * m, **f64), "cmax": torch.empty(E * m, **f64),
                  "sub_n": torch.empty(E * S ** self.mesh.dim * m, **f64),
                  "cmin_n": torch.empty(E * m, **f64), "cmax_n": torch.empty(E * m, **f64),
                  "troubled": torch.empty(self.mesh.cells, dtype=torch.uint8,
                                          device=self.device),
                  "idx": torch.empty(E, dtype=torch.int32, device=self.device),
                  "count": torch.zeros(1, dtype=torch.int32, device=self.device),
                  "failed": torch.zeros(1, dtype=torch.int32, device=self.device),
                  "sub_of": None}
            self._lim = lb
        return lb

    def _attempt_limited(self, row, trial):
        """_attempt_step + _limit on the device (driver.py:204-230, :265-299).
        Returns (accepted, limited_fraction, troubled flags)."""
        buf = self._buf
        lb = self._limiter_buffers()
        sp = self._h.stream()
        dt_dev = row[0:1]
        if lb["sub_of"] is not self._u or self._red_cur is None:
            # t^n subcell averages and their per-cell extrema (once per step)
            self._h.call("adg_project_subcells", self._gp(), _ptr(self._u), _ptr(lb["sub"]),
                         _ptr(lb["cmin"]), _ptr(lb["cmax"]), sp)
            lb["sub_of"] = self._u
        self._predict(dt_dev)
        self.sweep_log.append(None)
        self._faces()
        nxt = self._update(dt_dev, None)
        gh = self._exact_subcell_ghosts()
        ghp = _lib.ctypes.byref(gh) if gh is not None else None
        self._h.call("adg_detect", self._gp(), _ptr(lb["sub"]), _ptr(lb["cmin"]),
                     _ptr(lb["cmax"]), _ptr(self._u_next), _ptr(buf.pred_bad), self.dmp_delta0,
                     self.dmp_eps, int(bool(self.force_limit_all)), ghp, _ptr(lb["troubled"]),
                     _ptr(lb["idx"]), _ptr(lb["count"]), _ptr(lb["sub_n"]), _ptr(lb["cmin_n"]),
                     _ptr(lb["cmax_n"]), sp)
        n_tr = int(lb["count"].item())
        self.sweep_log[-1] = int(buf.sweeps.max().item())
        if n_tr:
            lb["failed"].zero_()
            self._h.call("adg_rescue", self._gp(), _ptr(lb["sub"]), _ptr(lb["idx"]),
                         _ptr(lb["count"]), n_tr, _ptr(dt_dev), ghp, _ptr(self._u_next),
                         _ptr(lb["failed"]), _ptr(lb["sub_n"]), _ptr(lb["cmin_n"]),
                         _ptr(lb["cmax_n"]), sp)
            if int(lb["failed"].item()):
                return False, 0.0, None   # driver.py:292-293 -> restart with dt/2
            # rescued cells changed u_next: redo its wave speeds / totals
            self._h.call("adg_wavespeed", self._gp(), _ptr(self._u_next), _ptr(buf.red[nxt]), sp)
        self._h.call("adg_totals", self._gp(), _ptr(self._u_next), _ptr(buf.partial),
                     _ptr(row[2:]), sp)
        self._h.call("adg_advance_time", _ptr(buf.t), _ptr(dt_dev), _ptr(row[1:2]), sp)
        self._u, self._u_next = self._u_next, self._u
        self._red_cur = nxt
        # the candidate's projection (rescued cells re-projected) is u^(n+1)'s
        for k in ("sub", "cmin", "cmax"):
            lb[k], lb[k + "_n"] = lb[k + "_n"], lb[k]
        lb["sub_of"] = self._u
        troubled = lb["troubled"].clone().bool()
        return True, n_tr / self.mesh.n_elements, troubled

    def run(self, t_end, max_steps=None, on_step=None):
        """March until t_end or max_steps (driver.py:186-202)."""
        if self._u is None:
            raise RuntimeError("no initial state set")
        self._ensure_buffers()
        scale = abs(t_end) if np.isfinite(t_end) else 1.0
        tiny = 1e-12 * max(1.0, scale)
        if self._exact_dev and not self._exact_cache:
            # node coordinates / index tables of the exact faces go to the
            # device once, outside any graph capture
            self._fill_exact_traces_device(self.t, 0.0)
            if self.use_limiter:
                self._exact_subcell_ghosts_device(self.t)
        fast = (on_step is None and not self.use_limiter and not np.isfinite(t_end)
                and max_steps is not None and (not self._exact_faces or self._exact_dev))
        if fast:
            self._run_batch(max(0, max_steps - self.step_count))
            return self.step_count
        if (self.use_limiter and (not self._exact_faces or self._exact_dev)
                and self._exchange is None):
            return self._run_limited(t_end, tiny, max_steps, on_step)
        while self.t < t_end - tiny:
            if max_steps is not None and self.step_count >= max_steps:
                break
            dt = min(self.max_timestep(), t_end - self.t)
            self.advance(dt)
            if not self._state_finite():
                raise RuntimeError(f"non-finite state after step {self.step_count}")
            if on_step is not None:
                on_step(self)
        return self.step_count

    def _run_limited(self, t_end, tiny, max_steps, on_step):
        """The limited run loop (driver.py:186-202 with _attempt_step and
        _limit) kept on the device: dt = min(max_timestep, t_end - t) is formed
        by adg_timestep, the attempt (predictor, faces, update, detection,
        rescue) is enqueued without reading anything back, and ONE host
        synchronisation per step fetches the step record (dt, t, totals,
        troubled count, rescue failure, status, non-finite count, max sweeps)
        to decide acceptance or the dt/2 restart (driver.py:170-184)."""
        buf = self._buf
        m = self._m
        dev = self.device
        row = torch.empty(2 + m, dtype=torch.float64, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        sw = torch.empty(1, dtype=torch.int32, device=dev)
        rec = torch.empty(2 + m, dtype=torch.float64).pin_memory()
        irec = torch.empty(5, dtype=torch.int64).pin_memory()
        ints = torch.empty(5, dtype=torch.int64, device=dev)
        lb = self._limiter_buffers()
        E = self.mesh.n_elements
        while self.t < t_end - tiny:
            if max_steps is not None and self.step_count >= max_steps:
                break
            buf.t.fill_(self.t)
            status.zero_()
            self._timestep_into(row[0:1], status, t_end)
            trial = None
            for attempt in range(MAX_HALVINGS + 1):
                if trial is not None:
                    row[0] = trial
                    buf.t.fill_(self.t)
                nxt = self._attempt_limited_device(row)
                torch.amax(buf.sweeps, dim=0, keepdim=True, out=sw)
                red = buf.red[nxt]
                torch.stack([lb["count"][0].long(), lb["failed"][0].long(), status[0].long(),
                             red[4], sw[0].long()], out=ints)
                rec.copy_(row, non_blocking=True)
                irec.copy_(ints, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
                n_tr, failed, st, nonfinite, sweeps = (int(x) for x in irec.tolist())
                if st & _lib.STATUS_NO_ADMISSIBLE:
                    raise RuntimeError("no admissible state found while sizing the time step")
                dt = float(rec[0])
                if not failed:
                    break
                trial = 0.5 * dt   # driver.py:183 restart with half the step
            else:
                raise RuntimeError(f"step at t={self.t:.6g} failed after "
                                   f"{MAX_HALVINGS} step halvings")
            self._commit_limited(nxt)
            self.t += dt
            self.step_count += 1
            self.last_limited_fraction = n_tr / E
            self.last_troubled = lb["troubled"].clone().bool()
            self.sweep_log.append(sweeps)
            self._record(dt, rec[2:2 + m].numpy().copy())
            if nonfinite:
                raise RuntimeError(f"non-finite state after step {self.step_count}")
            if on_step is not None:
                on_step(self)
        return self.step_count

    def _attempt_limited_device(self, row):
        """Enqueue one limited attempt of size row[0] with no host reads;
        returns the wave-speed slot of the candidate.  Nothing is committed:
        _commit_limited swaps the buffers once the host accepts it."""
        buf = self._buf
        lb = self._limiter_buffers()
        sp = self._h.stream()
        dt_dev = row[0:1]
        if lb["sub_of"] is not self._u or self._red_cur is None:
            self._h.call("adg_project_subcells", self._gp(), _ptr(self._u), _ptr(lb["sub"]),
                         _ptr(lb["cmin"]), _ptr(lb["cmax"]), sp)
            lb["sub_of"] = self._u
        ghp = None
        if self._exact_dev:
            # exact faces from the device clock: traces for this trial step,
            # subcell slabs at t^n
            self._fill_exact_traces_device(buf.t, dt_dev)
            ghp = _lib.ctypes.byref(self._exact_subcell_ghosts_device(buf.t))
        self._predict(dt_dev)
        self._faces()
        nxt = self._update(dt_dev, None)
        self._h.call("adg_detect", self._gp(), _ptr(lb["sub"]), _ptr(lb["cmin"]),
                     _ptr(lb["cmax"]), _ptr(self._u_next), _ptr(buf.pred_bad), self.dmp_delta0,
                     self.dmp_eps, int(bool(self.force_limit_all)), ghp, _ptr(lb["troubled"]),
                     _ptr(lb["idx"]), _ptr(lb["count"]), _ptr(lb["sub_n"]), _ptr(lb["cmin_n"]),
                     _ptr(lb["cmax_n"]), sp)
        lb["failed"].zero_()
        # a fixed grid of rescue blocks strides over the device-side count
        cap = min(self.mesh.n_elements, self._rescue_blocks)
        self._h.call("adg_rescue", self._gp(), _ptr(lb["sub"]), _ptr(lb["idx"]),
                     _ptr(lb["count"]), cap, _ptr(dt_dev), ghp, _ptr(self._u_next),
                     _ptr(lb["failed"]), _ptr(lb["sub_n"]), _ptr(lb["cmin_n"]),
                     _ptr(lb["cmax_n"]), sp)
        # rescued cells changed u_next: its wave speeds / counts again (the
        # update epilogue folded the candidate's) and the conserved totals, in
        # one pass over the state
        self._h.call("adg_state_record", self._gp(), _ptr(self._u_next), _ptr(buf.red[nxt]),
                     _ptr(buf.partial), _ptr(row[2:]), sp)
        self._h.call("adg_advance_time", _ptr(buf.t), _ptr(dt_dev), _ptr(row[1:2]), sp)
        return nxt

    # rescue blocks per launch (each strides over the troubled list)
    _rescue_blocks = 148 * 8

    def _commit_limited(self, nxt):
        lb = self._lim
        self._u, self._u_next = self._u_next, self._u
        self._red_cur = nxt
        for k in ("sub", "cmin", "cmax"):
            lb[k], lb[k + "_n"] = lb[k + "_n"], lb[k]
        lb["sub_of"] = self._u

    def _combine_rows(self, rows):
        """Hook: cross-rank SUM of per-step totals (decomp.SlabSimulation)."""

    def _state_finite(self):
        red = self._buf.red[self._red_cur]
        return int(red[4].item()) == 0

    def _step_into(self, rows, status, sweeps, s):
        """Enqueue one unlimited step writing its history row / status /
        sweep count into slot s of the given device buffers."""
        self._timestep_into(rows[s, 0:1], status[s:s + 1], math.inf)
        if self._exact_dev:
            self._fill_exact_traces_device(self._buf.t, rows[s, 0:1])
        self._enqueue_unlimited(rows[s, 0:1], rows[s, 2:], rows[s, 1:2])
        torch.amax(self._buf.sweeps, dim=0, keepdim=True, out=sweeps[s:s + 1])

    # CUDA graph of an even number of consecutive steps (the u / u_next and
    # wave-speed double buffers return to their starting roles after two
    # steps), replayed with a device-side slot counter; removes the per-launch
    # host cost that bounds small grids (C1: ~8 launches per step).  Batches
    # shorter than graph_steps (or their tail) replay a two-step graph.
    # Default 2: a longer graph saves ~1 us per C1 step but its first capture
    # costs ~4 ms (profiles/r01k_graph_unroll.jsonl, r01l_configs.jsonl).
    graphs_enabled = True
    graph_steps = 2

    def _batch_buffers(self, k):
        bb = getattr(self, "_bb", None)
        if bb is None or bb["cap"] < k:
            cap = max(k, 64)
            dev = self.device
            bb = {"cap": cap,
                  "rows": torch.zeros(cap, 2 + self._m, dtype=torch.float64, device=dev),
                  "status": torch.zeros(cap, dtype=torch.int32, device=dev),
                  "sweeps": torch.zeros(cap, dtype=torch.int32, device=dev),
                  "cnt": torch.zeros(1, dtype=torch.int64, device=dev),
                  "srow": torch.zeros(2, 2 + self._m, dtype=torch.float64, device=dev),
                  "sst": torch.zeros(2, dtype=torch.int32, device=dev),
                  "ssw": torch.zeros(2, dtype=torch.int32, device=dev),
                  "graphs": {}}
            self._bb = bb
        return bb

    def _pair_graph(self, bb, nsteps=2):
        # everything a replay bakes in: buffer roles, step count and the
        # scalar arguments of the captured launches
        key = (self._u.data_ptr(), self._red_cur, nsteps, self.cfl, self.picard_tol,
               self.min_picard_iter)
        g = bb["graphs"].get(key)
        if g is not None:
            return g
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        ncols = bb["rows"].shape[1]
        with torch.cuda.graph(g):
            for j in range(nsteps):
                srow, sst = bb["srow"][j % 2], bb["sst"][j % 2:j % 2 + 1]
                self._timestep_into(srow[0:1], sst, math.inf)
                if self._exact_dev:
                    self._fill_exact_traces_device(self._buf.t, srow[0:1])
                self._enqueue_unlimited(srow[0:1], srow[2:], srow[1:2])
                # history row, status and max sweep count into slot cnt
                self._h.call("adg_log_step", _ptr(srow), ncols, _ptr(sst),
                             _ptr(self._buf.sweeps), self.mesh.n_elements, _ptr(bb["rows"]),
                             _ptr(bb["status"]), _ptr(bb["sweeps"]), _ptr(bb["cnt"]),
                             self._h.stream())
        # capture only recorded the launches: state is back where it started
        bb["graphs"][key] = g
        return g

    def _pair_graphs_both(self, bb, nsteps):
        """The graph of the current buffer roles and of the swapped ones: a
        batch that starts on the other parity then replays instead of
        capturing inside the caller's (timed) region."""
        g = self._pair_graph(bb, nsteps)
        if self._red_cur is not None:
            self._u, self._u_next = self._u_next, self._u
            self._red_cur = 1 - self._red_cur
            try:
                self._pair_graph(bb, nsteps)
            finally:
                self._u, self._u_next = self._u_next, self._u
                self._red_cur = 1 - self._red_cur
        return g

    def _run_batch(self, k):
        """k device-resident steps with one host synchronisation at the end."""
        if k <= 0:
            return
        buf = self._buf
        m = self._m
        bb = self._batch_buffers(k)
        rows, status, sweeps = bb["rows"][:k], bb["status"][:k], bb["sweeps"][:k]
        rows.zero_()
        status.zero_()
        bb["sst"].zero_()   # timestep_kernel ORs status bits into the step slots
        buf.t.fill_(self.t)
        # only launch-bound grids gain from the graph (capture + instantiate
        # costs tens of ms once; a C2-size step is ~16 ms of GPU work)
        use_graph = (self.graphs_enabled and (self._exchange is None or self._capturable)
                     and self.mesh.n_elements * self._pd <= GRAPH_MAX_DOFS)
        s = 0
        while s < k:
            if use_graph and self._red_cur is not None and k - s >= 2:
                bb["cnt"].fill_(s)
                for n in sorted({max(2, self.graph_steps - self.graph_steps % 2), 2},
                                reverse=True):
                    if k - s < n:
                        continue
                    g = self._pair_graphs_both(bb, n)
                    while k - s >= n:
                        g.replay()
                        s += n
                continue
            self._step_into(bb["rows"], bb["status"], bb["sweeps"], s)
            s += 1
        self._combine_rows(rows)
        host = rows.cpu().numpy()
        st = status.cpu().numpy()
        sw = sweeps.cpu().numpy()
        final_nonfinite = not self._state_finite()
        for s in range(k):
            if st[s] & _lib.STATUS_NO_ADMISSIBLE:
                raise RuntimeError("no admissible state found while sizing the time step")
            if s > 0 and st[s] & _lib.STATUS_NONFINITE:
                raise RuntimeError(f"non-finite state after step {self.step_count}")
            self.t = float(host[s, 1])
            self.step_count += 1
            self.last_limited_fraction = 0.0
            self.last_troubled = None
            self.sweep_log.append(int(sw[s]))
            self._record(float(host[s, 0]), host[s, 2:2 + m])
        if final_nonfinite:
            raise RuntimeError(f"non-finite state after step {self.step_count}")

    # -- reductions ----------------------------------------------------
    def conserved_totals(self):
        """Domain integrals per quantity (driver.py:344-350), device reduction."""
        buf = self._ensure_buffers()
        out = torch.empty(self._m, dtype=torch.float64, device=self.device)
        self._h.call("adg_totals", self._gp(), _ptr(self._u), _ptr(buf.partial), _ptr(out),
                     self._h.stream())
        return out.cpu().numpy()

    def error_norms(self, reference=None, t=None):
        """Quadrature L1/L2/Linf errors (driver.py:352-367), evaluated on device."""
        fn = reference if reference is not None else self.exact_solution
        if fn is None:
            raise ValueError("no reference solution available")
        when = self.t if t is None else t
        ref = torch.as_tensor(np.asarray(fn(self.mesh.node_coords(self.tables), when), float),
                              device=self.device)
        diff = self._u - ref
        w = torch.as_tensor(weight_tensor(self.tables.weights, self.mesh.dim),
                            device=self.device)[..., None]
        vol = self.mesh.cell_volume
        red = tuple(range(diff.ndim - 1))
        return {"l1": (vol * (diff.abs() * w).sum(dim=red)).cpu().numpy(),
                "l2": torch.sqrt(vol * (diff * diff * w).sum(dim=red)).cpu().numpy(),
                "linf": diff.abs().amax(dim=red).cpu().numpy()}

    def _record(self, dt, totals):
        self.history.append({"step": self.step_count, "time": self.t, "dt": dt,
                             "totals": np.array(totals, dtype=float),
                             "limited_fraction": self.last_limited_fraction})
