"""Module-level predictor entry points on device tensors (reference
predictor.py: :57-62 PredictorResult, :99-126 startup_guess, :135-191
picard_solve, :194-215 weak_form_defect, :218-230 extract_traces).

Arrays are CUDA fp64 tensors in the reference layout with the grid axes in
front (numpy inputs are uploaded); every call is one or two launches of the
fused predictor (`adg_predict` / `adg_predict_ex`) or of the module kernels
(`adg_extract_traces`, `adg_spacetime_rate`).  The reference's leading
"batch axes" are the element grid here: u is (cells.., P.., m).
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .basis import basis_tables


@dataclass
class PredictorResult:
    q: torch.Tensor            # (cells.., P.., P_t, m) space-time states (conservative)
    iterations: int            # Picard sweeps (reference semantics, see picard_solve)
    converged: torch.Tensor    # (cells..,) bool
    admissible: torch.Tensor   # (cells..,) bool
    sweeps: torch.Tensor = None    # (cells..,) int32 sweeps each element took
    traces: dict = None            # {(j, side): (cells.., P^(d-1).., P_t, m)}
    volume: torch.Tensor = None    # corrector.volume_integral of q


def _grid(system, n_elem, spacings, degree, boundary_codes=None, mode="conservative"):
    """adg_grid of n_elem independent elements (the element-local calls: the
    reference's leading batch axes, flattened)."""
    g = _lib.Grid()
    d = system.dim
    g.dim, g.degree, g.nvars = d, degree, system.n_vars
    g.mode = _lib.MODE_CODES[mode]
    for j in range(3):
        g.cells[j] = max(int(n_elem), 1) if j == 0 else 1
        g.dx[j] = float(spacings[j]) if j < d else 1.0
    _lib.fill_system(g, system)
    for j in range(d):
        for s in (0, 1):
            g.bc[j][s] = 0 if boundary_codes is None else boundary_codes[j][s]
    return g


def _device_array(a, device=None):
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1808_03788_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, dtype=np.float64))
    if not t.is_cuda:
        t = t.to(device if device is not None else torch.cuda.current_device())
    return t.to(dtype=torch.float64).contiguous()


def _check_mode(mode):
    if mode not in _lib.MODE_CODES:
        raise ValueError(f"unknown predictor mode {mode!r}")


# the kernel writes each face's trace block in its owner role's order
# (x: [j][k][t], y: [k][t][i], z: [t][i][j]; 2-D y: [t][i]); these
# permutations present them in the reference layout
_TRACE_PERMS = {3: {0: (0, 1, 2), 1: (2, 0, 1), 2: (1, 2, 0)}, 2: {0: (0, 1), 1: (1, 0)},
                1: {0: (0,)}}


def run_predictor(u, system, spacings, dt, tables, tol=1e-12, max_iter=None, min_iter=1,
                  want_q=True, mode="conservative", initial=None, startup_only=False):
    """One fused predictor launch on u (cells.., P.., m).  Returns
    (PredictorResult, ok) with q, per-element sweeps and flags, traces and
    the volume accumulator of corrector.volume_integral (corrector.py:141-177);
    ok = converged & admissible.  `iterations` is the largest per-element
    sweep count of this launch."""
    _check_mode(mode)
    if getattr(system, "identity_primitives", False) and getattr(system, "name", "") != "euler":
        # cons_to_prim is the identity (advection): the primitive iteration
        # is the conservative one (the rate -a.grad q either way)
        mode = "conservative"
    d = system.dim
    m = system.n_vars
    P = tables.degree + 1
    u = _device_array(u)
    if u.ndim < d + 1 or tuple(u.shape[u.ndim - 1 - d:]) != (P,) * d + (m,):
        raise ValueError(f"u has shape {tuple(u.shape)}; expected (...,{P}^{d},{m})")
    cells = tuple(u.shape[:u.ndim - 1 - d])   # the reference's batch axes
    E = int(np.prod(cells)) if cells else 1
    h = _lib.Handle.get(u.device.index)
    h.ensure_tables(tables)
    g = _grid(system, E, spacings, tables.degree, mode=mode)
    pd = P ** d
    dev = u.device
    f64 = dict(dtype=torch.float64, device=dev)
    q = torch.empty(cells + (P,) * d + (P, m), **f64) if (want_q or startup_only) else None
    vol = torch.empty(u.shape, **f64)
    tb = pd * m + ((pd * m) & 1)   # padded trace element block (adg_trace_block)
    traces = torch.empty(2 * d, E, tb, **f64)
    bad = torch.empty(cells, dtype=torch.uint8, device=dev)
    sweeps = torch.empty(cells, dtype=torch.int32, device=dev)
    dt_dev = torch.full((1,), float(dt), **f64)
    mi = 0 if max_iter is None else int(max_iter)
    if initial is None and not startup_only:
        h.call("adg_predict", _lib.ctypes.byref(g), u.data_ptr(), dt_dev.data_ptr(), float(tol),
               mi, int(min_iter), q.data_ptr() if q is not None else None, vol.data_ptr(),
               traces.data_ptr(), bad.data_ptr(), sweeps.data_ptr(), h.stream())
    else:
        q0 = None
        if initial is not None:
            q0 = _device_array(initial, dev)
            if tuple(q0.shape) != cells + (P,) * d + (P, m):
                raise ValueError(f"initial has shape {tuple(q0.shape)}; expected "
                                 f"{cells + (P,) * d + (P, m)}")
        flags = _lib.PRED_STARTUP_ONLY if startup_only else 0
        h.call("adg_predict_ex", _lib.ctypes.byref(g), u.data_ptr(),
               q0.data_ptr() if q0 is not None else None, dt_dev.data_ptr(), float(tol), mi,
               int(min_iter), flags, q.data_ptr() if q is not None else None, vol.data_ptr(),
               traces.data_ptr(), bad.data_ptr(), sweeps.data_ptr(), h.stream())
    nc = len(cells)
    tr = {}
    for j in range(d):
        for s in (0, 1):
            blk = traces[2 * j + s][:, :pd * m].reshape(cells + (P,) * d + (m,))
            order = tuple(range(nc)) + tuple(nc + p for p in _TRACE_PERMS[d][j]) + (nc + d,)
            tr[(j, s)] = blk.permute(order).contiguous()
    converged = (bad & _lib.PRED_NOT_CONVERGED) == 0
    admissible = (bad & _lib.PRED_INADMISSIBLE) == 0
    res = PredictorResult(q=q, iterations=int(sweeps.max().item()) if E else 0,
                          converged=converged, admissible=admissible, sweeps=sweeps,
                          traces=tr, volume=vol)
    return res, converged & admissible


def startup_guess(u, system, spacings, dt, tables, mode="conservative", width=None):
    """Initial space-time iterate (predictor.py:99-126): one explicit rate for
    degree <= 1, the two-rate third-order guess otherwise; in the iterate
    variables (primitive states for mode="primitive").  `width` (the
    reference's host batching) has no meaning on the device."""
    res, _ = run_predictor(u, system, spacings, dt, tables, mode=mode, startup_only=True)
    return res.q


def picard_solve(u, system, spacings, dt, tables, tol=1e-12, max_iter=None,
                 mode="conservative", width=None, initial=None, min_iter=1,
                 sweep_rule="global"):
    """Space-time fixed point (predictor.py:135-191) on the device.

    sweep_rule="global" (default) reproduces the reference's loop: every
    element is swept until ALL have converged (or max_iter), and
    `iterations` is that common count.  The kernel freezes each element at
    its own first converged sweep, so this runs it twice: the first launch
    finds K = the largest per-element count, the second sweeps every
    element K times (min_iter = K).  sweep_rule="element" returns the first
    launch (per-element stopping, the Simulation rule; results differ from
    the global rule by <= 1e-14).

    `converged` and `admissible` are the kernel's separate flags; `initial`
    replaces the startup guess by a given iterate (iterate variables).
    """
    if sweep_rule not in ("global", "element"):
        raise ValueError(f"unknown sweep_rule {sweep_rule!r}")
    res, _ = run_predictor(u, system, spacings, dt, tables, tol, max_iter, min_iter,
                           mode=mode, initial=initial)
    k = res.iterations
    if sweep_rule == "global" and k > max(1, int(min_iter)) and \
            bool((res.sweeps < k).any().item()):
        res, _ = run_predictor(u, system, spacings, dt, tables, tol, max_iter, k, mode=mode,
                               initial=initial)
    return res


def extract_traces(q, tables=None, dim=None):
    """Face states of the space-time polynomial (predictor.py:218-230):
    {(j, side): (cells.., tangential nodes.., P_t, m)}, side 0 the low face.
    Accepts a raw q (cells.., P.. (dim axes), P_t, m) -- contracted on the
    device by adg_extract_traces -- or a PredictorResult (the fused
    predictor's traces)."""
    if isinstance(q, PredictorResult):
        if q.traces is not None:
            return q.traces
        q = q.q
    if tables is None or dim is None:
        raise ValueError("extract_traces(q, tables, dim) needs the tables and the dimension")
    q = _device_array(q)
    P = tables.degree + 1
    d = int(dim)
    if q.ndim < d + 2 or tuple(q.shape[-d - 2:-1]) != (P,) * (d + 1):
        raise ValueError(f"q has shape {tuple(q.shape)}; expected (cells.., {P}^{d + 1}, m)")
    m = int(q.shape[-1])
    batch = tuple(q.shape[:-d - 2])
    E = int(np.prod(batch)) if batch else 1
    g = _lib.Grid()
    g.dim, g.degree, g.nvars = d, tables.degree, m
    g.mode = 0
    g.system = {d + 2: 0, 1: 1, 9: 2}.get(m, 0)
    g.gamma = 1.4
    g.cells[0], g.cells[1], g.cells[2] = E, 1, 1
    g.dx[0] = g.dx[1] = g.dx[2] = 1.0
    h = _lib.Handle.get(q.device.index)
    h.ensure_tables(tables)
    out = torch.empty(2 * d, E, P ** (d - 1) * P * m, dtype=torch.float64, device=q.device)
    if E:
        h.call("adg_extract_traces", _lib.ctypes.byref(g), q.data_ptr(), out.data_ptr(),
               h.stream())
    shape = batch + (P,) * (d - 1) + (P, m)
    return {(j, s): out[2 * j + s].reshape(shape) for j in range(d) for s in (0, 1)}


def spacetime_rate(q, system, spacings, tables, mode="conservative"):
    """L(q) at every space-time node (predictor.py:74-96): conservative
    -sum_j (D/dx_j) F_j(q), or primitive_rhs(v, grad v) for mode="primitive"
    (q then holds primitive states).  Euler."""
    _check_mode(mode)
    if getattr(system, "identity_primitives", False) and getattr(system, "name", "") != "euler":
        mode = "conservative"
    q = _device_array(q)
    d = system.dim
    cells = tuple(q.shape[:q.ndim - 2 - d])
    E = int(np.prod(cells)) if cells else 1
    h = _lib.Handle.get(q.device.index)
    h.ensure_tables(tables)
    g = _grid(system, E, spacings, tables.degree, mode=mode)
    rate = torch.empty_like(q)
    if q.numel():
        h.call("adg_spacetime_rate", _lib.ctypes.byref(g), q.data_ptr(), rate.data_ptr(),
               h.stream())
    return rate


def weak_form_defect(q, u, system, spacings, dt, tables, mode="conservative", width=None):
    """Relative residual of the space-time weak form per element
    (predictor.py:194-215): ||K1 q - (phi(0) u + dt w L(q))|| / (1 + ||q||)
    over every space-time DOF of an element -- an implementation-independent
    check of a predictor result."""
    _check_mode(mode)
    q = _device_array(q)
    u = _device_array(u, q.device)
    d = system.dim
    if mode == "primitive":
        q_it, u_it = system.cons_to_prim(q), system.cons_to_prim(u)
    else:
        q_it, u_it = q, u
    rate = spacetime_rate(q_it, system, spacings, tables, mode)
    f64 = dict(dtype=torch.float64, device=q.device)
    k1 = torch.as_tensor(tables.k1, **f64)
    phi0 = torch.as_tensor(tables.left_vals, **f64)
    w = torch.as_tensor(tables.weights, **f64)
    lhs = torch.einsum("kl,...lv->...kv", k1, q_it)
    rhs = phi0[:, None] * u_it[..., None, :] + dt * w[:, None] * rate
    red = tuple(range(q.ndim - 2 - d, q.ndim))
    res = torch.sqrt(((lhs - rhs) ** 2).sum(dim=red))
    scale = 1.0 + torch.sqrt((q_it * q_it).sum(dim=red))
    return res / scale


__all__ = ["PredictorResult", "picard_solve", "run_predictor", "startup_guess",
           "extract_traces", "spacetime_rate", "weak_form_defect", "basis_tables"]
