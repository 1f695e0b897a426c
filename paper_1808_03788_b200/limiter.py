"""Limiter module functions on the device (reference: limiter.py).

Same names, arguments and results as the reference module for callers
that run the subcell limiter pieces themselves; Simulation uses the fused
adg_detect / adg_rescue path instead.  Every function runs in the library's
kernels (torch only holds the device buffers).  Inputs may be numpy arrays
or CUDA tensors; results are CUDA tensors.  The projection, recovery, MUSCL
step and flattening are Euler's; minmod, the bounds, the screen (Euler,
advection, elasticity-di) and the window gather take any state width.
"""

import numpy as np
import torch

from . import _lib
from ._pieces import as_device, flat_grid, handle_for, require_euler, scalar
from .basis import basis_tables

DMP_DELTA0 = 1e-3
DMP_EPS = 1e-3
MAX_HALVINGS = 3


def _system_for(dim, m, system=None):
    if system is not None:
        require_euler(system)
        return system
    from .systems import CompressibleEuler

    if m != dim + 2:
        raise NotImplementedError("Euler states only (m = d + 2)")
    return CompressibleEuler(dim)


def _lead(a, dim):
    lead = tuple(a.shape[:a.ndim - 1 - dim])
    return lead, int(np.prod(lead)) if lead else 1


def project_to_subcells(u, tables, dim):
    """(..., n.., m) -> (..., s.., m) subcell averages (limiter.py:27-33):
    adg_project_subcells."""
    u = as_device(u)
    m = u.shape[-1]
    sysd = _system_for(dim, m)
    lead, E = _lead(u, dim)
    S = tables.n_subcells
    out = torch.empty(lead + (S,) * dim + (m,), dtype=torch.float64, device=u.device)
    cmin = torch.empty(E * m, dtype=torch.float64, device=u.device)
    cmax = torch.empty_like(cmin)
    h = handle_for(u, tables)
    g = flat_grid(sysd, tables.degree, E)
    h.call("adg_project_subcells", _lib.ctypes.byref(g), u.data_ptr(), out.data_ptr(),
           cmin.data_ptr(), cmax.data_ptr(), h.stream())
    return out


def recover_from_subcells(ubar, tables, dim):
    """Mean-preserving recovery (limiter.py:36-42): adg_recover_subcells."""
    ubar = as_device(ubar)
    m = ubar.shape[-1]
    sysd = _system_for(dim, m)
    lead, E = _lead(ubar, dim)
    P = tables.degree + 1
    out = torch.empty(lead + (P,) * dim + (m,), dtype=torch.float64, device=ubar.device)
    h = handle_for(ubar, tables)
    g = flat_grid(sysd, tables.degree, E)
    h.call("adg_recover_subcells", _lib.ctypes.byref(g), ubar.data_ptr(), out.data_ptr(),
           h.stream())
    return out


def minmod(a, b):
    """Componentwise minmod (limiter.py:45-48): adg_minmod."""
    a, b = as_device(a), as_device(b)
    a, b = torch.broadcast_tensors(a, b)
    a, b = a.contiguous(), b.contiguous()
    out = torch.empty_like(a)
    h = _lib.Handle.get(a.device.index)
    h.call("adg_minmod", int(a.numel()), a.data_ptr(), b.data_ptr(), out.data_ptr(), h.stream())
    return out


def relaxed_bounds(prev_sub_cells, dim, delta0=DMP_DELTA0, eps=DMP_EPS):
    """DMP bounds over the own and 2d face-neighbour cells of a one-cell
    padded grid (limiter.py:51-73): adg_relaxed_bounds."""
    x = as_device(prev_sub_cells).contiguous()
    if x.ndim != 2 * dim + 1 or any(n < 3 for n in x.shape[:dim]):
        raise ValueError("prev_sub_cells must be (cells + 2.., s.., m) with a one-cell pad")
    m = int(x.shape[-1])
    cells = [int(n) - 2 for n in x.shape[:dim]]
    nsub = int(np.prod(x.shape[dim:2 * dim]))
    npad = int(np.prod(x.shape[:dim]))
    f64 = dict(dtype=torch.float64, device=x.device)
    cmin, cmax = torch.empty(npad * m, **f64), torch.empty(npad * m, **f64)
    lo, hi = torch.empty(tuple(cells) + (m,), **f64), torch.empty(tuple(cells) + (m,), **f64)
    carr = (_lib.ctypes.c_int64 * dim)(*cells)
    h = _lib.Handle.get(x.device.index)
    h.call("adg_relaxed_bounds", dim, m, carr, nsub, x.data_ptr(), float(delta0), float(eps),
           cmin.data_ptr(), cmax.data_ptr(), lo.data_ptr(), hi.data_ptr(), h.stream())
    return lo, hi


def detect_troubled(candidate, cand_sub, bounds, system, dim):
    """True where a candidate cell needs the FV rescue (limiter.py:76-86):
    adg_detect_cells."""
    from .corrector import _device_system

    _device_system(system)
    cand = as_device(candidate).contiguous()
    sub = as_device(cand_sub).contiguous()
    lo, hi = (as_device(b).contiguous() for b in bounds)
    lead, E = _lead(cand, dim)
    P = int(cand.shape[-2])
    out = torch.empty(lead if lead else (1,), dtype=torch.uint8, device=cand.device)
    g = flat_grid(system, P - 1, E)
    h = _lib.Handle.get(cand.device.index)
    h.ensure_tables(basis_tables(P - 1))
    h.call("adg_detect_cells", _lib.ctypes.byref(g), cand.data_ptr(), sub.data_ptr(),
           lo.data_ptr(), hi.data_ptr(), out.data_ptr(), h.stream())
    out = out.bool()
    return out if lead else out[0]


def gather_windows(padded, starts, size, dim):
    """(T, size.., m) windows out of a padded global subcell field
    (limiter.py:89-101): adg_gather_windows."""
    x = as_device(padded).contiguous()
    st = torch.as_tensor(np.asarray(starts), dtype=torch.int64, device=x.device).reshape(-1, dim)
    st = st.contiguous()
    n, m = int(st.shape[0]), int(x.shape[-1])
    out = torch.empty((n,) + (int(size),) * dim + (m,), dtype=torch.float64, device=x.device)
    darr = (_lib.ctypes.c_int64 * dim)(*[int(v) for v in x.shape[:dim]])
    h = _lib.Handle.get(x.device.index)
    h.call("adg_gather_windows", dim, m, darr, x.data_ptr(), st.data_ptr(), n, int(size),
           out.data_ptr(), h.stream())
    return out


def muscl_subcell_step(windows, system, sub_spacings, dt, mode="conservative"):
    """One MUSCL-Hancock step with first-order retry on batched windows
    (T, S+4.., m) -> (new (T, S.., m), failed (T,)) (limiter.py:104-121):
    adg_muscl_windows (the fused rescue kernel's window stage)."""
    require_euler(system)
    win = as_device(windows)
    dim = system.dim
    T = win.shape[0]
    W = win.shape[1]
    S = W - 4
    if S < 1 or S % 2 == 0:
        raise ValueError("windows must be (T, S+4, .., m) with S = 2N + 1")
    N = (S - 1) // 2
    tables = basis_tables(N)
    out = torch.empty((T,) + (S,) * dim + (system.n_vars,), dtype=torch.float64,
                      device=win.device)
    failed = torch.zeros(T, dtype=torch.uint8, device=win.device)
    if T == 0:
        return out, failed.bool()
    count = torch.full((1,), T, dtype=torch.int32, device=win.device)
    # for adg_muscl_windows the grid's dx are the subcell widths
    g = flat_grid(system, N, 1, sub_spacings, mode=mode)
    hnd = handle_for(win, tables)
    dt_dev = scalar(dt, win.device)
    hnd.call("adg_muscl_windows", _lib.ctypes.byref(g), win.data_ptr(), int(T),
             count.data_ptr(), dt_dev.data_ptr(), out.data_ptr(), failed.data_ptr(), hnd.stream())
    return out, failed.bool()


def flatten_inadmissible(nodal, averages, system, tables, dim):
    """Replace cells with inadmissible nodal or subcell-projected states by
    their subcell mean (limiter.py:205-223); returns (nodal, count)."""
    require_euler(system)
    nod = as_device(nodal).clone()
    avg = as_device(averages)
    lead, E = _lead(nod, dim)
    nflat = torch.zeros(1, dtype=torch.int32, device=nod.device)
    h = handle_for(nod, tables)
    g = flat_grid(system, tables.degree, E)
    h.call("adg_flatten_cells", _lib.ctypes.byref(g), nod.data_ptr(), avg.data_ptr(),
           nflat.data_ptr(), h.stream())
    return nod, int(nflat.item())


__all__ = ["DMP_DELTA0", "DMP_EPS", "MAX_HALVINGS", "project_to_subcells",
           "recover_from_subcells", "minmod", "relaxed_bounds", "detect_troubled",
           "gather_windows", "muscl_subcell_step", "flatten_inadmissible"]
