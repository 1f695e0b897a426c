"""Corrector module functions on the device (reference: corrector.py).

Same names, arguments and error conventions as the reference module, for
callers that drive the pieces themselves; Simulation uses the fused
kernels instead.  Inputs may be numpy arrays or CUDA tensors; results are
CUDA fp64 tensors in the reference layouts.  The pointwise face terms cover
the three device plugins (Euler, advection, elasticity-di); face_integral /
element_update are linear and take any number of quantities;
volume_integral is the Euler kernel.
"""

import math

import numpy as np
import torch

from . import _lib
from ._pieces import as_device, flat_grid, handle_for, require_euler, scalar
from .basis import basis_tables
from .basis import weight_tensor as _weights


def max_cfl_number(degree):
    """corrector.py:25-27."""
    return 1.0 / (2 * degree + 1)


def weight_tensor(tables, dim):
    """Tensor-product quadrature weights (corrector.py:132-138)."""
    return _weights(np.asarray(tables.weights, dtype=float), dim)


def _grid_cells(u, system, degree):
    d = system.dim
    lead = u.shape[:u.ndim - 1 - d]
    return int(np.prod(lead)) if lead else 1


def _device_system(system):
    if getattr(system, "name", None) not in _lib.SYSTEM_CODES:
        raise NotImplementedError(
            f"system '{getattr(system, 'name', system)}' has no B200 kernels "
            "(euler, advection, elasticity-di)")


def compute_timestep(u, system, spacings, cfl, degree):
    """Largest stable dt over the admissible nodes (corrector.py:30-55);
    adg_wavespeed + adg_timestep."""
    if not cfl < max_cfl_number(degree):
        raise ValueError(
            f"cfl {cfl} violates the stability bound 1/(2N+1) = "
            f"{max_cfl_number(degree):.6g} for degree {degree}")
    _device_system(system)
    u = as_device(u)
    tables = basis_tables(degree)
    h = handle_for(u, tables)
    E = _grid_cells(u, system, degree)
    g = flat_grid(system, degree, E, spacings)
    red = torch.zeros(_lib.REDUCE_WORDS, dtype=torch.int64, device=u.device)
    dt = torch.empty(1, dtype=torch.float64, device=u.device)
    st = torch.zeros(1, dtype=torch.int32, device=u.device)
    gp = _lib.ctypes.byref(g)
    h.call("adg_wavespeed", gp, u.data_ptr(), red.data_ptr(), h.stream())
    h.call("adg_timestep", gp, red.data_ptr(), float(cfl), None, math.inf, dt.data_ptr(),
           st.data_ptr(), h.stream())
    if int(st.item()) & _lib.STATUS_NO_ADMISSIBLE:
        raise RuntimeError("no admissible state found while sizing the time step")
    return float(dt.item())


def rusanov_theta(q_minus, q_plus, normal, system):
    """max |eigenvalue| over both states (corrector.py:58-62):
    adg_riemann_points, speed mode (Euler, advection; the NCP system's c_p
    speed is a short device expression of its plugin)."""
    qm, qp = as_device(q_minus), as_device(q_plus)
    if getattr(system, "name", None) not in ("euler", "advection"):
        n = torch.as_tensor(np.asarray(normal, dtype=float), device=qm.device)
        return torch.maximum(system.max_abs_eigenvalue(qm, n), system.max_abs_eigenvalue(qp, n))
    qm, qp = torch.broadcast_tensors(qm, qp)
    qm, qp = qm.contiguous(), qp.contiguous()
    lead = tuple(qm.shape[:-1])
    n = int(np.prod(lead)) if lead else 1
    out = torch.empty(lead, dtype=torch.float64, device=qm.device)
    nv = np.zeros(3)
    nv[:system.dim] = np.asarray(normal, dtype=float)
    nvec = (_lib.ctypes.c_double * 3)(*nv)
    g = flat_grid(system, 0, n)
    h = _lib.Handle.get(qm.device.index)
    h.ensure_tables(basis_tables(0))
    h.call("adg_riemann_points", _lib.ctypes.byref(g), n, nvec, 2, qm.data_ptr(), qp.data_ptr(),
           out.data_ptr(), None, None, h.stream())
    return out


def _points(q_minus, q_plus, system, normal, mode, want_b=False):
    """adg_riemann_points on state pairs (..., m): (out_a, out_b, bpath)."""
    _device_system(system)
    qm, qp = as_device(q_minus), as_device(q_plus, q_minus.device
                                            if isinstance(q_minus, torch.Tensor) else None)
    m = system.n_vars
    if qm.shape != qp.shape or qm.shape[-1] != m:
        raise ValueError("q_minus / q_plus must share a (..., n_vars) shape")
    n = qm.numel() // m
    nv = np.zeros(3)
    nv[:system.dim] = np.asarray(normal, dtype=float)[:system.dim]
    nvec = (_lib.ctypes.c_double * 3)(*nv)
    out_a = torch.empty_like(qm) if mode >= 0 else None
    out_b = torch.empty_like(qm) if mode == 1 else None
    bpath = (torch.empty(tuple(qm.shape) + (m,), dtype=torch.float64, device=qm.device)
             if want_b else None)
    h = handle_for(qm, basis_tables(0))
    g = flat_grid(system, 0, 1)
    h.call("adg_riemann_points", _lib.ctypes.byref(g), int(n), nvec, int(mode), qm.data_ptr(),
           qp.data_ptr(), None if out_a is None else out_a.data_ptr(),
           None if out_b is None else out_b.data_ptr(),
           None if bpath is None else bpath.data_ptr(), h.stream())
    return out_a, out_b, bpath


def path_integral_B(q_minus, q_plus, normal, system, n_points=3):
    """int_0^1 B(psi(s)).n ds along q- -> q+ by the 3-point Gauss rule
    (corrector.py:65-78); zeros for flux-only systems."""
    if n_points != 3:
        raise NotImplementedError("the device path rule is the reference's 3-point Gauss rule")
    if not getattr(system, "has_ncp", False):
        qm = as_device(q_minus)
        m = system.n_vars
        return torch.zeros(tuple(qm.shape[:-1]) + (m, m), dtype=torch.float64, device=qm.device)
    return _points(q_minus, q_plus, system, normal, -1, want_b=True)[2]


def riemann_dminus(q_minus, q_plus, normal, system):
    """One-sided face term for the element with outward normal `normal`
    (corrector.py:81-97)."""
    return _points(q_minus, q_plus, system, normal, 0)[0]


def face_fluxes(q_minus, q_plus, axis, system):
    """Both one-sided face terms of an interface with normal +e_axis
    (corrector.py:100-129); d_low + d_high == 0 bit for bit for flux systems.
    Euler goes through adg_face_fluxes (the subcell rescue's pair), the
    other plugins through adg_riemann_points."""
    if getattr(system, "name", None) != "euler":
        nv = np.zeros(system.dim)
        nv[axis] = 1.0
        d_low, d_high, _ = _points(q_minus, q_plus, system, nv, 1)
        return d_low, d_high
    qm, qp = as_device(q_minus), as_device(q_plus)
    if qm.shape != qp.shape or qm.shape[-1] != system.n_vars:
        raise ValueError("q_minus / q_plus must share a (..., n_vars) shape")
    n = qm.numel() // system.n_vars
    dlow = torch.empty_like(qm)
    dhigh = torch.empty_like(qm)
    h = handle_for(qm, basis_tables(0))
    g = flat_grid(system, 0, 1)
    h.call("adg_face_fluxes", _lib.ctypes.byref(g), int(axis), int(n), qm.data_ptr(),
           qp.data_ptr(), dlow.data_ptr(), dhigh.data_ptr(), h.stream())
    return dlow, dhigh


def volume_integral(q, system, spacings, dt, tables, width=None):
    """Space-time volume accumulator from a given predictor q
    (..., n_1..n_d, T, m) -> (..., n_1..n_d, m) (corrector.py:141-177)."""
    require_euler(system)
    q = as_device(q)
    d = system.dim
    P = tables.degree + 1
    lead = q.shape[:q.ndim - 2 - d]
    E = int(np.prod(lead)) if lead else 1
    if tuple(q.shape[q.ndim - 2 - d:]) != (P,) * (d + 1) + (system.n_vars,):
        raise ValueError(f"q has shape {tuple(q.shape)}; expected (..., {P}^{d + 1}, m)")
    vol = torch.empty(tuple(lead) + (P,) * d + (system.n_vars,), dtype=torch.float64,
                      device=q.device)
    h = handle_for(q, tables)
    g = flat_grid(system, tables.degree, E, spacings)
    dt_dev = scalar(dt, q.device)
    h.call("adg_volume_integral", _lib.ctypes.byref(g), q.data_ptr(), dt_dev.data_ptr(),
           vol.data_ptr(), h.stream())
    return vol


def face_integral(d_values, axis, side, spacings, dt, tables, dim):
    """Face accumulator (corrector.py:180-196): d_values (..., P^(d-1)
    tangential.., T, m) -> (..., n_1..n_d, m)."""
    dv = as_device(d_values)
    P = tables.degree + 1
    m = dv.shape[-1]
    lead = dv.shape[:dv.ndim - 1 - dim]
    E = int(np.prod(lead)) if lead else 1
    out = torch.empty(tuple(lead) + (P,) * dim + (m,), dtype=torch.float64, device=dv.device)
    system = _Shape(dim, m)
    h = handle_for(dv, tables)
    g = flat_grid(system, tables.degree, E, spacings)
    dt_dev = scalar(dt, dv.device)
    h.call("adg_face_integral", _lib.ctypes.byref(g), int(axis), int(side), dv.data_ptr(),
           dt_dev.data_ptr(), out.data_ptr(), h.stream())
    return out


def element_update(u, volume_acc, face_accs, spacings, tables, dim):
    """u + M^-1 (volume - sum of face integrals) (corrector.py:199-205)."""
    u = as_device(u)
    vol = as_device(volume_acc)
    accs = [as_device(a) for a in face_accs]
    if len(accs) > 6:
        raise ValueError("at most 2 dim face accumulators")
    m = u.shape[-1]
    lead = u.shape[:u.ndim - 1 - dim]
    E = int(np.prod(lead)) if lead else 1
    out = torch.empty_like(u)
    ptrs = (_lib.ctypes.c_void_p * max(len(accs), 1))(*[a.data_ptr() for a in accs])
    h = handle_for(u, tables)
    g = flat_grid(_Shape(dim, m), tables.degree, E, spacings)
    h.call("adg_element_update", _lib.ctypes.byref(g), u.data_ptr(), vol.data_ptr(),
           _lib.ctypes.cast(ptrs, _lib.ctypes.c_void_p), len(accs), out.data_ptr(), h.stream())
    return out


class _Shape:
    """Minimal descriptor for the linear, system-independent calls."""

    name = "euler"
    gamma = 1.4

    def __init__(self, dim, m):
        self.dim = dim
        self.n_vars = m


__all__ = ["max_cfl_number", "weight_tensor", "compute_timestep", "rusanov_theta",
           "path_integral_B", "riemann_dminus", "face_fluxes", "volume_integral",
           "face_integral", "element_update"]
