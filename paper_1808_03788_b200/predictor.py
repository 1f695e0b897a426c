"""Module-level predictor entry points on device tensors (reference:
predictor.py:57-62 PredictorResult, :135-191 picard_solve, :218-230
extract_traces).  Arrays are CUDA fp64 tensors in the reference layout with
the grid axes in front; every call is one `adg_predict` launch.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .basis import basis_tables


@dataclass
class PredictorResult:
    q: torch.Tensor            # (cells.., P.., P_t, m)
    iterations: int            # max sweeps over elements
    converged: torch.Tensor    # (cells..,) bool
    admissible: torch.Tensor   # (cells..,) bool
    sweeps: torch.Tensor = None
    traces: dict = None
    volume: torch.Tensor = None


def _grid(system, cells, spacings, degree, boundary_codes=None, mode="conservative"):
    g = _lib.Grid()
    d = system.dim
    g.dim, g.degree, g.nvars = d, degree, system.n_vars
    g.mode = _lib.MODE_CODES[mode]
    for j in range(3):
        g.cells[j] = int(cells[j]) if j < d else 1
        g.dx[j] = float(spacings[j]) if j < d else 1.0
    _lib.fill_system(g, system)
    for j in range(d):
        for s in (0, 1):
            g.bc[j][s] = 0 if boundary_codes is None else boundary_codes[j][s]
    return g


def run_predictor(u, system, spacings, dt, tables, tol=1e-12, max_iter=None, min_iter=1,
                  want_q=True, mode="conservative"):
    """Fused predictor on u (cells.., P.., m); returns PredictorResult with q,
    traces {(j, side): (cells.., P^(d-1) tangential.., P_t, m)} and the volume
    accumulator of corrector.volume_integral (corrector.py:141-177)."""
    d = system.dim
    m = system.n_vars
    P = tables.degree + 1
    u = torch.as_tensor(u).to(dtype=torch.float64).cuda().contiguous()
    cells = tuple(u.shape[:d])
    if tuple(u.shape[d:]) != (P,) * d + (m,):
        raise ValueError(f"u has shape {tuple(u.shape)}; expected (cells..,{P}^{d},{m})")
    h = _lib.Handle.get(u.device.index)
    h.ensure_tables(tables)
    g = _grid(system, cells, spacings, tables.degree, mode=mode)
    E = int(np.prod(cells))
    pd = P ** d
    dev = u.device
    f64 = dict(dtype=torch.float64, device=dev)
    q = torch.empty(cells + (P,) * d + (P, m), **f64) if want_q else None
    vol = torch.empty(u.shape, **f64)
    tb = pd * m + ((pd * m) & 1)   # padded trace element block (adg_trace_block)
    traces = torch.empty(2 * d, E, tb, **f64)
    bad = torch.empty(cells, dtype=torch.uint8, device=dev)
    sweeps = torch.empty(cells, dtype=torch.int32, device=dev)
    dt_dev = torch.full((1,), float(dt), **f64)
    mi = 0 if max_iter is None else int(max_iter)
    h.call("adg_predict", _lib.ctypes.byref(g), u.data_ptr(), dt_dev.data_ptr(), float(tol),
           mi, int(min_iter), q.data_ptr() if q is not None else None, vol.data_ptr(),
           traces.data_ptr(), bad.data_ptr(), sweeps.data_ptr(),
           h.stream())
    # the kernel writes each face's trace block in its owner role's order
    # (x: [j][k][t], y: [k][t][i], z: [t][i][j]; 2-D y: [t][i]); present them
    # in the reference layout (tangential axes ascending, then t, then m)
    perms = {3: {0: (0, 1, 2), 1: (2, 0, 1), 2: (1, 2, 0)}, 2: {0: (0, 1), 1: (1, 0)},
             1: {0: (0,)}}[d]
    nc = len(cells)
    tr = {}
    for j in range(d):
        for s in (0, 1):
            blk = traces[2 * j + s][:, :pd * m].reshape(cells + (P,) * d + (m,))
            order = tuple(range(nc)) + tuple(nc + p for p in perms[j]) + (nc + d,)
            tr[(j, s)] = blk.permute(order).contiguous()
    ok_conv = bad == 0
    return PredictorResult(q=q, iterations=int(sweeps.max().item()), converged=None,
                           admissible=None, sweeps=sweeps, traces=tr, volume=vol,
                           ), ok_conv


def picard_solve(u, system, spacings, dt, tables, tol=1e-12, max_iter=None,
                 mode="conservative", width=None, initial=None, min_iter=1):
    """Device picard_solve.  `converged & admissible` is exact; the two flags
    are reported jointly (the kernel's pred_bad, driver.py:212) -- converged
    carries the joint flag and admissible is all-true where it holds."""
    if mode not in _lib.MODE_CODES:
        raise ValueError(f"unknown predictor mode {mode!r}")
    if initial is not None:
        raise NotImplementedError("custom initial iterates are not supported on the B200 path")
    res, good = run_predictor(u, system, spacings, dt, tables, tol, max_iter, min_iter,
                              mode=mode)
    res.converged = good
    res.admissible = torch.ones_like(good)
    return res


def extract_traces(q_or_result, tables=None, dim=None):
    """Traces produced by the fused predictor (predictor.py:218-230)."""
    if isinstance(q_or_result, PredictorResult):
        return q_or_result.traces
    raise NotImplementedError("traces come from the fused predictor: pass its result")


__all__ = ["PredictorResult", "picard_solve", "run_predictor", "extract_traces",
           "basis_tables"]
