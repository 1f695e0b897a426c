"""Oracle: a posteriori subcell MOOD limiter (Euler, conservative mode).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates reference `pkg/src/aderdg/limiter.py`.
"""

import numpy as np

from .dg import contract, face_fluxes

DMP_DELTA0 = 1e-3   # limiter.py:22 (SPEC.md says 1e-4; the code is the oracle)
DMP_EPS = 1e-3      # limiter.py:23
MAX_HALVINGS = 3    # limiter.py:24


def to_subcells(u, tab, dim):
    """Nodal -> (2N+1)^d subcell averages (limiter.py:27-33)."""
    first = u.ndim - 1 - dim
    for j in range(dim):
        u = contract(tab.sub_project, u, first + j)
    return u


def from_subcells(ubar, tab, dim):
    """Subcell averages -> nodal, mean preserving (limiter.py:36-42)."""
    first = ubar.ndim - 1 - dim
    for j in range(dim):
        ubar = contract(tab.sub_recover, ubar, first + j)
    return ubar


def minmod(a, b):
    """limiter.py:45-48."""
    return np.where(a * b > 0.0, np.where(np.abs(a) <= np.abs(b), a, b), 0.0)


def relaxed_bounds(prev_cells, dim, delta0=DMP_DELTA0, eps=DMP_EPS):
    """DMP bounds over own + 2d face neighbours (limiter.py:51-73).

    prev_cells: (g1+2, .., gd+2, s.., m) subcell averages, 1 ghost cell/side.
    """
    sub = tuple(range(dim, 2 * dim))
    cmin = prev_cells.min(axis=sub)
    cmax = prev_cells.max(axis=sub)
    inner = tuple(slice(1, -1) for _ in range(dim))
    lo = cmin[inner].copy()
    hi = cmax[inner].copy()
    for j in range(dim):
        for sh in (-1, 1):
            sl = tuple(slice(1 + sh, (-1 + sh) or None) if i == j else slice(1, -1)
                       for i in range(dim))
            np.minimum(lo, cmin[sl], out=lo)
            np.maximum(hi, cmax[sl], out=hi)
    delta = np.maximum(delta0, eps * (hi - lo))
    return lo - delta, hi + delta


def detect(candidate, cand_sub, bounds, phys, dim):
    """Troubled-cell screen (limiter.py:76-86)."""
    lo, hi = bounds
    g = candidate.ndim - 1 - dim
    sub = tuple(range(g, g + dim))
    ex = (slice(None),) * g + (None,) * dim
    out = (cand_sub < lo[ex]) | (cand_sub > hi[ex])
    flags = np.any(out, axis=sub + (cand_sub.ndim - 1,))
    node_ok = np.all(phys.admissible(candidate), axis=sub)
    sub_ok = np.all(phys.admissible(cand_sub), axis=sub)
    return flags | ~node_ok | ~sub_ok


def windows(padded, starts, size, dim):
    """(T, size^d, m) windows out of a padded global field (limiter.py:89-101)."""
    n = starts.shape[0]
    idx = []
    for j in range(dim):
        shape = [n] + [1] * dim
        shape[1 + j] = size
        idx.append((starts[:, j][:, None] + np.arange(size)[None, :]).reshape(shape))
    return padded[tuple(idx)]


def _hancock(win, phys, h, dt, flat, mode="conservative"):
    """One MUSCL-Hancock pass over windows (limiter.py:124-202)."""
    d = phys.dim
    m = phys.n_vars
    prim = mode == "primitive"
    cons = win
    if prim:
        win = phys.cons_to_prim(win)

    def g(sls):
        return (slice(None),) + sls + (slice(None),)

    inner = tuple(slice(1, -1) for _ in range(d))
    c = win[g(inner)]
    slope = np.zeros(c.shape[:-1] + (d, m))
    if not flat:
        for j in range(d):
            up = tuple(slice(2, None) if i == j else slice(1, -1) for i in range(d))
            dn = tuple(slice(None, -2) if i == j else slice(1, -1) for i in range(d))
            fwd = (win[g(up)] - c) / h[j]
            bwd = (c - win[g(dn)]) / h[j]
            slope[..., j, :] = minmod(fwd, bwd)
    if prim:
        half = c + (0.5 * dt) * phys.primitive_rhs(c, slope)
    else:
        rate = np.zeros_like(c)
        for j in range(d):
            off = 0.5 * h[j] * slope[..., j, :]
            fh = phys.flux(c + off)[..., j, :]
            fl = phys.flux(c - off)[..., j, :]
            rate = rate - (fh - fl) / h[j]
        half = c + (0.5 * dt) * rate
    ok = np.ones(win.shape[0], dtype=bool)
    lo_f, hi_f = [], []
    axes = tuple(range(1, 1 + d))
    for j in range(d):
        off = 0.5 * h[j] * slope[..., j, :]
        lo_q, hi_q = half - off, half + off
        if prim:
            lo_q, hi_q = phys.prim_to_cons(lo_q), phys.prim_to_cons(hi_q)
        lo_f.append(lo_q)
        hi_f.append(hi_q)
        ok &= np.all(phys.admissible(lo_q), axis=axes)
        ok &= np.all(phys.admissible(hi_q), axis=axes)
    new = cons[g(tuple(slice(2, -2) for _ in range(d)))].copy()
    for j in range(d):
        qm_sl = tuple(slice(None, -1) if i == j else slice(1, -1) for i in range(d))
        qp_sl = tuple(slice(1, None) if i == j else slice(1, -1) for i in range(d))
        d_lo, d_hi = face_fluxes(hi_f[j][g(qm_sl)], lo_f[j][g(qp_sl)], j, phys)
        hi_faces = tuple(slice(1, None) if i == j else slice(None) for i in range(d))
        lo_faces = tuple(slice(None, -1) if i == j else slice(None) for i in range(d))
        new -= (dt / h[j]) * (d_lo[g(hi_faces)] + d_hi[g(lo_faces)])
    ok &= np.all(phys.admissible(new), axis=axes)
    return new, ~ok


def muscl_step(win, phys, h, dt, mode="conservative"):
    """MUSCL-Hancock with first-order retry (limiter.py:104-121)."""
    new, bad = _hancock(win, phys, h, dt, flat=False, mode=mode)
    failed = np.zeros(win.shape[0], dtype=bool)
    if np.any(bad):
        redo, still = _hancock(win[bad], phys, h, dt, flat=True, mode=mode)
        new[bad] = redo
        failed[np.flatnonzero(bad)[still]] = True
    return new, failed


def flatten(nodal, averages, phys, tab, dim):
    """Flatten cells whose nodal or subcell states are inadmissible
    (limiter.py:205-223)."""
    axes = tuple(range(1, 1 + dim))
    ok = np.all(phys.admissible(nodal), axis=axes)
    ok &= np.all(phys.admissible(to_subcells(nodal, tab, dim)), axis=axes)
    if np.all(ok):
        return nodal, 0
    mean = averages.mean(axis=axes)
    flat = np.broadcast_to(mean[(slice(None),) + (None,) * dim], nodal.shape).copy()
    bad = ~ok
    nodal[bad] = flat[bad]
    return nodal, int(bad.sum())
