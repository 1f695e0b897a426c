"""Oracle: ADER-DG predictor and corrector array kernels (Euler only).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Layout is the reference's: spatial data (..., n_1..n_d, m), space-time
data (..., n_1..n_d, T, m), grid axes in front (predictor.py:1-8).
"""

from dataclasses import dataclass

import numpy as np

from .basis import oracle_tables, weight_tensor


def contract(mat, arr, axis):
    """out[..k..] = sum_l mat[k, l] arr[..l..] along `axis` (predictor.py:50-54)."""
    axis %= arr.ndim
    return np.moveaxis(np.tensordot(mat, arr, axes=(1, axis)), 0, axis)


def dg_rate(q, phys, spacings, tab):
    """L(q) = -sum_j (D/dx_j) F_j(q), accumulated x, y, z (predictor.py:74-91).

    q: (..., n_1..n_d, T, m).  Euler has no source and no NCP, so the
    accumulator starts from zero.
    """
    d = phys.dim
    m = phys.n_vars
    first = q.ndim - 2 - d
    f = phys.flux(q.reshape(-1, m)).reshape(q.shape[:-1] + (d, m))
    out = np.zeros(q.shape)
    for j in range(d):
        out -= contract(tab.diff / spacings[j], f[..., j, :], first + j)
    return out


def prim_rate(v, phys, spacings, tab):
    """primitive_rhs(v, grad v) with nodal gradients (predictor.py:65-71, :94-96)."""
    d = phys.dim
    first = v.ndim - 2 - d
    g = np.empty(v.shape[:-1] + (d, v.shape[-1]))
    for j in range(d):
        g[..., j, :] = contract(tab.diff / spacings[j], v, first + j)
    return phys.primitive_rhs(v, g)


def _with_time(u, n):
    return np.repeat(u[..., None, :], n, axis=-2)


def startup_guess(u, phys, spacings, dt, tab, mode="conservative"):
    """Initial space-time iterate (predictor.py:99-126).  In primitive mode
    u is converted first and the guess is built in primitive variables."""
    n = tab.degree
    if mode == "primitive":
        u = phys.cons_to_prim(u)
        rate = lambda w: prim_rate(w, phys, spacings, tab)  # noqa: E731
    else:
        rate = lambda w: dg_rate(w, phys, spacings, tab)  # noqa: E731
    k1 = rate(_with_time(u, 1))[..., 0, :]
    q = np.empty(u.shape[:-1] + (n + 1, u.shape[-1]))
    if n <= 1:
        for t in range(n + 1):
            q[..., t, :] = u + (tab.nodes[t] * dt) * k1
        return q
    k2 = rate(_with_time(u + dt * k1, 1))[..., 0, :]
    for t in range(n + 1):
        s = tab.nodes[t] * dt
        q[..., t, :] = u + s * k1 + (0.5 * s * s / dt) * (k2 - k1)
    return q


@dataclass
class PicardOut:
    q: np.ndarray
    iterations: int
    converged: np.ndarray
    admissible: np.ndarray
    sweeps: np.ndarray  # per element: first sweep at which it converged (0 = never)


def picard_solve(u, phys, spacings, dt, tab, tol=1e-12, max_iter=None,
                 initial=None, per_element=False, mode="conservative"):
    """Space-time Picard fixed point (predictor.py:135-191).

    per_element=False reproduces the reference's global stopping rule
    (iterate every element until all have converged).  per_element=True
    freezes each element at its own first converged sweep, the rule the
    GPU kernel uses; SURVEY.md Appendix A measured the two within 1e-14.
    """
    d = phys.dim
    if max_iter is None:
        max_iter = 2 * tab.degree + 2
    prim = mode == "primitive"
    q = startup_guess(u, phys, spacings, dt, tab, mode) if initial is None \
        else np.array(initial, dtype=float)
    u_it = phys.cons_to_prim(u) if prim else u
    red = tuple(range(u.ndim - 1 - d, q.ndim))
    grid_shape = u.shape[:-1 - d]
    converged = np.zeros(grid_shape, dtype=bool)
    first_conv = np.zeros(grid_shape, dtype=np.int32)
    frozen = np.zeros(grid_shape, dtype=bool)
    it = 0
    for _ in range(max_iter):
        rate = prim_rate(q, phys, spacings, tab) if prim else dg_rate(q, phys, spacings, tab)
        q_new = contract(tab.gw, rate, -2)
        q_new *= dt
        q_new += tab.g0[:, None] * u_it[..., None, :]
        it += 1
        delta = q - q_new
        res = tab.k1_opnorm * np.sqrt(np.sum(delta * delta, axis=red))
        scale = 1.0 + np.sqrt(np.sum(q_new * q_new, axis=red))
        conv_now = res <= tol * scale
        if per_element:
            upd = ~frozen
            q[upd] = q_new[upd]
            newly = upd & conv_now
            first_conv[newly] = it
            converged = np.where(upd, conv_now, converged)
            frozen |= conv_now
            if np.all(frozen):
                break
        else:
            q = q_new
            converged = conv_now
            first_conv[(first_conv == 0) & conv_now] = it
            if np.all(converged):
                break
    if prim:
        q = phys.prim_to_cons(q)
    ok = np.all(phys.admissible(q), axis=tuple(range(len(grid_shape), q.ndim - 1)))
    return PicardOut(q=q, iterations=it, converged=converged, admissible=ok,
                     sweeps=first_conv)


def weak_form_defect(q, u, phys, spacings, dt, tab):
    """Per-element relative weak-form residual (predictor.py:194-215)."""
    d = phys.dim
    rate = dg_rate(q, phys, spacings, tab)
    lhs = contract(tab.k1, q, -2)
    rhs = np.einsum("t,...v->...tv", tab.left_vals, u) + dt * tab.weights[:, None] * rate
    red = tuple(range(u.ndim - 1 - d, q.ndim))
    res = np.sqrt(np.sum((lhs - rhs) ** 2, axis=red))
    return res / (1.0 + np.sqrt(np.sum(q * q, axis=red)))


def extract_traces(q, tab, dim):
    """{(j, side): (..., tangential, T, m)} (predictor.py:218-230)."""
    out = {}
    for j in range(dim):
        ax = q.ndim - 2 - dim + j
        out[(j, 0)] = np.tensordot(tab.left_vals, q, axes=(0, ax))
        out[(j, 1)] = np.tensordot(tab.right_vals, q, axes=(0, ax))
    return out


def compute_timestep(u, phys, spacings, cfl, degree):
    """dt = cfl / sum_j lambda_j / dx_j over admissible nodes (corrector.py:30-55)."""
    if not cfl < 1.0 / (2 * degree + 1):
        raise ValueError("cfl violates the stability bound 1/(2N+1)")
    states = u.reshape(-1, phys.n_vars)
    ok = phys.admissible(states)
    if not np.any(ok):
        raise RuntimeError("no admissible state found while sizing the time step")
    states = states[ok]
    denom = 0.0
    for j in range(phys.dim):
        denom += float(np.max(phys.max_abs_eigenvalue_axis(states, j))) / spacings[j]
    if denom == 0.0:
        return np.inf
    return cfl / denom


def wave_speeds(u, phys):
    """Per-axis max |lambda| over admissible nodes (the GPU's reduction)."""
    states = u.reshape(-1, phys.n_vars)
    ok = phys.admissible(states)
    good = states[ok]
    lam = np.array([float(np.max(phys.max_abs_eigenvalue_axis(good, j)))
                    if good.shape[0] else 0.0 for j in range(phys.dim)])
    return lam, int(ok.sum())


def face_fluxes(qm, qp, axis, phys):
    """Rusanov one-sided face terms (corrector.py:58-62, :100-129)."""
    jump = qp - qm
    s = np.maximum(phys.max_abs_eigenvalue_axis(qm, axis),
                   phys.max_abs_eigenvalue_axis(qp, axis))
    diss = 0.5 * s[..., None] * jump
    central = 0.5 * (phys.flux(qm)[..., axis, :] + phys.flux(qp)[..., axis, :])
    zero = np.zeros_like(jump)
    return central + zero - diss, -central + zero + diss


def volume_integral(q, phys, spacings, dt, tab):
    """Space-time volume accumulator, pure-flux part (corrector.py:141-177)."""
    d = phys.dim
    m = phys.n_vars
    first = q.ndim - 2 - d
    w = tab.weights
    vol = float(np.prod(spacings))
    f = phys.flux(q.reshape(-1, m)).reshape(q.shape[:-1] + (d, m))
    wt = weight_tensor(w, d)[..., None]
    acc = dt * vol * wt * np.einsum("t,...tv->...v", w, np.zeros(q.shape))
    stiff = (tab.diff * w[:, None]).T
    for j in range(d):
        fbar = np.einsum("t,...tv->...v", w, f[..., j, :])
        contrib = contract(stiff, fbar, first + j)
        shape = [1] * d
        shape[j] = -1
        scale = (wt[..., 0] / w.reshape(shape))[..., None]
        acc += (dt * vol / spacings[j]) * scale * contrib
    return acc


def face_integral(dvals, axis, side, spacings, dt, tab, dim):
    """Face accumulator from one-sided terms (corrector.py:180-196)."""
    w = tab.weights
    dbar = np.einsum("t,...tv->...v", w, dvals)
    if dim > 1:
        dbar = dbar * weight_tensor(w, dim - 1)[..., None]
    area = float(np.prod(spacings)) / spacings[axis]
    vec = tab.right_vals if side == 1 else tab.left_vals
    out = np.moveaxis(np.tensordot(vec, dbar, axes=0), 0, dbar.ndim - dim + axis)
    return dt * area * out


def element_update(u, vol_acc, face_accs, spacings, tab, dim):
    """u* = u + (vol - sum faces) / (|cell| w_k) (corrector.py:199-205)."""
    total = vol_acc.copy()
    for a in face_accs:
        total -= a
    mass = float(np.prod(spacings)) * weight_tensor(tab.weights, dim)[..., None]
    return u + total / mass


def tables(degree):
    return oracle_tables(degree)
