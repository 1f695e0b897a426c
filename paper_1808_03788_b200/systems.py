"""PDE plugin descriptors (reference contract: systems.py:16-74).

On the B200 path the physics is a compile-time policy inside the CUDA
kernels (csrc/adg_common.cuh: flux_all, max_abs_eig, admissible); these
classes carry the plugin's identity and parameters (`name`, `dim`,
`n_vars`, `gamma`, ...) across the C-ABI, exactly the attributes the
reference's driver reads.  The elementwise methods are kept for API
compatibility (user-side IC / diagnostics code calls them); they accept
numpy arrays or torch tensors and are never on the time-step path.
"""

import numpy as np


def _xp(a):
    try:
        import torch

        if isinstance(a, torch.Tensor):
            return torch
    except ImportError:  # pragma: no cover
        pass
    return np


class HyperbolicSystem:
    name = "base"
    has_flux = False
    has_ncp = False
    has_source = False
    identity_primitives = True
    diss_mask = None

    def __init__(self, dim, n_vars, quantity_names):
        self.dim = dim
        self.n_vars = n_vars
        self.quantity_names = tuple(quantity_names)


class CompressibleEuler(HyperbolicSystem):
    """Ideal-gas Euler, conserved (rho, rho v_1..d, rho E) (systems.py:112-234)."""

    name = "euler"
    has_flux = True

    def __init__(self, dim, gamma=1.4):
        if not 1 <= dim <= 3:
            raise ValueError("dim must be 1, 2 or 3")
        names = ("rho",) + tuple(f"mom_{'xyz'[j]}" for j in range(dim)) + ("energy",)
        super().__init__(dim, dim + 2, names)
        self.gamma = float(gamma)
        self.identity_primitives = False

    def pressure(self, q):
        kin = q[..., 1] * q[..., 1]
        for j in range(1, self.dim):
            kin = kin + q[..., 1 + j] * q[..., 1 + j]
        return (self.gamma - 1.0) * (q[..., -1] - 0.5 * kin / q[..., 0])

    def sound_speed(self, q):
        xp = _xp(q)
        return xp.sqrt(self.gamma * self.pressure(q) / q[..., 0])

    def flux(self, q):
        xp = _xp(q)
        d = self.dim
        r = 1.0 / q[..., 0]
        p = self.pressure(q)
        ep = q[..., d + 1] + p
        rows = []
        for j in range(d):
            vj = q[..., 1 + j] * r
            comp = [q[..., 1 + j]] + [q[..., 1 + i] * vj + (p if i == j else 0.0)
                                     for i in range(d)] + [ep * vj]
            rows.append(xp.stack(comp, axis=-1) if xp is np else xp.stack(comp, dim=-1))
        return np.stack(rows, axis=-2) if xp is np else xp.stack(rows, dim=-2)

    def max_abs_eigenvalue(self, q, normal):
        un = 0.0
        for j in range(self.dim):
            un = un + q[..., 1 + j] * float(normal[j])
        return abs(un / q[..., 0]) + self.sound_speed(q)

    def admissible(self, q):
        xp = _xp(q)
        if xp is np:
            fin = np.all(np.isfinite(q), axis=-1)
            with np.errstate(invalid="ignore", divide="ignore"):
                return fin & (q[..., 0] > 0.0) & (self.pressure(q) > 0.0)
        return xp.isfinite(q).all(dim=-1) & (q[..., 0] > 0.0) & (self.pressure(q) > 0.0)

    def reflect(self, q, axis):
        out = q.copy() if _xp(q) is np else q.clone()
        out[..., 1 + axis] = -q[..., 1 + axis]
        return out


class LinearAdvection(HyperbolicSystem):
    """Scalar transport q_t + a . grad q = 0 with constant velocity a
    (systems.py:77-109); device kernels in csrc/adg_advection.cu."""

    name = "advection"
    has_flux = True

    def __init__(self, dim, velocity=None):
        if not 1 <= dim <= 3:
            raise ValueError("dim must be 1, 2 or 3")
        super().__init__(dim, 1, ("q",))
        if velocity is None:
            velocity = [1.0] * dim
        self.velocity = np.asarray(velocity, dtype=float)
        if self.velocity.shape != (dim,):
            raise ValueError("advection velocity must have one entry per dimension")

    def flux(self, q):
        out = np.empty(q.shape[:-1] + (self.dim, 1))
        for j in range(self.dim):
            out[..., j, 0] = self.velocity[j] * q[..., 0]
        return out

    def max_abs_eigenvalue(self, q, normal):
        a_n = abs(float(np.dot(self.velocity, normal)))
        return np.broadcast_to(a_n, q.shape[:-1]).copy()

    def admissible(self, q):
        xp = _xp(q)
        if xp is np:
            return np.all(np.isfinite(q), axis=-1)
        return xp.isfinite(q).all(dim=-1)

    def cons_to_prim(self, q):
        return q

    def prim_to_cons(self, v):
        return v

    def reflect(self, q, axis):
        return q.copy() if _xp(q) is np else q.clone()


ALPHA_FLOOR = 1e-3   # systems.py:13


class DiffuseInterfaceElasticity(HyperbolicSystem):
    """2-D linear elasticity with a diffuse solid boundary (systems.py:237-345):
    state (sxx, syy, sxy, avx, avy, alpha, lam, mu, rho), a pure
    nonconservative product B(q).grad q, wave speeds c_p / c_s from the
    material constants.  Device kernels in csrc/adg_elasticity.cu (predictor
    with rate -ncp(q, grad q), path-conservative faces, update)."""

    name = "elasticity-di"
    has_flux = False
    has_ncp = True
    SXX, SYY, SXY, AVX, AVY, ALPHA, LAM, MU, RHO = range(9)
    # alpha and the material constants obey d/dt = 0: no jump dissipation
    diss_mask = np.array([1.0, 1.0, 1.0, 1.0, 1.0, 0.0, 0.0, 0.0, 0.0])

    def __init__(self, dim=2):
        if dim != 2:
            raise ValueError("the diffuse-interface elasticity system is 2-D")
        super().__init__(2, 9, ("sxx", "syy", "sxy", "avx", "avy", "alpha", "lam", "mu", "rho"))

    def max_abs_eigenvalue(self, q, normal):
        xp = _xp(q)
        return xp.sqrt((q[..., self.LAM] + 2.0 * q[..., self.MU]) / q[..., self.RHO])

    def eigenvalues(self, q, normal):
        c_p = np.sqrt((q[..., self.LAM] + 2.0 * q[..., self.MU]) / q[..., self.RHO])
        c_s = np.sqrt(q[..., self.MU] / q[..., self.RHO])
        out = np.zeros(q.shape[:-1] + (9,))
        out[..., 0] = -c_p
        out[..., 1] = -c_s
        out[..., 7] = c_s
        out[..., 8] = c_p
        return out

    def admissible(self, q):
        xp = _xp(q)
        if xp is np:
            return np.all(np.isfinite(q), axis=-1)
        return xp.isfinite(q).all(dim=-1)

    def cons_to_prim(self, q):
        return q

    def prim_to_cons(self, v):
        return v

    def reflect(self, q, axis):
        out = q.copy() if _xp(q) is np else q.clone()
        if axis == 0:
            out[..., self.SXX] = -q[..., self.SXX]
            out[..., self.SXY] = -q[..., self.SXY]
        else:
            out[..., self.SYY] = -q[..., self.SYY]
            out[..., self.SXY] = -q[..., self.SXY]
        return out


_SYSTEMS = {"euler": CompressibleEuler, "advection": LinearAdvection,
            "elasticity-di": DiffuseInterfaceElasticity}


def make_system(name, dim, **params):
    """Registered systems (systems.py:355-361): Euler, advection and the 2-D
    diffuse-interface elasticity all have a B200 path."""
    try:
        cls = _SYSTEMS[name]
    except KeyError:
        raise ValueError(f"unknown system '{name}' (choose from ['advection', "
                         "'elasticity-di', 'euler'])")
    return cls(dim, **params)
