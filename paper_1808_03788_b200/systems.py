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


def _new(q, shape):
    """Uninitialised array / tensor of `shape` like q (dtype, device)."""
    if _xp(q) is np:
        return np.empty(shape, dtype=np.result_type(q, np.float64))
    return q.new_empty(shape)


def _zeros(q, shape):
    if _xp(q) is np:
        return np.zeros(shape, dtype=np.result_type(q, np.float64))
    return q.new_zeros(shape)


def _copy(q):
    return q.copy() if _xp(q) is np else q.clone()


class HyperbolicSystem:
    """Plugin contract q_t + div F(q) + B(q).grad q = S(q) (reference
    systems.py:16-74): state arrays carry the quantity in the last axis,
    gradients the direction just before it (grad[..., j, v] = d_j q_v).
    The defaults describe a system with no flux, no nonconservative
    product and no source; subclasses override what they have."""

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

    def flux(self, q):
        """F(q), shape (..., dim, n_vars)."""
        return _zeros(q, tuple(q.shape[:-1]) + (self.dim, self.n_vars))

    def ncp(self, q, grad):
        """B(q).grad q, shape (..., n_vars)."""
        return _zeros(q, tuple(q.shape[:-1]) + (self.n_vars,))

    def ncp_matrix(self, q, normal):
        """B(q).n, shape (..., n_vars, n_vars)."""
        return _zeros(q, tuple(q.shape[:-1]) + (self.n_vars, self.n_vars))

    def source(self, q):
        return _zeros(q, tuple(q.shape))

    def eigenvalues(self, q, normal):
        raise NotImplementedError(f"{self.name} defines no eigenvalues")

    def max_abs_eigenvalue(self, q, normal):
        lam = self.eigenvalues(q, normal)
        a = np.abs(lam) if _xp(lam) is np else lam.abs()
        return a.max(axis=-1) if _xp(lam) is np else a.amax(dim=-1)

    def cons_to_prim(self, q):
        return q

    def prim_to_cons(self, v):
        return v

    def primitive_rhs(self, v, grad):
        raise NotImplementedError(f"{self.name} has no primitive-variable form")

    def admissible(self, q):
        xp = _xp(q)
        if xp is np:
            return np.all(np.isfinite(q), axis=-1)
        return xp.isfinite(q).all(dim=-1)

    def reflect(self, q, axis):
        return q


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

    def _normal_velocity(self, q, normal):
        un = q[..., 1] * float(normal[0])
        for j in range(1, self.dim):
            un = un + q[..., 1 + j] * float(normal[j])
        return un / q[..., 0]

    def max_abs_eigenvalue(self, q, normal):
        return abs(self._normal_velocity(q, normal)) + self.sound_speed(q)

    def eigenvalues(self, q, normal):
        """(u.n - c, u.n (d times), u.n + c) (systems.py:158-171)."""
        un = self._normal_velocity(q, normal)
        c = self.sound_speed(q)
        out = _new(q, tuple(q.shape))
        out[..., 0] = un - c
        out[..., 1:-1] = un[..., None]
        out[..., -1] = un + c
        return out

    def cons_to_prim(self, q):
        """(rho, rho v, rho E) -> (rho, v, p) (systems.py:180-186)."""
        v = _new(q, tuple(q.shape))
        v[..., 0] = q[..., 0]
        v[..., 1:-1] = q[..., 1:-1] / q[..., 0:1]
        v[..., -1] = self.pressure(q)
        return v

    def prim_to_cons(self, v):
        """(rho, v, p) -> conserved, E = p / (gamma - 1) + rho |v|^2 / 2
        (systems.py:188-198)."""
        rho = v[..., 0]
        vv = v[..., 1] * v[..., 1]
        for j in range(1, self.dim):
            vv = vv + v[..., 1 + j] * v[..., 1 + j]
        q = _new(v, tuple(v.shape))
        q[..., 0] = rho
        q[..., 1:-1] = rho[..., None] * v[..., 1:-1]
        q[..., -1] = v[..., -1] / (self.gamma - 1.0) + 0.5 * rho * vv
        return q

    def primitive_rhs(self, v, grad):
        """Quasi-linear primitive form (systems.py:200-223):
        rho_t = -(v.grad rho + rho div v), v_t = -(v.grad v + grad p / rho),
        p_t = -(v.grad p + gamma p div v)."""
        d = self.dim
        rho, p = v[..., 0], v[..., -1]

        def along_v(k):   # sum_j v_j d_j (quantity k), j ascending
            acc = v[..., 1] * grad[..., 0, k]
            for j in range(1, d):
                acc = acc + v[..., 1 + j] * grad[..., j, k]
            return acc

        div = grad[..., 0, 1]
        for j in range(1, d):
            div = div + grad[..., j, 1 + j]
        out = _new(v, tuple(v.shape))
        out[..., 0] = -(along_v(0) + rho * div)
        for i in range(d):
            out[..., 1 + i] = -(along_v(1 + i) + grad[..., i, d + 1] / rho)
        out[..., -1] = -(along_v(d + 1) + self.gamma * p * div)
        return out

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

    def eigenvalues(self, q, normal):
        a_n = float(np.dot(self.velocity, normal))
        return np.full(tuple(q.shape[:-1]) + (1,), a_n)

    def primitive_rhs(self, v, grad):
        """-a . grad q (systems.py:104-108)."""
        out = np.zeros(tuple(v.shape))
        for j in range(self.dim):
            out[..., 0] -= self.velocity[j] * np.asarray(grad)[..., j, 0]
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

    def _kin(self, q):
        """alpha_eff = max(alpha, ALPHA_FLOOR) and the velocities (v_x, v_y)."""
        a = np.maximum(q[..., self.ALPHA], ALPHA_FLOOR)
        return a, q[..., self.AVX] / a, q[..., self.AVY] / a

    def ncp(self, q, grad):
        """B(q).grad q (systems.py:269-296): Hooke's law on the effective
        velocity gradient d v_i / d x_j = (d_j(alpha v_i) - v_i d_j alpha) /
        alpha, momentum from the divergence of alpha sigma plus the
        interface terms sigma . grad alpha."""
        S = self
        a, vx, vy = self._kin(q)
        lam, mu, rho = q[..., S.LAM], q[..., S.MU], q[..., S.RHO]
        g = [grad[..., 0, :], grad[..., 1, :]]
        vel = (vx, vy)
        av = (S.AVX, S.AVY)

        def dv(i, j):   # d v_i / d x_j
            return (g[j][..., av[i]] - vel[i] * g[j][..., S.ALPHA]) / a

        exx, eyy = dv(0, 0), dv(1, 1)
        out = np.zeros(q.shape)
        out[..., S.SXX] = -(lam * (exx + eyy) + 2.0 * mu * exx)
        out[..., S.SYY] = -(lam * (exx + eyy) + 2.0 * mu * eyy)
        out[..., S.SXY] = -mu * (dv(0, 1) + dv(1, 0))
        # traction rows: (sxx, sxy) for the x momentum, (sxy, syy) for y
        for comp, (r0, r1) in ((S.AVX, (S.SXX, S.SXY)), (S.AVY, (S.SXY, S.SYY))):
            out[..., comp] = -(a * (g[0][..., r0] + g[1][..., r1])
                               + q[..., r0] * g[0][..., S.ALPHA]
                               + q[..., r1] * g[1][..., S.ALPHA]) / rho
        return out

    def ncp_matrix(self, q, normal):
        """B(q).n (systems.py:298-318), the matrix whose product with a jump
        the path-conservative faces integrate."""
        S = self
        nx, ny = float(normal[0]), float(normal[1])
        a, vx, vy = self._kin(q)
        lam, mu, rho = q[..., S.LAM], q[..., S.MU], q[..., S.RHO]
        lp2m = lam + 2.0 * mu
        b = np.zeros(q.shape[:-1] + (9, 9))
        entries = {
            (S.SXX, S.AVX): -lp2m * nx / a, (S.SXX, S.AVY): -lam * ny / a,
            (S.SXX, S.ALPHA): (lp2m * vx * nx + lam * vy * ny) / a,
            (S.SYY, S.AVX): -lam * nx / a, (S.SYY, S.AVY): -lp2m * ny / a,
            (S.SYY, S.ALPHA): (lam * vx * nx + lp2m * vy * ny) / a,
            (S.SXY, S.AVX): -mu * ny / a, (S.SXY, S.AVY): -mu * nx / a,
            (S.SXY, S.ALPHA): mu * (vx * ny + vy * nx) / a,
            (S.AVX, S.SXX): -a * nx / rho, (S.AVX, S.SXY): -a * ny / rho,
            (S.AVX, S.ALPHA): -(q[..., S.SXX] * nx + q[..., S.SXY] * ny) / rho,
            (S.AVY, S.SXY): -a * nx / rho, (S.AVY, S.SYY): -a * ny / rho,
            (S.AVY, S.ALPHA): -(q[..., S.SXY] * nx + q[..., S.SYY] * ny) / rho,
        }
        for (r, c), val in entries.items():
            b[..., r, c] = val
        return b

    def primitive_rhs(self, v, grad):
        return -self.ncp(v, grad)

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
