"""Oracle: ideal-gas compressible Euler pointwise physics.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates reference `pkg/src/aderdg/systems.py:112-234` (CompressibleEuler)
with the same per-quantity operation order, so batched evaluation equals
a per-point loop lane for lane.
"""

import numpy as np


class EulerOracle:
    name = "euler"

    def __init__(self, dim, gamma=1.4):
        self.dim = int(dim)
        self.n_vars = self.dim + 2
        self.gamma = float(gamma)

    # systems.py:128-133
    def pressure(self, q):
        d = self.dim
        kin = q[..., 1] * q[..., 1]
        for j in range(1, d):
            kin = kin + q[..., 1 + j] * q[..., 1 + j]
        return (self.gamma - 1.0) * (q[..., -1] - 0.5 * kin / q[..., 0])

    # systems.py:135-138
    def sound_speed(self, q):
        with np.errstate(invalid="ignore", divide="ignore"):
            return np.sqrt(self.gamma * self.pressure(q) / q[..., 0])

    # systems.py:140-156: F[..., j, v]
    def flux(self, q):
        d = self.dim
        r = 1.0 / q[..., 0]
        kin = q[..., 1] * q[..., 1]
        for j in range(1, d):
            kin = kin + q[..., 1 + j] * q[..., 1 + j]
        p = (self.gamma - 1.0) * (q[..., -1] - 0.5 * kin * r)
        ep = q[..., d + 1] + p
        f = np.empty(q.shape[:-1] + (d, d + 2))
        for j in range(d):
            vel = q[..., 1 + j] * r
            f[..., j, 0] = q[..., 1 + j]
            for i in range(d):
                f[..., j, 1 + i] = q[..., 1 + i] * vel
            f[..., j, 1 + j] += p
            f[..., j, d + 1] = ep * vel
        return f

    # systems.py:173-178 for a unit axis normal e_axis
    def max_abs_eigenvalue_axis(self, q, axis):
        un = np.zeros_like(q[..., 0])
        for j in range(self.dim):
            un = un + q[..., 1 + j] * (1.0 if j == axis else 0.0)
        return np.abs(un / q[..., 0]) + self.sound_speed(q)

    # systems.py:225-229
    def admissible(self, q):
        finite = np.all(np.isfinite(q), axis=-1)
        with np.errstate(invalid="ignore", divide="ignore"):
            pos = (q[..., 0] > 0.0) & (self.pressure(q) > 0.0)
        return finite & pos

    # systems.py:231-234
    def reflect(self, q, axis):
        out = q.copy()
        out[..., 1 + axis] = -q[..., 1 + axis]
        return out

    # systems.py:180-198
    def cons_to_prim(self, q):
        v = np.empty_like(q)
        v[..., 0] = q[..., 0]
        for j in range(self.dim):
            v[..., 1 + j] = q[..., 1 + j] / q[..., 0]
        v[..., -1] = self.pressure(q)
        return v

    def prim_to_cons(self, v):
        q = np.empty_like(v)
        rho = v[..., 0]
        q[..., 0] = rho
        kin = v[..., 1] * v[..., 1]
        for j in range(1, self.dim):
            kin = kin + v[..., 1 + j] * v[..., 1 + j]
        for j in range(self.dim):
            q[..., 1 + j] = rho * v[..., 1 + j]
        q[..., -1] = v[..., -1] / (self.gamma - 1.0) + 0.5 * rho * kin
        return q

    # systems.py:200-223: quasi-linear primitive time derivative
    def primitive_rhs(self, v, grad):
        d = self.dim
        rho = v[..., 0]
        p = v[..., -1]
        div = grad[..., 0, 1]
        for j in range(1, d):
            div = div + grad[..., j, 1 + j]
        out = np.empty_like(v)
        arho = v[..., 1] * grad[..., 0, 0]
        ap = v[..., 1] * grad[..., 0, d + 1]
        for j in range(1, d):
            arho = arho + v[..., 1 + j] * grad[..., j, 0]
            ap = ap + v[..., 1 + j] * grad[..., j, d + 1]
        out[..., 0] = -(arho + rho * div)
        for i in range(d):
            av = v[..., 1] * grad[..., 0, 1 + i]
            for j in range(1, d):
                av = av + v[..., 1 + j] * grad[..., j, 1 + i]
            out[..., 1 + i] = -(av + grad[..., i, d + 1] / rho)
        out[..., d + 1] = -(ap + self.gamma * p * div)
        return out

