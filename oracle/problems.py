"""Oracle: initial conditions of the BASELINE configs.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

`vortex` restates reference `pkg/src/aderdg/problems.py:14-51`.  The 3-D
density wave (C2/C3/C5) and the 2-D circular explosion (C4) are not in the
reference registry; they are the closed-form states BASELINE.json writes
down, passed to `project_initial_condition` as callables.
`sod` and `blast` restate problems.py:96-132 (limiter / wall coverage).
"""

import numpy as np


def vortex(gamma=1.4, beta=5.0, center=(5.0, 5.0), size=(10.0, 10.0)):
    cx, cy = center
    sx, sy = size

    def state(dx, dy):
        r2 = dx * dx + dy * dy
        env = np.exp(0.5 * (1.0 - r2))
        du = -beta / (2.0 * np.pi) * env * dy
        dv = beta / (2.0 * np.pi) * env * dx
        temp = 1.0 - (gamma - 1.0) * beta * beta / (8.0 * gamma * np.pi * np.pi) \
            * np.exp(1.0 - r2)
        rho = temp ** (1.0 / (gamma - 1.0))
        p = temp ** (gamma / (gamma - 1.0))
        u = 1.0 + du
        v = 1.0 + dv
        e = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)
        return np.stack([rho, rho * u, rho * v, e], axis=-1)

    def exact(x, t):
        dx = x[..., 0] - cx - t
        dy = x[..., 1] - cy - t
        dx -= sx * np.round(dx / sx)
        dy -= sy * np.round(dy / sy)
        return state(dx, dy)

    return (lambda x: exact(x, 0.0)), exact


def density_wave(gamma=1.4, amp=0.2, vel=(1.0, 1.0, 1.0), p0=1.0):
    """rho = 1 + amp sin(2 pi sum x), u = vel, p = p0 (BASELINE C2)."""
    vel = tuple(float(v) for v in vel)

    def exact(x, t):
        d = x.shape[-1]
        phase = np.zeros(x.shape[:-1])
        for j in range(d):
            phase = phase + (x[..., j] - vel[j] * t)
        rho = 1.0 + amp * np.sin(2.0 * np.pi * phase)
        out = np.empty(x.shape[:-1] + (d + 2,))
        out[..., 0] = rho
        kin = np.zeros_like(rho)
        for j in range(d):
            out[..., 1 + j] = rho * vel[j]
            kin = kin + vel[j] * vel[j]
        out[..., -1] = p0 / (gamma - 1.0) + 0.5 * rho * kin
        return out

    return (lambda x: exact(x, 0.0)), exact


def explosion(gamma=1.4, radius=0.5):
    """Circular explosion (BASELINE C4): r<0.5 -> (1,0,0,1) else (0.125,0,0,0.1)."""

    def ic(x):
        r2 = x[..., 0] ** 2 + x[..., 1] ** 2
        inside = r2 < radius * radius
        rho = np.where(inside, 1.0, 0.125)
        p = np.where(inside, 1.0, 0.1)
        z = np.zeros_like(rho)
        return np.stack([rho, z, z, p / (gamma - 1.0)], axis=-1)

    return ic, None


def sod(gamma=1.4, split=0.5):
    def ic(x):
        xx = x[..., 0]
        rho = np.where(xx < split, 1.0, 0.125)
        p = np.where(xx < split, 1.0, 0.1)
        return np.stack([rho, np.zeros_like(rho), p / (gamma - 1.0)], axis=-1)

    return ic, None


def blast(gamma=1.4, r0=0.1, e0=1.0, p_ambient=1e-14):
    p_in = (gamma - 1.0) * e0 / (np.pi * r0 * r0)

    def ic(x):
        r2 = x[..., 0] ** 2 + x[..., 1] ** 2
        p = np.where(r2 <= r0 * r0, p_in, p_ambient)
        z = np.zeros_like(p)
        return np.stack([np.ones_like(p), z, z, p / (gamma - 1.0)], axis=-1)

    return ic, None
