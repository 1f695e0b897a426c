"""Initial conditions of the benchmark configurations (setup, host side).

`build_problem(name, system, **params)` mirrors the reference registry
(problems.py:208-242) for the Euler cases and adds the two BASELINE
initial states the reference lacks: the 3-D smooth
density wave (C2/C3/C5) and the 2-D circular explosion (C4).  Each builder
returns (ic, exact): ic(points) -> states, exact(points, t) or None.
"""

import numpy as np


def _xp(a):
    """numpy, or torch for a torch tensor: the closed-form exact solutions
    below evaluate on either, so `Simulation` can form "exact" boundary data
    on the device (their `device_capable` attribute says so); t may then be
    a one-element device tensor."""
    if type(a).__module__.split(".")[0] == "torch":
        import torch
        return torch
    return np


def _device_capable(fn):
    fn.device_capable = True
    return fn


def isentropic_vortex(system, beta=5.0, center=(5.0, 5.0), domain_size=(10.0, 10.0)):
    """problems.py:14-51 (C1)."""
    if system.name != "euler" or system.dim != 2:
        raise ValueError("the vortex case needs 2-D Euler")
    g = system.gamma
    cx, cy = (float(c) for c in center)
    lx, ly = (float(s) for s in domain_size)
    amp = float(beta) / (2.0 * np.pi)
    b = float(beta)
    tcoef = (g - 1.0) * b * b / (8.0 * g * np.pi * np.pi)

    @_device_capable
    def exact(points, t):
        xp = _xp(points)
        rx = points[..., 0] - cx - t
        ry = points[..., 1] - cy - t
        rx = rx - lx * xp.round(rx / lx)
        ry = ry - ly * xp.round(ry / ly)
        r2 = rx * rx + ry * ry
        bump = xp.exp(0.5 * (1.0 - r2))
        vx = 1.0 + (-amp * bump * ry)
        vy = 1.0 + amp * bump * rx
        temp = 1.0 - tcoef * xp.exp(1.0 - r2)
        rho = temp ** (1.0 / (g - 1.0))
        p = temp ** (g / (g - 1.0))
        energy = p / (g - 1.0) + 0.5 * rho * (vx * vx + vy * vy)
        return xp.stack([rho, rho * vx, rho * vy, energy], -1)

    return (lambda points: exact(points, 0.0)), exact


def density_wave(system, amplitude=0.2, velocity=None, pressure=1.0):
    """rho = 1 + a sin(2 pi sum_j x_j), v = velocity (default all ones),
    p = pressure; exact solution is translation (BASELINE C2/C3/C5)."""
    if system.name != "euler":
        raise ValueError("the density wave needs Euler")
    d = system.dim
    g = system.gamma
    vel = np.ones(d) if velocity is None else np.asarray(velocity, float)

    @_device_capable
    def exact(points, t):
        xp = _xp(points)
        arg = xp.zeros_like(points[..., 0])
        for j in range(d):
            arg = arg + (points[..., j] - float(vel[j]) * t)
        rho = 1.0 + amplitude * xp.sin(2.0 * np.pi * arg)
        cols = [rho]
        v2 = 0.0
        for j in range(d):
            cols.append(rho * float(vel[j]))
            v2 = v2 + float(vel[j]) * float(vel[j])
        cols.append(pressure / (g - 1.0) + 0.5 * rho * v2)
        return xp.stack(cols, -1)

    return (lambda points: exact(points, 0.0)), exact


def circular_explosion(system, radius=0.5, inner=(1.0, 1.0), outer=(0.125, 0.1)):
    """(rho, p) = inner for r < radius else outer, at rest (BASELINE C4)."""
    if system.name != "euler" or system.dim != 2:
        raise ValueError("the explosion case needs 2-D Euler")
    g = system.gamma

    def ic(points):
        inside = points[..., 0] ** 2 + points[..., 1] ** 2 < radius * radius
        rho = np.where(inside, inner[0], outer[0])
        p = np.where(inside, inner[1], outer[1])
        zero = np.zeros_like(rho)
        return np.stack([rho, zero, zero, p / (g - 1.0)], axis=-1)

    return ic, None


def sod_shock_tube(system, split=0.5):
    """problems.py:96-110."""
    if system.name != "euler" or system.dim != 1:
        raise ValueError("the shock tube needs 1-D Euler")
    g = system.gamma

    def ic(points):
        left = points[..., 0] < split
        rho = np.where(left, 1.0, 0.125)
        p = np.where(left, 1.0, 0.1)
        return np.stack([rho, np.zeros_like(rho), p / (g - 1.0)], axis=-1)

    return ic, None


def blast_2d(system, r0=0.1, e0=1.0, p_ambient=1e-14):
    """problems.py:113-132."""
    if system.name != "euler" or system.dim != 2:
        raise ValueError("the blast case needs 2-D Euler")
    g = system.gamma
    p_in = (g - 1.0) * e0 / (np.pi * r0 * r0)

    def ic(points):
        inside = points[..., 0] ** 2 + points[..., 1] ** 2 <= r0 * r0
        p = np.where(inside, p_in, p_ambient)
        zero = np.zeros_like(p)
        return np.stack([np.ones_like(p), zero, zero, p / (g - 1.0)], axis=-1)

    return ic, None


def advected_sine(system):
    """problems.py:54-66: sin(2 pi sum_j x_j) carried by the advection velocity."""
    if system.name != "advection":
        raise ValueError("the sine case needs the advection system")
    vel = system.velocity

    @_device_capable
    def exact(points, t):
        xp = _xp(points)
        phase = xp.zeros_like(points[..., 0])
        for j in range(system.dim):
            phase = phase + (points[..., j] - float(vel[j]) * t)
        return xp.sin(2.0 * np.pi * phase)[..., None]

    return (lambda points: exact(points, 0.0)), exact


def gaussian_pulse(system, center=0.25, width=0.08, amplitude=1.0):
    """problems.py:69-82: a Gaussian translated by the advection velocity."""
    if system.name != "advection":
        raise ValueError("the pulse case needs the advection system")
    vel = system.velocity

    @_device_capable
    def exact(points, t):
        xp = _xp(points)
        r2 = xp.zeros_like(points[..., 0])
        for j in range(system.dim):
            d = points[..., j] - center - float(vel[j]) * t
            r2 = r2 + d * d
        return (amplitude * xp.exp(-r2 / (2.0 * width * width)))[..., None]

    return (lambda points: exact(points, 0.0)), exact


def step_function(system, position=0.5, left=1.0, right=0.0):
    """problems.py:85-93: a discontinuous transport profile in x."""
    if system.name != "advection":
        raise ValueError("the step case needs the advection system")

    def ic(points):
        return np.where(points[..., 0] < position, left, right)[..., None]

    return ic, None


def constant_state(system, values=None):
    """problems.py:176-192."""
    if values is None:
        values = {"advection": [0.75],
                  "elasticity-di": [0.3, 0.2, 0.1, 0.05, -0.04, 0.7, 2.0, 1.0, 1.0]}.get(
                      system.name, [1.0] + [0.1] * system.dim + [2.5])
    q0 = np.asarray(values, float)
    if q0.shape != (system.n_vars,):
        raise ValueError(f"constant state needs {system.n_vars} entries")

    @_device_capable
    def exact(points, t):
        if _xp(points) is not np:
            import torch
            q = torch.as_tensor(q0, dtype=points.dtype, device=points.device)
            return q.expand(tuple(points.shape[:-1]) + tuple(q0.shape)).clone()
        return np.broadcast_to(q0, points.shape[:-1] + q0.shape).copy()

    return (lambda points: exact(points, 0.0)), exact


def elastic_pwave(system, alpha_min=1e-3, interface=0.7, pulse_center=0.3,
                  pulse_width=0.05, amplitude=1e-3, lam=2.0, mu=1.0, rho=1.0,
                  interface_width=0.05):
    """problems.py:135-173: a right-moving plane P-wave pulse in solid
    (alpha = 1) running toward a tanh ramp to alpha_min (the free surface)."""
    if system.name != "elasticity-di":
        raise ValueError("the P-wave case needs the diffuse-interface system")
    if interface_width <= 0.0:
        raise ValueError("interface_width must be positive")
    cp = np.sqrt((lam + 2.0 * mu) / rho)

    def exact(points, t):
        x = points[..., 0]
        vx = amplitude * np.exp(-((x - pulse_center - cp * t) / pulse_width) ** 2)
        sxx = -rho * cp * vx
        syy = lam / (lam + 2.0 * mu) * sxx
        ramp = 0.5 * (1.0 - np.tanh((x - interface) / interface_width))
        alpha = alpha_min + (1.0 - alpha_min) * ramp
        out = np.zeros(points.shape[:-1] + (9,))
        out[..., 0] = sxx
        out[..., 1] = syy
        out[..., 3] = alpha * vx
        out[..., 5] = alpha
        out[..., 6] = lam
        out[..., 7] = mu
        out[..., 8] = rho
        return out

    return (lambda points: exact(points, 0.0)), None


class ProblemSpec:
    def __init__(self, builder, dim, extents, boundary, suggested_tend, system="euler"):
        self.builder = builder
        self.system = system
        self.dim = dim
        self.extents = extents
        self.boundary = boundary
        self.suggested_tend = suggested_tend


PROBLEMS = {
    "vortex": ProblemSpec(isentropic_vortex, 2, ((0.0, 10.0), (0.0, 10.0)), "periodic", 10.0),
    "sod": ProblemSpec(sod_shock_tube, 1, ((0.0, 1.0),), "outflow", 0.2),
    "blast": ProblemSpec(blast_2d, 2, ((-1.0, 1.0), (-1.0, 1.0)), "wall", 0.05),
    "constant": ProblemSpec(constant_state, None, None, "periodic", 1.0, system=None),
    "sine": ProblemSpec(advected_sine, None, None, "periodic", 1.0, system="advection"),
    "pulse": ProblemSpec(gaussian_pulse, None, None, {0: ("exact", "outflow")}, 0.5,
                         system="advection"),
    "step": ProblemSpec(step_function, None, None, "periodic", 0.5, system="advection"),
    "pwave": ProblemSpec(elastic_pwave, 2, ((0.0, 1.0), (0.0, 0.25)), "outflow", 0.15,
                         system="elasticity-di"),
    "density_wave": ProblemSpec(density_wave, None, None, "periodic", 1.0),
    "explosion": ProblemSpec(circular_explosion, 2, ((-1.0, 1.0), (-1.0, 1.0)), "outflow",
                             0.25),
}


def build_problem(name, system, **params):
    try:
        spec = PROBLEMS[name]
    except KeyError:
        raise ValueError(f"unknown problem '{name}' (choose from {sorted(PROBLEMS)})")
    if spec.system is not None and system.name != spec.system:
        raise ValueError(f"problem '{name}' needs the {spec.system} system, got {system.name}")
    if spec.dim is not None and system.dim != spec.dim:
        raise ValueError(f"problem '{name}' is {spec.dim}-D")
    return spec.builder(system, **params)
