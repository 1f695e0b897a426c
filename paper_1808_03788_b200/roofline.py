"""Algorithmic work model of one Euler ADER-DG step.

Counts 1 add / mul / div / sqrt = 1 flop (an FMA = 2).  Per element:

    Ff = d^2 + 5d + 5 (pointwise flux), Ef = 4d + 8 (eigenvalue)
    startup (N >= 2) = 2 (Ff P^d + 2dm P^(d+1) + dm P^d) + 2m P^d + 5m P^(d+1)
    sweep            = Ff P^(d+1) + 2(d+1) m P^(d+2) + (d+8) m P^(d+1)
    volume           = Ff P^(d+1) + 4dm P^(d+1) + 3dm P^d
    traces           = 4dm P^(d+1)
    faces            = d P^d (2Ff + 2Ef + 7m)
    face integral    = 8dm P^d;  update = (2d+2) m P^d;  dt scan = P^d (2d+4+d Ef)

Compulsory HBM bytes per element-step: 8 m P^d (2 + 4d) -- u^n read,
u^(n+1) written, the 2d space-time face traces written once and read once.
"""


def _parts(degree, dim):
    P = degree + 1
    d = dim
    m = d + 2
    Ff = d * d + 5 * d + 5
    Ef = 4 * d + 8
    rate_s = Ff * P ** d + 2 * d * m * P ** (d + 1) + d * m * P ** d
    if degree >= 2:
        startup = 2 * rate_s + 2 * m * P ** d + 5 * m * P ** (d + 1)
    else:
        startup = rate_s + 2 * m * P ** (d + 1)
    sweep = Ff * P ** (d + 1) + 2 * (d + 1) * m * P ** (d + 2) + (d + 8) * m * P ** (d + 1)
    volume = Ff * P ** (d + 1) + 4 * d * m * P ** (d + 1) + 3 * d * m * P ** d
    traces = 4 * d * m * P ** (d + 1)
    faces = d * P ** d * (2 * Ff + 2 * Ef + 7 * m)
    rest = 8 * d * m * P ** d + (2 * d + 2) * m * P ** d + P ** d * (2 * d + 4 + d * Ef)
    return dict(P=P, m=m, startup=startup, sweep=sweep, volume=volume, traces=traces,
                faces=faces, rest=rest)


def predictor_flops(degree, dim, sweeps_total, n_elem):
    """Algorithmic flops of one adg_predict launch: startup + executed sweeps
    + volume integral + traces over n_elem elements."""
    p = _parts(degree, dim)
    return n_elem * (p["startup"] + p["volume"] + p["traces"]) + sweeps_total * p["sweep"]


def step_flops_per_dof(degree, dim, sweeps):
    p = _parts(degree, dim)
    fl = (p["startup"] + sweeps * p["sweep"] + p["volume"] + p["traces"] + p["faces"]
          + p["rest"])
    return fl / p["P"] ** dim


def step_bytes_per_dof(degree, dim):
    m = dim + 2
    return 8 * m * (2 + 4 * dim)


def roofline_dofs(degree, dim, sweeps, fp64_flops, hbm_bytes):
    return min(fp64_flops / step_flops_per_dof(degree, dim, sweeps),
               hbm_bytes / step_bytes_per_dof(degree, dim))
