"""Oracle: 1-D Gauss-Legendre nodal tables and ADER time operators.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates reference `pkg/src/aderdg/basis.py` (tables) and
`pkg/src/aderdg/predictor.py:21-47` (TimeOperators).
"""

import numpy as np

MAX_DEGREE = 9  # basis.py:11


def _legendre_pair(n, x):
    """(P_n(x), P_{n-1}(x)) by the three-term recurrence."""
    p_nm1 = np.zeros_like(x)
    p_n = np.ones_like(x)
    for k in range(1, n + 1):
        p_nm1, p_n = p_n, ((2 * k - 1) * x * p_n - (k - 1) * p_nm1) / k
    return p_n, p_nm1


def gauss_legendre(n):
    """n-point Gauss-Legendre rule on [0, 1]; follows basis.py:16-52.

    Newton on P_n from Chebyshev-like seeds cos(pi (k + 3/4) / (n + 1/2)),
    iterated until the update falls below 1e-15, then mapped to [0, 1]
    in ascending order with weights halved.
    """
    if n < 1:
        raise ValueError("need at least one quadrature node")
    x = np.cos(np.pi * (np.arange(n) + 0.75) / (n + 0.5))
    for _ in range(100):
        p, pm = _legendre_pair(n, x)
        dp = n * (x * p - pm) / (x * x - 1.0)
        step = p / dp
        x = x - step
        if np.max(np.abs(step)) < 1e-15:
            break
    p, pm = _legendre_pair(n, x)
    dp = n * (x * p - pm) / (x * x - 1.0)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    return (np.ascontiguousarray(0.5 * (1.0 + x[::-1])),
            np.ascontiguousarray(0.5 * w[::-1]))


def cardinal_values(nodes, pts):
    """L[j, k] = ell_k(pts[j]) (basis.py:55-74)."""
    nodes = np.asarray(nodes, float)
    pts = np.atleast_1d(np.asarray(pts, float))
    out = np.ones((pts.size, nodes.size))
    for k in range(nodes.size):
        for j in range(nodes.size):
            if j != k:
                out[:, k] *= (pts - nodes[j]) / (nodes[k] - nodes[j])
    return out


def cardinal_derivatives(nodes, pts):
    """L'[j, k] = ell_k'(pts[j]) by the product rule (basis.py:77-100)."""
    nodes = np.asarray(nodes, float)
    pts = np.atleast_1d(np.asarray(pts, float))
    p = nodes.size
    out = np.zeros((pts.size, p))
    for k in range(p):
        denom = 1.0
        for j in range(p):
            if j != k:
                denom *= nodes[k] - nodes[j]
        for i in range(p):
            if i == k:
                continue
            term = np.ones(pts.size)
            for j in range(p):
                if j != k and j != i:
                    term *= pts - nodes[j]
            out[:, k] += term / denom
    return out


def _recovery(proj, w):
    """Mean-preserving least-squares left inverse of the subcell projection
    (basis.py:135-163): minimise ||proj R ubar - ubar|| subject to
    w . (R ubar) = mean(ubar).  Same constraint elimination on the pivot of
    the largest weight, then a least-squares solve."""
    n_sub, p = proj.shape
    mean_row = np.full(n_sub, 1.0 / n_sub)
    piv = int(np.argmax(w))
    free = [k for k in range(p) if k != piv]
    if not free:
        return mean_row.reshape(1, n_sub).copy()
    basis = np.zeros((p, p - 1))
    for c, k in enumerate(free):
        basis[k, c] = 1.0
        basis[piv, c] = -w[k] / w[piv]
    lhs = proj @ basis
    rhs = np.eye(n_sub) - np.outer(proj[:, piv], mean_row) / w[piv]
    z = np.linalg.lstsq(lhs, rhs, rcond=None)[0]
    rec = basis @ z
    rec[piv, :] += mean_row / w[piv]
    return rec


class OracleTables:
    """Per-degree constants (basis.py:166-195 and predictor.py:21-41)."""

    def __init__(self, degree):
        if not 0 <= degree <= MAX_DEGREE:
            raise ValueError(f"degree must be in 0..{MAX_DEGREE}")
        self.degree = degree
        p = degree + 1
        self.nodes, self.weights = gauss_legendre(p)
        self.diff = cardinal_derivatives(self.nodes, self.nodes)
        self.left_vals = cardinal_values(self.nodes, [0.0])[0]
        self.right_vals = cardinal_values(self.nodes, [1.0])[0]
        n_sub = 2 * degree + 1
        self.n_subcells = n_sub
        proj = np.empty((n_sub, p))
        for s in range(n_sub):
            proj[s] = self.weights @ cardinal_values(
                self.nodes, (s + self.nodes) / n_sub)
        self.sub_project = proj
        self.sub_recover = _recovery(proj, self.weights)
        # time operators (predictor.py:21-41)
        w = self.weights
        self.k1 = np.outer(self.right_vals, self.right_vals) - self.diff.T * w[None, :]
        self.k1_inv = np.linalg.inv(self.k1)
        self.g0 = self.k1_inv @ self.left_vals
        self.gw = self.k1_inv * w[None, :]
        self.k1_opnorm = float(np.linalg.norm(self.k1, 2))


_cache = {}


def oracle_tables(degree):
    if degree not in _cache:
        _cache[degree] = OracleTables(degree)
    return _cache[degree]


def time_operators(degree):
    return oracle_tables(degree)


def weight_tensor(w, dim):
    """((w_i w_j) w_k) outer products (corrector.py:132-138)."""
    out = w
    for _ in range(dim - 1):
        out = np.multiply.outer(out, w)
    return out
