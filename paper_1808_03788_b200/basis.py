"""Per-degree nodal tables, computed on the host and uploaded once.

Same contents as the reference's `BasisTables` (basis.py:166-202) and
`TimeOperators` (predictor.py:21-47), derived independently:

* Gauss-Legendre nodes from the Golub-Welsch Jacobi eigenproblem, polished
  by Newton on P_n; weights from 2 / ((1 - x^2) P_n'(x)^2).
* derivative matrix from barycentric weights (ell_k'(x_j) = (b_k/b_j) /
  (x_j - x_k), diagonal = minus the row sum).
* subcell projection by exact Gauss quadrature of the cardinal functions
  over the 2N+1 equal subcells; recovery as the mean-constrained least
  squares left inverse, solved through its KKT system.

`tests/test_host.py::test_product_tables_match_reference` pins all of them
against the reference's tables to 1e-13 (golden vectors from
`tests/golden/make_golden.py`).
"""

import numpy as np

MAX_DEGREE = 9


def _legendre(n, x):
    p0 = np.ones_like(x)
    if n == 0:
        return p0, np.zeros_like(x)
    p1 = x.copy()
    for k in range(2, n + 1):
        p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
    return p1, p0


def gauss_legendre(n):
    """n-point rule on [0, 1], ascending nodes, weights summing to one."""
    if n < 1:
        raise ValueError("need at least one quadrature node")
    if n == 1:
        return np.array([0.5]), np.array([1.0])
    k = np.arange(1, n)
    beta = k / np.sqrt(4.0 * k * k - 1.0)
    x = np.linalg.eigvalsh(np.diag(beta, 1) + np.diag(beta, -1))
    for _ in range(8):  # Newton polish of the eigenvalues
        p, pm = _legendre(n, x)
        dp = n * (x * p - pm) / (x * x - 1.0)
        x = x - p / dp
    p, pm = _legendre(n, x)
    dp = n * (x * p - pm) / (x * x - 1.0)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    order = np.argsort(x)
    return 0.5 * (1.0 + x[order]), 0.5 * w[order]


def lagrange_values(nodes, pts):
    """V[j, k] = ell_k(pts[j])."""
    nodes = np.asarray(nodes, float)
    pts = np.atleast_1d(np.asarray(pts, float))
    out = np.empty((pts.size, nodes.size))
    for k in range(nodes.size):
        others = np.delete(nodes, k)
        out[:, k] = np.prod((pts[:, None] - others[None, :]) / (nodes[k] - others[None, :]),
                            axis=1)
    return out


def derivative_matrix(nodes):
    """D[j, k] = ell_k'(x_j) via barycentric weights."""
    x = np.asarray(nodes, float)
    p = x.size
    if p == 1:
        return np.zeros((1, 1))
    b = np.array([1.0 / np.prod(x[k] - np.delete(x, k)) for k in range(p)])
    dmat = np.zeros((p, p))
    for j in range(p):
        for k in range(p):
            if j != k:
                dmat[j, k] = (b[k] / b[j]) / (x[j] - x[k])
        dmat[j, j] = -np.sum(dmat[j, np.arange(p) != j])
    return dmat


def subcell_projection(nodes, weights):
    p = len(nodes)
    s = 2 * p - 1
    return np.stack([weights @ lagrange_values(nodes, (r + np.asarray(nodes)) / s)
                     for r in range(s)])


def subcell_recovery(proj, weights):
    """argmin ||proj x - b|| s.t. weights . x = mean(b), for every b = e_r."""
    s, p = proj.shape
    kkt = np.zeros((p + 1, p + 1))
    kkt[:p, :p] = 2.0 * proj.T @ proj
    kkt[:p, p] = weights
    kkt[p, :p] = weights
    rhs = np.zeros((p + 1, s))
    rhs[:p, :] = 2.0 * proj.T
    rhs[p, :] = 1.0 / s
    return np.linalg.solve(kkt, rhs)[:p, :]


class BasisTables:
    """Immutable per-degree tables (reference attribute names)."""

    def __init__(self, degree):
        if not 0 <= degree <= MAX_DEGREE:
            raise ValueError(f"degree must be in 0..{MAX_DEGREE}, got {degree}")
        self.degree = degree
        self.nodes, self.weights = gauss_legendre(degree + 1)
        self.diff = derivative_matrix(self.nodes)
        self.left_vals = lagrange_values(self.nodes, [0.0])[0]
        self.right_vals = lagrange_values(self.nodes, [1.0])[0]
        self.sub_project = subcell_projection(self.nodes, self.weights)
        self.sub_recover = subcell_recovery(self.sub_project, self.weights)
        self.n_subcells = 2 * degree + 1
        w = self.weights
        self.k1 = np.outer(self.right_vals, self.right_vals) - self.diff.T * w[None, :]
        self.k1_inv = np.linalg.inv(self.k1)
        self.g0 = self.k1_inv @ self.left_vals
        self.gw = self.k1_inv * w[None, :]
        self.k1_opnorm = float(np.linalg.svd(self.k1, compute_uv=False)[0])
        for a in (self.nodes, self.weights, self.diff, self.left_vals, self.right_vals,
                  self.sub_project, self.sub_recover, self.k1, self.k1_inv, self.g0, self.gw):
            a.flags.writeable = False

    def device_blob(self):
        """Flat fp64 blob in the adg_set_tables layout (include/aderdg_b200.h)."""
        return np.ascontiguousarray(np.concatenate([
            self.nodes, self.weights, self.diff.ravel(), self.left_vals, self.right_vals,
            self.gw.ravel(), self.g0, [self.k1_opnorm], self.sub_project.ravel(),
            self.sub_recover.ravel()]), dtype=np.float64)

    def __repr__(self):
        return f"BasisTables(degree={self.degree})"


_cache = {}


def basis_tables(degree):
    if degree not in _cache:
        _cache[degree] = BasisTables(degree)
    return _cache[degree]


def weight_tensor(weights, dim):
    out = weights
    for _ in range(dim - 1):
        out = np.multiply.outer(out, weights)
    return out
