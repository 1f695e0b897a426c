"""Plugin-contract methods of the drop-in systems (reference systems.py:16-74,
:158-223, :269-318) against the reference's outputs on seeded states
(tests/golden/plugins.npz, make_golden.py gen_plugins).  Host formulas: the
kernels carry the same physics as compile-time policies."""

import numpy as np
import pytest

from paper_1808_03788_b200 import systems


@pytest.mark.parametrize("d", [1, 2, 3])
def test_euler_contract(golden, d):
    g = golden("plugins")
    e = systems.CompressibleEuler(d, gamma=1.4)
    q, grad, n = g[f"e{d}_q"], g[f"e{d}_grad"], g[f"e{d}_normal"]
    np.testing.assert_allclose(e.eigenvalues(q, n), g[f"e{d}_eig"], rtol=1e-15, atol=1e-15)
    v = e.cons_to_prim(q)
    np.testing.assert_array_equal(v, g[f"e{d}_prim"])
    np.testing.assert_allclose(e.prim_to_cons(v), g[f"e{d}_cons"], rtol=1e-15)
    np.testing.assert_allclose(e.primitive_rhs(v, grad), g[f"e{d}_prim_rhs"], rtol=1e-14,
                               atol=1e-14)
    np.testing.assert_allclose(e.max_abs_eigenvalue(q, n),
                               np.max(np.abs(g[f"e{d}_eig"]), axis=-1), rtol=1e-15)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_advection_contract(golden, d):
    g = golden("plugins")
    a = systems.LinearAdvection(d, velocity=g[f"a{d}_vel"])
    n = g[f"e{d}_normal"]
    np.testing.assert_array_equal(a.eigenvalues(g[f"a{d}_q"], n), g[f"a{d}_eig"])
    np.testing.assert_allclose(a.primitive_rhs(g[f"a{d}_q"], g[f"a{d}_grad"]),
                               g[f"a{d}_prim_rhs"], rtol=1e-15, atol=1e-16)


def test_elasticity_contract(golden):
    g = golden("plugins")
    el = systems.DiffuseInterfaceElasticity(2)
    q, grad, n = g["el_q"], g["el_grad"], g["el_normal"]
    np.testing.assert_allclose(el.ncp(q, grad), g["el_ncp"], rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(el.ncp_matrix(q, n), g["el_ncp_matrix"], rtol=1e-15,
                               atol=1e-15)
    np.testing.assert_allclose(el.primitive_rhs(q, grad), g["el_prim_rhs"], rtol=1e-14,
                               atol=1e-14)
    np.testing.assert_allclose(el.eigenvalues(q, n), g["el_eig"], rtol=1e-15)


def test_base_defaults(golden):
    g = golden("plugins")
    base = systems.HyperbolicSystem(2, 3, ("a", "b", "c"))
    q = g["el_q"][:4, :3]
    np.testing.assert_array_equal(base.flux(q), g["base_flux"])
    np.testing.assert_array_equal(base.ncp_matrix(q, g["el_normal"]), g["base_ncp_matrix"])
    np.testing.assert_array_equal(base.ncp(q, np.zeros((4, 2, 3))), np.zeros((4, 3)))
    np.testing.assert_array_equal(base.source(q), np.zeros_like(q))
    assert base.cons_to_prim(q) is q and base.prim_to_cons(q) is q
    with pytest.raises(NotImplementedError):
        base.primitive_rhs(q, None)
    with pytest.raises(NotImplementedError):
        base.eigenvalues(q, (1.0, 0.0))
