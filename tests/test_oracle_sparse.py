"""Pins of the oracle's Smolyak sparse grids (Sec. 4.2 "Sparse grids"; construction
per SPEC S:128 and DESIGN.md reading R27: combination technique over nested Chebyshev /
Clenshaw-Curtis levels, level 0 = {0}, level j = the 2^j + 1 Chebyshev points).

What fixes them independently of the code:
* node counts of Clenshaw-Curtis sparse grids (textbook values, e.g. D = 2: 5, 13, 29, 65;
  the paper's "Full grid vs sparse grid" figure, contrasts 25 with 13 in 2-D);
* D = 1 collapses to the full 1-D grid: the basis equals the barycentric basis on
  2^q + 1 Chebyshev nodes (oracle.basis, pinned in test_oracle_interp.py);
* nested nodes make the combination technique interpolatory: Phi_h(n_h') = delta_hh';
* polynomial exactness on the Smolyak space sum_{|j| = q} P_{m(j_1)-1} x ... x P_{m(j_D)-1}, and a
  monomial outside it (x^3 y at D = 2, q = 2) is NOT reproduced -- so the grid is really sparse;
* the whole F^3M with a sparse grid: D = 1 equals the tensor-grid run with P = 2^q + 1, and the
  error against the exact sum decreases as the level grows (no dropped pairs).
"""
import itertools

import numpy as np
import pytest

import datagen
import oracle


def s1(q):
    return np.cos(np.arange(2 ** q + 1) * np.pi / 2 ** q)


@pytest.mark.parametrize("D,q,n", [(2, 1, 5), (2, 2, 13), (2, 3, 29), (2, 4, 65), (3, 1, 7), (3, 2, 25), (3, 3, 69),
                                   (5, 2, 61), (7, 2, 113), (7, 3, 589)])
def test_node_counts(D, q, n):
    assert oracle.sparse_nodes(D, q).shape == (n, D)


@pytest.mark.parametrize("q", [1, 2, 3, 4])
def test_one_dimension_is_the_full_grid(q):
    nodes = oracle.sparse_nodes(1, q)[:, 0]
    np.testing.assert_array_equal(nodes, np.arange(2 ** q + 1))
    for t in np.linspace(-1, 1, 13):
        np.testing.assert_allclose(oracle.sparse_basis(1, q, [t]), oracle.basis(2 ** q + 1, t), atol=1e-14)


@pytest.mark.parametrize("D,q", [(2, 2), (3, 2), (3, 3), (5, 2)])
def test_interpolatory_and_partition_of_unity(D, q):
    H = oracle.sparse_nodes(D, q)
    x = s1(q)[H]  # node coordinates
    for i in range(0, len(H), max(1, len(H) // 17)):
        phi = oracle.sparse_basis(D, q, x[i])
        e = np.zeros(len(H))
        e[i] = 1.0
        np.testing.assert_allclose(phi, e, atol=1e-12)
    rng = np.random.default_rng(D * 10 + q)
    for _ in range(10):
        assert abs(oracle.sparse_basis(D, q, rng.uniform(-1, 1, D)).sum() - 1.0) < 1e-12


def smolyak_degrees(D, q):
    """Maximal per-dimension degrees of the Smolyak space of level q (terms |j| = q)."""
    m1 = lambda j: 0 if j == 0 else 2 ** j  # noqa: E731  (degree m(j) - 1)
    return [tuple(m1(j) for j in js) for js in itertools.product(range(q + 1), repeat=D) if sum(js) == q]


@pytest.mark.parametrize("D,q", [(2, 2), (2, 3), (3, 2), (4, 2)])
def test_polynomial_exactness_on_the_smolyak_space(D, q):
    H = oracle.sparse_nodes(D, q)
    xn = s1(q)[H]
    rng = np.random.default_rng(7)
    pts = rng.uniform(-1, 1, (8, D))
    for deg in smolyak_degrees(D, q):
        f = lambda x: np.prod([x[..., d] ** deg[d] for d in range(D)], axis=0)  # noqa: E731
        vals = f(xn)
        for x in pts:
            assert abs(oracle.sparse_basis(D, q, x) @ vals - f(x)) < 1e-12, deg


def test_not_a_full_tensor_grid():
    # D = 2, q = 2: x^3 y is outside the Smolyak space (no term has degrees >= (3, 1))
    H = oracle.sparse_nodes(2, 2)
    xn = s1(2)[H]
    vals = xn[:, 0] ** 3 * xn[:, 1]
    x = np.array([0.37, -0.61])
    assert abs(oracle.sparse_basis(2, 2, x) @ vals - x[0] ** 3 * x[1]) > 1e-3


def test_f3m_sparse_d1_equals_tensor_grid():
    X = datagen.points("uniform", 4000, 1, seed=0)
    b = datagen.weights(4000, seed=1)
    g = datagen.gamma_for_ev("uniform", 1, 1.0)
    for q in (2, 3):
        rs = oracle.f3m(X, b, g, P=4, sparse_level=q)
        rt = oracle.f3m(X, b, g, P=2 ** q + 1)
        np.testing.assert_allclose(rs.v, rt.v, rtol=0, atol=1e-10 * np.max(np.abs(rt.v)))


def test_f3m_sparse_converges_with_the_level():
    X = datagen.points("uniform", 3000, 3, seed=2)
    b = datagen.weights(3000, seed=3)
    g = datagen.gamma_for_ev("uniform", 3, 1.0)
    ve = oracle.direct(X, b, g)
    errs = []
    for q in (1, 2, 3):
        r = oracle.f3m(X, b, g, P=4, sparse_level=q, flags=oracle.NO_DROP, zeta=1, rho=1, node_cap=4096)
        errs.append(oracle.subset_error(r.v, ve)[0])
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 1e-5
    # linearity (the tree does not depend on b)
    b2 = datagen.weights(3000, seed=4)
    r1 = oracle.f3m(X, b, g, sparse_level=2)
    r2 = oracle.f3m(X, b2, g, sparse_level=2)
    r3 = oracle.f3m(X, 2 * b.double() - b2.double(), g, sparse_level=2)
    np.testing.assert_allclose(r3.v, 2 * r1.v - r2.v, atol=1e-10 * np.max(np.abs(r3.v)))
