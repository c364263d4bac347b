"""Pins for the oracle's interpolation machinery (CPU only).

Each test checks the oracle against something the paper or mathematics fixes, never
against a retyped copy of the oracle's own formula:
closed forms (golden/paper_closed_forms.json), L_i(s_j) = delta_ij (App. C), the product
form of Sec. 3 (a different formula for the same polynomial), polynomial reproduction,
Prop. 1's order and App. B's variance bound.
"""
import itertools
import math

import numpy as np
import pytest

import oracle


@pytest.mark.parametrize("P", ["2", "3", "5"])
def test_cheb_nodes_closed_form(golden, P):
    # PAPER.md:141, App. C
    want = np.array(golden["cheb_nodes"][P])
    got = oracle.cheb_nodes(int(P))
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-15)
    assert np.all(np.diff(got) < 0)  # strictly decreasing, s_0 = 1, s_r = -1


@pytest.mark.parametrize("P", ["2", "3", "5"])
def test_bary_weights_closed_form(golden, P):
    # PAPER.md:652-656
    np.testing.assert_array_equal(oracle.bary_weights(int(P)), np.array(golden["bary_weights"][P]))


def _product_form(P, t):
    """Sec. 3 L_i(t) = prod_{j!=i}(t-s_j)/prod_{j!=i}(s_i-s_j), nodes cos(i pi/r)."""
    s = np.cos(np.arange(P) * math.pi / (P - 1))
    L = np.ones(P)
    for i in range(P):
        for j in range(P):
            if j != i:
                L[i] *= (t - s[j]) / (s[i] - s[j])
    return L


@pytest.mark.parametrize("P", [2, 3, 4, 5, 8, 12])
def test_basis_delta_at_nodes(P):
    # App. C PAPER.md:649 "when t = s_j, we set L_i(s_j) = delta_ij"
    for j, sj in enumerate(oracle.cheb_nodes(P)):
        np.testing.assert_array_equal(oracle.basis(P, sj), np.eye(P)[j])


@pytest.mark.parametrize("P", [2, 3, 4, 5, 8, 12, 16])
def test_barycentric_equals_product_form(P):
    rng = np.random.default_rng(P)
    for t in rng.uniform(-1, 1, 300):
        np.testing.assert_allclose(oracle.basis(P, t), _product_form(P, t), rtol=0, atol=1e-12)


@pytest.mark.parametrize("P", [2, 3, 4, 6, 9])
def test_partition_of_unity_and_polynomial_reproduction(P):
    rng = np.random.default_rng(100 + P)
    s = oracle.cheb_nodes(P)
    for deg in range(P):  # every polynomial of degree <= P-1 is reproduced
        c = rng.normal(size=deg + 1)
        f = lambda t: np.polyval(c, t)
        for t in rng.uniform(-1, 1, 50):
            L = oracle.basis(P, t)
            assert abs(L.sum() - 1.0) < 1e-13
            assert abs(L @ f(s) - f(t)) < 1e-12 * max(1.0, np.abs(c).sum())


def test_cubic_reproduction_spec_example():
    # r = 8 (P = 9), f = t^3 at 100 random t -> max abs error <= 1e-13
    rng = np.random.default_rng(7)
    s = oracle.cheb_nodes(9)
    err = max(abs(oracle.basis(9, t) @ s ** 3 - t ** 3) for t in rng.uniform(-1, 1, 100))
    assert err <= 1e-13


@pytest.mark.parametrize("D,P", [(1, 4), (2, 3), (3, 4), (4, 2), (3, 5)])
def test_tensor_basis_reproduces_multivariate_polynomials(D, P):
    # Sec. 3 PAPER.md:145 tensor basis; SPEC.md:157 per-dimension degree <= P-1 reproduced
    rng = np.random.default_rng(D * 10 + P)
    s = oracle.cheb_nodes(P)
    # node multi-index k = sum_d k_d P^d (dimension 1 fastest)
    nodes = np.array([[s[(k // P ** d) % P] for d in range(D)] for k in range(P ** D)])
    expo = [tuple(rng.integers(0, P, size=D)) for _ in range(4)]
    coef = rng.normal(size=len(expo))

    def f(x):
        return sum(c * np.prod([x[d] ** e[d] for d in range(D)]) for c, e in zip(coef, expo))

    fn = np.array([f(n) for n in nodes])
    for _ in range(30):
        tau = rng.uniform(-1, 1, D)
        Lk = oracle.tensor_basis(D, P, tau)
        assert abs(Lk.sum() - 1.0) < 1e-12
        assert abs(Lk @ fn - f(tau)) < 1e-11


def test_prop1_interpolation_order():
    """Prop. 1 (App. D): with d(x,y) <= eta and degree
    r = 2p (p = 2 -> P = 5 nodes), the bivariate interpolant's pointwise error is O(eta^{p+1}).
    SPEC.md:158/626: log-log slope over eta in {0.5, 0.25, 0.125} must be >= 2.5."""
    gamma, P = 1.0, 5
    s = oracle.cheb_nodes(P)
    errs = []
    etas = [0.5, 0.25, 0.125]
    for eta in etas:
        h = gamma * math.sqrt(2 * eta)  # one box [0,h]: d(x,y) <= h^2/(2 gamma^2) = eta
        nodes = h * (s + 1) / 2
        Kn = np.exp(-(nodes[:, None] - nodes[None, :]) ** 2 / (2 * gamma ** 2))
        grid = np.linspace(0, h, 41)
        Lg = np.array([oracle.basis(P, 2 * x / h - 1) for x in grid])
        approx = Lg @ Kn @ Lg.T
        exact = np.exp(-(grid[:, None] - grid[None, :]) ** 2 / (2 * gamma ** 2))
        errs.append(np.abs(approx - exact).max())
    slope = np.polyfit(np.log(etas), np.log(errs), 1)[0]
    assert slope >= 2.5, (errs, slope)


def test_appB_variance_bound():
    """App. B: Var(X) <= (M-m)^2/4 on [m, M]; SPEC.md:627 (10^4 trials)."""
    rng = np.random.default_rng(3)
    for _ in range(10000):
        m, M = np.sort(rng.normal(size=2) * 10)
        x = rng.uniform(m, M, size=rng.integers(2, 50))
        if rng.random() < 0.3:  # extreme two-point laws attain the bound
            x = np.where(rng.random(x.size) < 0.5, m, M)
        assert x.var() <= (M - m) ** 2 / 4 * (1 + 1e-12)


def test_smooth_bound_example(golden):
    # SPEC.md:318 worked example of the Sec. 4.3 O(1) bound D l^2/(4 gamma^2)
    g = golden["smooth_example"]
    bound = ((g["D"] * g["l"]) * g["l"]) / ((4 * g["gamma"]) * g["gamma"])
    assert abs(bound - g["bound"]) < 1e-12 and bound <= g["eta"]


def test_kernel_values(golden):
    # PAPER.md:286 Gaussian kernel via the oracle's direct sum with a single source, b = 1
    for c in golden["kernel"]["cases"]:
        X = np.array([c["x"]])
        Y = np.array([c["y"]])
        v = oracle.direct(X, np.ones(1), c["gamma"], Y=Y)
        assert abs(v[0] - c["k"]) < 1e-15


def test_grid_size_cap():
    # PAPER.md:286 "a cap at r = 2048": 3^7 = 2187 > 2048 -> grid-too-large (reading R20)
    X = np.random.default_rng(0).uniform(size=(50, 7))
    with pytest.raises(oracle.OracleError) as e:
        oracle.f3m(X, np.ones(50), 1.0, P=3)
    assert e.value.status == 6
    oracle.f3m(X, np.ones(50), 1.0, P=3, node_cap=2187)  # raising the cap is allowed


def test_invalid_inputs():
    X = np.zeros((4, 3))
    with pytest.raises(oracle.OracleError) as e:
        oracle.f3m(X, np.ones(4), -1.0)
    assert e.value.status == 5
    X[1, 2] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.f3m(X, np.ones(4), 1.0)
    assert e.value.status == 2
