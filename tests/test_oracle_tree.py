"""Pins for the oracle's binning, permutation, box tables, interaction division and
classification (CPU only).

The checks are geometric or combinatorial properties fixed by the paper (box membership,
Fig. 6 division, Thm. 2 accounting, Prop. 3 depth bound, the far/smooth/small/adaptive
rules re-derived from box centres), the SPEC worked examples, and brute force.
"""
import math

import numpy as np
import pytest

import datagen
import oracle


def deinterleave(keys, D, T, t):
    """Cell coordinates i_{p,d} at depth t from nested-Morton keys at depth T (test-side
    decoding: bit s of the prefix group belongs to dimension s)."""
    pre = np.asarray(keys, dtype=np.uint64) >> np.uint64(D * (T - t))
    cells = np.zeros((pre.size, D), dtype=np.int64)
    for s in range(t):  # level-s group, most significant first
        grp = (pre >> np.uint64(D * (t - 1 - s))) & np.uint64((1 << D) - 1)
        for d in range(D):
            bit = ((grp >> np.uint64(d)) & np.uint64(1)).astype(np.int64)
            cells[:, d] |= bit << (t - 1 - s)
    return cells


def test_box_index_worked_examples(golden):
    for c in golden["box_index"]["cases"]:
        assert oracle.box_index(c["x"], c["t"], c["E"], c["alpha"]) == c["beta"]


def test_group_points_example(golden):
    # keys [1,0,1,2,3] at depth 2, D=1 (last point sets E = 1)
    X = np.array([[0.3], [0.0], [0.3], [0.55], [1.0]])
    r = oracle.f3m(X, np.ones(5), gamma=0.25, P=2, zeta=1, rho=0)
    assert r.T_sort == 2
    np.testing.assert_array_equal(r.keys[0], [1, 0, 1, 2, 3])
    np.testing.assert_array_equal(r.perm[0][:4], golden["group_points"]["pi"])


CASES = [("uniform", 3000, 3, 0.05), ("normal", 3000, 3, 0.2), ("uniform", 2000, 1, 0.01),
         ("normal", 1500, 2, 0.1), ("uniform", 600, 5, 0.3), ("normal", 500, 7, 0.6)]


@pytest.mark.parametrize("kind,n,D,gamma", CASES)
def test_permutation_and_box_membership(kind, n, D, gamma):
    X = datagen.points(kind, n, D, seed=5).double().numpy()
    hiD = D >= 5  # keep the D >= 5 cases cheap: no division (zeta = n), keys to depth 3
    r = oracle.f3m(X, np.ones(n), gamma, P=2, zeta=n if hiD else 8, rho=4, max_depth=3 if hiD else -1)
    T = r.T_sort
    assert T >= 1
    key, pi = r.keys[0], r.perm[0]
    # bijection, sorted keys, stability (reading R13)
    np.testing.assert_array_equal(np.sort(pi), np.arange(n))
    ks = key[pi]
    assert np.all(ks[1:] >= ks[:-1])
    eq = ks[1:] == ks[:-1]
    assert np.all(pi[1:][eq] > pi[:-1][eq])
    # membership of every point in its cube at every depth, max face clamped
    for t in range(T + 1):
        l = math.ldexp(r.E, -t)
        cells = deinterleave(key, D, T, t)
        lo = r.alphaX + cells * l
        hi = lo + l
        assert np.all(X >= lo - 1e-12 * r.E)
        assert np.all(X <= hi + 1e-12 * r.E)
        top = cells == (1 << t) - 1
        assert np.all((X < hi - 1e-12 * r.E) | top | (np.abs(X - hi) <= 1e-12 * r.E))
        # box tables: distinct prefixes, contiguous, counts sum to n, no empty box
        bk, bs, bc = r.boxes[(0, t)]
        assert np.all(bc > 0) and bc.sum() == n
        np.testing.assert_array_equal(bs, np.concatenate([[0], np.cumsum(bc)[:-1]]))
        pre = ks >> np.uint64(D * (T - t))
        np.testing.assert_array_equal(bk, np.unique(pre))
        assert np.all(bk[1:] > bk[:-1])


def test_fig6_division_example(golden):
    # D = 1: the root pair (0,0) divides into [(0,0),(0,1),(1,0),(1,1)] (Fig. 6)
    X = np.array([[0.0], [0.4], [0.6], [1.0]])
    r = oracle.f3m(X, np.ones(4), gamma=0.05, P=2, zeta=1, rho=0)
    kp, kq, tg = r.pairs[1]
    np.testing.assert_array_equal(np.stack([kp, kq], 1), golden["fig6_division"]["children_pairs"])
    assert np.all(tg == oracle.TAG_NEAR)


def _check_division_and_accounting(r, D):
    """Thm. 2 (App. E) in its exact form:
    at every depth the expansion of the previous near list is partitioned into removed-empty,
    far, smooth, small and near pairs, and the new pairs are exactly the non-empty children."""
    st = r.stats
    prev_near = {(0, 0)}
    for t in range(1, r.depth_reached + 1):
        kp, kq, tg = r.pairs[t]
        M = len(tg)
        assert st["M"][t] == M
        assert st["m_far"][t] + st["m_smooth"][t] + st["m_small"][t] + st["m_near"][t] == M
        assert st["m_far"][t] == np.sum((tg == 1) | (tg == 2))
        assert st["m_far_dropped"][t] == np.sum(tg == 2)
        assert st["expanded"][t] == len(prev_near) * 4 ** D
        # sorted by construction (Sec. 4.1, Fig. 6)
        order = np.lexsort((kq, kp))
        np.testing.assert_array_equal(order, np.arange(M))
        # parents are exactly the previous near pairs; child counts match the box tables
        parents = set(zip((kp >> np.uint64(D)).tolist(), (kq >> np.uint64(D)).tolist()))
        assert parents == prev_near
        bxk, _, _ = r.boxes[(0, t)]
        byk, _, _ = r.boxes[(1, t)]
        ncx = {}
        for k in bxk.tolist():
            ncx[k >> D] = ncx.get(k >> D, 0) + 1
        ncy = {}
        for k in byk.tolist():
            ncy[k >> D] = ncy.get(k >> D, 0) + 1
        assert M == sum(ncx[p] * ncy[q] for p, q in prev_near)
        prev_near = set(zip(kp[tg == 0].tolist(), kq[tg == 0].tolist()))
    assert len(prev_near) == r.n_near_flushed


def _check_classification(r, X, Y, D, gamma, P, eta, rho, maxnorm=False):
    """Re-derive every tag from box geometry: far <=> ||c_p - c_q|| >= 2l (Sec. 3),
    smooth <=> D l^2/(4 gamma^2) <= eta (Sec. 4.3), small <=> |B_p|+|B_q| <= rho
    (Sec. 4.2), dropped <=> far with l^2/(2 gamma^2) > 5."""
    T = r.T_sort
    for t in range(1, r.depth_reached + 1):
        l = math.ldexp(r.E, -t)
        kp, kq, tg = r.pairs[t]
        cp = r.alphaX + (deinterleave(kp << np.uint64(D * (T - t)), D, T, t) + 0.5) * l
        cq = r.alphaY + (deinterleave(kq << np.uint64(D * (T - t)), D, T, t) + 0.5) * l
        dist = np.abs(cp - cq).max(1) if maxnorm else np.sqrt(((cp - cq) ** 2).sum(1))
        bxk, _, bxc = r.boxes[(0, t)]
        byk, _, byc = r.boxes[(1, t)]
        cntp = bxc[np.searchsorted(bxk, kp)]
        cntq = byc[np.searchsorted(byk, kq)]
        far = dist >= 2 * l * (1 - 1e-12)
        smooth = D * l * l / (4 * gamma * gamma) <= eta
        small = cntp + cntq <= rho
        q = l * l / (2 * gamma * gamma)
        want = np.where(far, np.where(q > 5, 2, 1), np.where(smooth, 3, np.where(small, 4, 0)))
        np.testing.assert_array_equal(tg, want)
        expect_pfar = min(P, 3) if q <= 0.01 else (P if q <= 5 else 0)
        assert r.stats["pfar"][t] == expect_pfar


ACC_CASES = [  # kind, n, D, gamma, P, eta, rho, zeta, k(X,Y)?
    ("uniform", 4000, 3, 0.08, 2, 0.5, 16, 8, False),
    ("normal", 4000, 3, 0.25, 2, 0.5, 16, 8, False),
    ("normal", 3000, 2, 0.05, 3, 0.3, 20, 10, False),
    ("uniform", 2000, 1, 0.004, 4, 0.5, 8, 4, False),
    ("uniform", 2500, 3, 0.1, 2, 0.5, 16, 8, True),
    ("normal", 800, 5, 0.35, 2, 0.5, 64, 32, False),
]


@pytest.mark.parametrize("kind,n,D,gamma,P,eta,rho,zeta,xy", ACC_CASES)
def test_thm2_accounting_and_classification(kind, n, D, gamma, P, eta, rho, zeta, xy):
    X = datagen.points(kind, n, D, seed=11).double().numpy()
    Y = datagen.points("normal", n // 2, D, seed=12).double().numpy() * 0.3 + 0.5 if xy else None
    b = datagen.weights(n // 2 if xy else n, seed=13).double().numpy()
    r = oracle.f3m(X, b, gamma, P=P, eta=eta, rho=rho, zeta=zeta, Y=Y)
    assert r.depth_reached >= 2
    _check_division_and_accounting(r, D)
    _check_classification(r, X, X if Y is None else Y, D, gamma, P, eta, rho)


@pytest.mark.parametrize("q,expect", [(0.005, 3), (1.0, 5), (6.0, 0)])
def test_adaptive_rule_branches(golden, q, expect):
    # E = 1 exactly; depth 2 edge l = 1/4; q = l^2/(2 gamma^2)
    X = np.linspace(0.0, 1.0, 64)[:, None]
    gamma = math.sqrt(0.0625 / (2 * q))
    r = oracle.f3m(X, np.ones(64), gamma, P=5, eta=0.001, zeta=1, rho=0)
    assert r.depth_reached >= 2
    assert r.stats["pfar"][2] == expect
    case = [c for c in golden["adaptive_rule"]["cases"] if c["q"] == q][0]
    assert case["P_far"] == expect


def test_prop3_depth_bound_on_lattice():
    """Prop. 3 (App. E): max divisions log_{2^D} n; a 16^3
    lattice with zeta = 1 stops in <= 4 divisions."""
    g = (np.arange(16) + 0.5) / 16
    X = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    r = oracle.f3m(X, np.ones(len(X)), gamma=0.05, P=2, zeta=1, rho=0)
    assert 1 <= r.depth_reached <= 4
    assert r.boxes[(0, 4)][2].max() == 1


def test_thm1_depth_bound():
    """Thm. 1 (App. E): depth <= ceil(log2(D E^2/(4 gamma^2 eta))) + 1
    (SPEC.md:347)."""
    for gamma in (0.05, 0.1, 0.3):
        X = datagen.points("uniform", 3000, 3, seed=2).double().numpy()
        r = oracle.f3m(X, np.ones(3000), gamma, P=2, zeta=1, rho=0)
        bound = math.ceil(math.log2(3 * r.E ** 2 / (4 * gamma ** 2 * 0.5))) + 1
        assert r.depth_reached <= bound
        assert r.t_star <= bound


@pytest.mark.parametrize("kind,n,D,gamma,P,eta,rho,zeta,xy", [ACC_CASES[0], ACC_CASES[4], ACC_CASES[5]])
def test_maxnorm_admissibility_classification(kind, n, D, gamma, P, eta, rho, zeta, xy):
    """F3M_ADMISSIBLE_MAXNORM: far <=> max_d |c_p - c_q| >= 2l, every tag
    re-derived from box geometry; Thm. 2 accounting unchanged."""
    X = datagen.points(kind, n, D, seed=11).double().numpy()
    Y = datagen.points("normal", n // 2, D, seed=12).double().numpy() * 0.3 + 0.5 if xy else None
    b = datagen.weights(n // 2 if xy else n, seed=13).double().numpy()
    r = oracle.f3m(X, b, gamma, P=P, eta=eta, rho=rho, zeta=zeta, Y=Y, flags=oracle.MAXNORM)
    assert r.depth_reached >= 2
    _check_division_and_accounting(r, D)
    _check_classification(r, X, X if Y is None else Y, D, gamma, P, eta, rho, maxnorm=True)


def test_maxnorm_corner_touching_boxes_are_not_far():
    """D = 4, two unit boxes touching at a corner: ||c_p - c_q|| = 2 l (far by the literal
    Euclidean rule of PAPER.md:135), max-norm distance l (not far)."""
    D = 4
    X = np.array([[0.1] * D, [0.9] * D, [0.4] * D, [1.9] * D], dtype=np.float64)  # cube edge 1.8
    b = np.ones(4)
    euc = oracle.f3m(X, b, 10.0, P=2, rho=0, zeta=1, max_depth=1, flags=oracle.NO_SMOOTH)
    mx = oracle.f3m(X, b, 10.0, P=2, rho=0, zeta=1, max_depth=1, flags=oracle.NO_SMOOTH | oracle.MAXNORM)
    # depth 1: the points sit in the boxes (0,0,0,0) and (1,1,1,1) (keys 0 and 15)
    kp, kq, tg = euc.pairs[1]
    kpm, kqm, tgm = mx.pairs[1]
    i = int(np.where((kp == 0) & (kq == 15))[0][0])
    assert tg[i] in (1, 2)       # Euclidean: corner-touching boxes are far
    assert tgm[i] not in (1, 2)  # max norm: they are near
