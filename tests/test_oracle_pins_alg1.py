"""Independent pins of two Alg. 1 decisions of the oracle (VERDICT r1 "oracle pins with gaps").

1. The smooth depth t* (Sec. 4.3 "Smoothness criteria"): the variance of a box of
   edge l along one dimension is at most l^2 / 4 (App. B), so the effective variance of a box
   pair is at most 2 * D * (l^2 / 4) / (2 gamma^2) = D l^2 / (4 gamma^2) =: s_t with l = E 2^-t,
   and t* = min{t >= 1 : s_t <= eta}.  The table below is worked by hand from that bound for
   several (E, gamma, D) -- literal numbers, not the formula re-typed -- and is chosen so that
   the plausible slips (2 gamma^2 for 4 gamma^2, l for l^2, 2^t for 4^t, a strict < for the
   paper's <=) each move t* in at least one row.
2. MaxBox in the loop condition of Alg. 1 (reading R9 / SURVEY Q9): MaxBox is
   taken over the boxes that still occur in I_near.  A constructed k(X, Y) case where the
   largest X box is fully resolved by the far field while a smaller X box stays near: under R9
   the loop stops at depth 2; with MaxBox over all boxes of the depth it would divide again.
"""
import numpy as np
import pytest

import oracle

# (D, E, gamma^2, eta, t* by hand, note)
T_STAR_TABLE = [
    # s_t = 3 * 4^-t / (4/8) = 6 * 4^-t: s1 = 1.5, s2 = 0.375 <= 0.5            -> t* = 2  (C4 EV = 1)
    (3, 1.0, 1.0 / 8.0, 0.5, 2, "C4 EV=1"),
    # s_t = 3 * 4^-t * 80 / 4 = 60 * 4^-t: 15, 3.75, 0.9375, 0.234375 <= 0.5   -> t* = 4  (C4 EV = 10)
    #   (with 2 gamma^2 instead of 4 gamma^2: 30 * 4^-t, s3 = 0.469 -> t* = 3)
    (3, 1.0, 1.0 / 80.0, 0.5, 4, "C4 EV=10"),
    # s_t = 5 * 4 * 4^-t / 4 = 5 * 4^-t: 1.25, 0.3125 <= 0.5                  -> t* = 2
    (5, 2.0, 1.0, 0.5, 2, "D=5, E=2"),
    # same with eta = 0.25: 1.25, 0.3125, 0.078125 <= 0.25                     -> t* = 3
    #   (with l instead of l^2: 5 * 2 * 2^-t / 4 = 2.5 * 2^-t: 1.25, 0.625, 0.3125, 0.156 -> t* = 4)
    (5, 2.0, 1.0, 0.25, 3, "D=5, eta=1/4"),
    # s_t = 64 * 4^-t / (4 * 1/4) = 64 * 4^-t: 16, 4, 1 <= 1 (inclusive)     -> t* = 3
    #   (a strict < would give s4 = 0.25 -> t* = 4)
    (1, 8.0, 0.25, 1.0, 3, "D=1, eta = s_3 exactly"),
    # s_t = 7 * 4^-t / (4 * 7/24) = 6 * 4^-t                                  -> t* = 2  (C5 D = 7 EV = 1)
    (7, 1.0, 7.0 / 24.0, 0.5, 2, "C5 D=7 EV=1"),
    # E = 2, gamma^2 = 1/32: s_t = 2 * 4 * 4^-t / (4/32) = 64 * 4^-t: 16, 4, 1, 0.25 <= 0.3       -> t* = 4
    (2, 2.0, 1.0 / 32.0, 0.3, 4, "D=2"),
]


@pytest.mark.parametrize("D,E,g2,eta,tstar,note", T_STAR_TABLE)
def test_smooth_depth_hand_table(D, E, g2, eta, tstar, note):
    # two points spanning the cube [0, E]^D: the enclosing edge is exactly E
    X = np.zeros((2, D))
    X[1, :] = E
    b = np.ones(2)
    r = oracle.f3m(X, b, float(np.sqrt(g2)), P=2, eta=eta, details=False)
    assert r.E == E
    assert r.t_star == tstar, note


def test_maxbox_over_near_boxes_stops_the_loop():
    """D = 1, P = 2, eta tiny (no smooth level), rho = 60, zeta = 50, gamma = 1.
    X: A = 200 points in [0, 0.1], B = 20 points in [0.9, 1.0];  Y: C = 200 points in [0.85, 1.0].
    E = 1 (X spans [0, 1]), alpha_X = 0, alpha_Y = min(C) (separate cubes, one edge).
    depth 1 (l = 1/2): X boxes {A}, {B}; Y box {C}; both pairs have centre distance < 2l = 1
      and 200 + 200, 20 + 200 > rho -> near.  MaxBox_X = 200, MaxBox_Y = 200 > zeta: divide.
    depth 2 (l = 1/4): children (A, C) at distance ~0.85 >= 2l = 0.5 -> far (q = 1/32: P nodes);
      (B, C) at distance < 0.5 and 20 + 200 > rho -> near.  I_near = {(B, C)}:
      MaxBox_X over I_near = 20 <= zeta -> the loop stops, depth_reached = 2, one near pair flushed.
      (MaxBox over every depth-2 X box would be 200 > zeta and divide again.)"""
    rng = np.random.default_rng(0)
    A = rng.uniform(0.0, 0.1, 200)
    B = rng.uniform(0.9, 1.0, 20)
    A[0], B[-1] = 0.0, 1.0
    C = rng.uniform(0.85, 1.0, 200)
    X = np.concatenate([A, B])[:, None]
    Y = C[:, None]
    b = rng.normal(size=200)
    r = oracle.f3m(X, b, 1.0, Y=Y, P=2, eta=1e-12, rho=60, zeta=50)
    assert r.E == 1.0
    assert r.depth_reached == 2
    assert r.n_near_flushed == 1
    _, _, tags2 = r.pairs[2]
    assert sorted(tags2.tolist()) == sorted([oracle.TAG_FAR, oracle.TAG_NEAR])
    # the same points with zeta = 10 (< 20): the near box B still exceeds zeta -> divides to depth 3
    r3 = oracle.f3m(X, b, 1.0, Y=Y, P=2, eta=1e-12, rho=60, zeta=10)
    assert r3.depth_reached >= 3
