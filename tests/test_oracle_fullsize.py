"""Pins for the oracle's full-size helpers (CPU only).

The 1e9-point parity test cannot run the whole oracle; it uses three helpers that take the
fp32 points directly (step 2 cube, step 4 keys, stage 1 for one box) and the oracle's
subset-target mode (v only for the first rows, PAPER.md:286 evaluates the error on the
first rows).  Each is pinned here against something other than itself:

* cube_f32: numpy's min / max (a library routine) of the same fp32 values;
* keys_f32: the worked box-index example and the keys the
  whole-oracle run produces (pinned in test_oracle_tree.py);
* s2m_box_f32: the charges of the whole-oracle run for every source box (pinned by the
  brute-force K^ construction in test_oracle_f3m.py), and a closed form: one point on a
  Chebyshev node gives W = b e_k (Lagrange basis is the Kronecker delta at nodes);
* subset mode: v on the evaluated rows is bit-identical to the full run, the rest is 0.
"""
import numpy as np
import pytest

import datagen
import oracle


def test_cube_f32_matches_numpy():
    X = datagen.points("normal", 5001, 3, seed=3).numpy()
    alpha, E = oracle.cube_f32(X)
    Xd = X.astype(np.float64)
    np.testing.assert_array_equal(alpha, Xd.min(0))
    assert E == (Xd.max(0) - Xd.min(0)).max()


def test_keys_f32_worked_example_and_whole_run():
    # D = 2, E = 2, alpha = 0, x = (1.5, 0.5): depth-1 cells (1, 0) -> Morton key 1 (dim 1 lsb)
    X = np.array([[1.5, 0.5], [0.0, 0.0], [2.0, 2.0]], dtype=np.float32)
    k = oracle.keys_f32(X, 1, 2.0, [0.0, 0.0])
    np.testing.assert_array_equal(k, [1, 0, 3])  # max face clamps to 2^t - 1
    X = datagen.points("uniform", 20000, 3, seed=0)
    b = datagen.weights(20000, seed=1)
    g = datagen.gamma_for_ev("uniform", 3, 10.0)
    r = oracle.f3m(X, b, g)
    assert r.T_sort == 4
    k = oracle.keys_f32(X.numpy(), r.T_sort, r.E, r.alphaX)
    np.testing.assert_array_equal(k.astype(np.uint64), r.keys[0])


def test_s2m_box_matches_whole_run_charges():
    X = datagen.points("uniform", 20000, 3, seed=0)
    b = datagen.weights(20000, seed=1)
    g = datagen.gamma_for_ev("uniform", 3, 1.0)
    r = oracle.f3m(X, b, g)
    assert r.charges
    D = 3
    for ch in r.charges:
        t, P = ch["t"], ch["P"]
        for j, key in enumerate(ch["src_key"][:8]):
            # box cell coordinates from the nested Morton key (dimension d at bit d of each level)
            cell = [0] * D
            for s in range(t):
                lv = (int(key) >> (D * (t - 1 - s))) & ((1 << D) - 1)
                for d in range(D):
                    cell[d] = (cell[d] << 1) | ((lv >> d) & 1)
            W = oracle.s2m_box_f32(X.numpy(), b.numpy(), P, r.T_sort, t, r.E, r.alphaX, cell)
            np.testing.assert_allclose(W, ch["W"][j], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("P", [2, 3, 4])
def test_s2m_box_point_on_node(P):
    # box [0, 1)^2 at t = 1 of the cube alpha = 0, E = 2; node s_k maps to x = (s_k + 1) / 2
    s = oracle.cheb_nodes(P)
    for k0 in range(P):
        for k1 in range(P):
            x = np.array([[(s[k0] + 1) / 2, (s[k1] + 1) / 2], [2.0, 2.0]], dtype=np.float32)
            if not (np.float64(x[0, 0]) * 2 - 1 == s[k0] and np.float64(x[0, 1]) * 2 - 1 == s[k1]):
                continue  # node not exactly representable in fp32
            if x[0].max() >= 1.0:
                continue  # a node on the upper face belongs to the neighbouring cell (R12)
            W = oracle.s2m_box_f32(x, np.array([0.75, 5.0], dtype=np.float32), P, 1, 1, 2.0, [0.0, 0.0], [0, 0])
            e = np.zeros(P * P)
            e[k0 + P * k1] = 0.75
            np.testing.assert_allclose(W, e, atol=1e-15)


@pytest.mark.parametrize("kind,ev", [("uniform", 1.0), ("normal", 1.0)])
def test_subset_mode_equals_full_run_on_evaluated_rows(kind, ev):
    X = datagen.points(kind, 20000, 3, seed=0)
    b = datagen.weights(20000, seed=1)
    g = datagen.gamma_for_ev(kind, 3, ev)
    full = oracle.f3m(X, b, g, details=False)
    sub = oracle.f3m(X, b, g, details=False, n_eval=700)
    np.testing.assert_array_equal(sub.v[:700], full.v[:700])
    assert not np.any(sub.v[700:])
