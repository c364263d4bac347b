"""GPU parity at the BASELINE configs' own scale (VERDICT r1 "Make parity
green at the BASELINE configs' own scale").  Each case is the config's size and data
distribution, compared with the oracle through the C ABI:

* C2 (n = 1e6, D = 3, N(0, I), EV = 1): the FULL oracle -- bit-exact pi and keys, every depth's
  classified pair list, the Thm. 2 counters, the charges / locals of every (depth, P') group and
  v element by element (relative L2 <= 1e-5; largest element error <= 1e-4 of max |v|).
* C4 with EV = 10 at n = 2e7 (12-bit keys: two LSD passes, sorted far field, exact multi-level
  M2M / L2L, the LSD un-permutation): the oracle in subset-target mode (whole tree and every
  charge, v for the first rows) -- charges of every source box, locals of the evaluated boxes,
  v on the evaluated rows.
* C5 (n = 1e6 uniform, D = 5 P = 4 (m = 1024) and D = 7 P = 2 (m = 128)): subset-target mode
  with a few rows (the oracle's dense m^2 M2L per pair is the cost) -- v on those rows, every
  charge set's W, the evaluated boxes' U.
* The ablation flags F3M_NO_SMALL and F3M_NO_DROP on C2-shaped data (full oracle).
"""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-5
TOL_MAX = 1e-4  # element-wise (see tests/test_gpu_parity.py TOL_MAX)


@pytest.fixture(scope="module")
def f3m():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2202_01085_b200 as m
    return m


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def relmax(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def gpu_run(f3m, X, b, gamma, **kw):
    f3m.debug.enable(True)
    try:
        v, st = f3m.matvec(X.cuda(), b.cuda(), gamma, return_stats=True, **kw)
        torch.cuda.synchronize()
        n = X.shape[0]
        out = dict(v=v.cpu().numpy(), st=st, perm=f3m.debug.perm(0, n), keys=f3m.debug.keys(0, n),
                   pairs={t: f3m.debug.pairs(t) for t in range(1, st.depth_reached + 1)},
                   charges=f3m.debug.charges(X.shape[1]))
    finally:
        f3m.debug.enable(False)
    return out


def compare_charges(g, r, evaluated_only):
    """W of every source box; U of the target boxes the oracle computed (all of them, or the
    evaluated ones in subset-target mode), matched by box key."""
    assert len(g["charges"]) == len(r.charges)
    for gc, oc in zip(g["charges"], r.charges):
        assert (gc["t"], gc["P"]) == (oc["t"], oc["P"])
        gs, os_ = np.argsort(gc["src_key"]), np.argsort(oc["src_key"])
        np.testing.assert_array_equal(gc["src_key"][gs], oc["src_key"][os_])
        assert rel(gc["W"][gs], oc["W"][os_]) <= TOL
        assert relmax(gc["W"][gs], oc["W"][os_]) <= TOL_MAX
        pos = {int(k): i for i, k in enumerate(gc["tgt_key"])}
        np.testing.assert_array_equal(gc["tgt_key"], oc["tgt_key"])
        # subset-target mode: the oracle runs stage 2 only for target boxes holding an evaluated
        # row (the others keep U = 0)
        rows = np.flatnonzero(np.any(oc["U"] != 0, axis=1)) if evaluated_only else np.arange(len(oc["tgt_key"]))
        assert len(rows) > 0
        idx = [pos[int(oc["tgt_key"][i])] for i in rows]
        U = gc["U"][idx]
        assert rel(U, oc["U"][rows]) <= TOL
        assert relmax(U, oc["U"][rows]) <= TOL_MAX


def compare_full(g, r):
    st = g["st"]
    assert (st.t_star, st.t_sort, st.depth_reached) == (r.t_star, r.T_sort, r.depth_reached)
    assert st.E == r.E
    np.testing.assert_array_equal(g["perm"], r.perm[0])
    np.testing.assert_array_equal(g["keys"], r.keys[0][r.perm[0]])
    for t in range(1, r.depth_reached + 1):
        for a, o in zip(g["pairs"][t], r.pairs[t]):
            np.testing.assert_array_equal(a, o)
    for name in ("M", "expanded", "m_far", "m_far_dropped", "m_smooth", "m_small", "m_near", "boxes_x", "empty_x"):
        np.testing.assert_array_equal(np.array(getattr(st, name))[: r.depth_reached + 1],
                                      r.stats[name][: r.depth_reached + 1], err_msg=name)


def test_c2_full_oracle_1e6(f3m):
    n, D = 1_000_000, 3
    X = datagen.points("normal", n, D, seed=0)
    b = datagen.weights(n, seed=1)
    g = datagen.gamma_for_ev("normal", D, 1.0)
    gr = gpu_run(f3m, X, b, g, P=4, eta=0.5)
    r = oracle.f3m(X, b, g, P=4, eta=0.5)
    compare_full(gr, r)
    assert gr["st"].near_pairs > 0  # the small field is exercised at this size
    compare_charges(gr, r, evaluated_only=False)
    assert rel(gr["v"], r.v) <= TOL
    assert relmax(gr["v"], r.v) <= TOL_MAX


@pytest.mark.parametrize("flags", [8, 16], ids=["NO_SMALL", "NO_DROP"])
def test_ablation_flags_full_oracle(f3m, flags):
    n, D = 200_000, 3
    X = datagen.points("normal", n, D, seed=2)
    b = datagen.weights(n, seed=3)
    g = datagen.gamma_for_ev("normal", D, 1.0)
    gr = gpu_run(f3m, X, b, g, P=4, eta=0.5, flags=flags)
    r = oracle.f3m(X, b, g, P=4, eta=0.5, flags=flags)
    compare_full(gr, r)
    if flags == 8:
        assert int(np.sum(r.stats["m_small"])) == 0
    else:
        assert int(np.sum(r.stats["m_far_dropped"])) == 0
    compare_charges(gr, r, evaluated_only=False)
    assert rel(gr["v"], r.v) <= TOL
    assert relmax(gr["v"], r.v) <= TOL_MAX


def test_c4_ev10_subset_2e7(f3m):
    n, D, m = 20_000_003, 3, 300
    X = datagen.points("uniform", n, D, seed=0)
    b = datagen.weights(n, seed=1)
    g = datagen.gamma_for_ev("uniform", D, 10.0)
    gr = gpu_run(f3m, X, b, g, P=4, eta=0.5)
    st = gr["st"]
    assert st.t_sort == 4 and st.num_sort_passes == 2  # the multi-pass path at scale
    r = oracle.f3m(X, b, g, P=4, eta=0.5, n_eval=m)
    compare_full(gr, r)
    compare_charges(gr, r, evaluated_only=True)
    assert rel(gr["v"][:m], r.v[:m]) <= TOL
    assert relmax(gr["v"][:m], r.v[:m]) <= TOL_MAX


@pytest.mark.parametrize("D,P,m", [(5, 4, 2), (7, 2, 4)])
def test_c5_uniform_subset_1e6(f3m, D, P, m):
    n = 1_000_000
    X = datagen.points("uniform", n, D, seed=0)
    b = datagen.weights(n, seed=1)
    g = datagen.gamma_for_ev("uniform", D, 1.0)
    gr = gpu_run(f3m, X, b, g, P=P, eta=0.5)
    r = oracle.f3m(X, b, g, P=P, eta=0.5, n_eval=m)
    compare_full(gr, r)
    compare_charges(gr, r, evaluated_only=True)
    assert rel(gr["v"][:m], r.v[:m]) <= TOL
    assert relmax(gr["v"][:m], r.v[:m]) <= TOL_MAX
