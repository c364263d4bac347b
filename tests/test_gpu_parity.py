"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Bit-exact for keys, permutations and classified pair lists; relative L2 <= 1e-5
for charges, locals and v (north_star); F^3M vs exact err^2 <= 1e-3 at the defaults."""
import math

import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu

TOL_V = 1e-5
# element-wise check (relmax below): a bad box or point shows as an O(1) error; the bound
# leaves room for fp32 near-field sums with cancellation (error ~ 2^-23 * sum_j |k b_j|, which can
# be ~10x |v_i| for small-field pairs of a few hundred N(0, 1) weights)
TOL_MAX = 1e-4


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
    """Largest element-wise error over the largest magnitude: one bad box or point shows here
    even when the relative L2 over millions of elements hides it."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def run_both(f3m, X, b, gamma, Y=None, **kw):
    f3m.debug.enable(True)
    try:
        v, st = f3m.matvec(X.cuda(), b.cuda(), gamma, Y=None if Y is None else Y.cuda(), return_stats=True, **kw)
        torch.cuda.synchronize()
        g = dict(v=v.cpu().numpy(), st=st)
        if st.t_sort >= 1 and not (kw.get("flags", 0) & 1):
            g["perm"] = [f3m.debug.perm(0, X.shape[0]), f3m.debug.perm(1, (X if Y is None else Y).shape[0])]
            g["keys"] = [f3m.debug.keys(0, X.shape[0]), f3m.debug.keys(1, (X if Y is None else Y).shape[0])]
            g["pairs"] = {t: f3m.debug.pairs(t) for t in range(1, st.depth_reached + 1)}
            g["charges"] = f3m.debug.charges(X.shape[1])
    finally:
        f3m.debug.enable(False)
    okw = {k: v for k, v in kw.items() if k in ("P", "eta", "rho", "zeta", "max_depth", "flags", "node_cap",
                                                "sparse_level")}
    if "max_depth" not in okw:
        okw["max_depth"] = -1
    r = oracle.f3m(X, b, gamma, Y=Y, **okw)
    return g, r


CASES = [  # kind, n, D, ev, P, extra
    ("uniform", 10000, 3, 1.0, 4, {}),                   # C1-like, t* = 2, single pass
    ("uniform", 10000, 3, 0.1, 4, {}),                   # t* = 1, smooth only
    ("normal", 20000, 3, 1.0, 4, {}),                    # C2-like: drops at depth 1, small pairs, 2 passes
    ("uniform", 30001, 3, 10.0, 4, {}),                  # t* = 4: 12-bit keys, 2 passes, ragged tile
    ("uniform", 5000, 2, 1.0, 6, {}),
    ("normal", 6000, 1, 1.0, 8, {}),
    ("uniform", 3000, 5, 1.0, 2, {}),
    ("normal", 2000, 7, 1.0, 2, {"max_depth": 1}),
    ("normal", 12000, 3, 1.0, 3, {"zeta": 16, "rho": 40}),  # deeper tree, near flush
    ("uniform", 8000, 3, 1.0, 4, {"flags": 2 | 4}),     # NO_SMOOTH | NO_ADAPTIVE
    ("uniform", 20000, 4, 1.0, 2, {}),                  # 256 leaf boxes: tile-local piece mode
    ("normal", 50000, 1, 100.0, 4, {}),                 # D = 1, deep single-pass tree (128 boxes)
    ("uniform", 3000, 5, 1.0, 2, {"flags": 32}),        # F3M_ADMISSIBLE_MAXNORM
]


@pytest.fixture(params=["local", "global"])
def far_path(request, monkeypatch):
    """Both far-field implementations: tile-local (default where applicable) and the
    global-sorted kernels (forced with F3M_NO_LOCAL)."""
    if request.param == "global":
        monkeypatch.setenv("F3M_NO_LOCAL", "1")
    else:
        monkeypatch.delenv("F3M_NO_LOCAL", raising=False)
    return request.param


@pytest.mark.parametrize("kind,n,D,ev,P,extra", CASES)
def test_parity_end_to_end(f3m, far_path, kind, n, D, ev, P, extra):
    X = datagen.points(kind, n, D, seed=0)
    b = datagen.weights(n, seed=1)
    gamma = datagen.gamma_for_ev(kind, D, ev)
    check_case(f3m, X, b, gamma, P=P, **extra)


# Large interpolation grids (128 < P^D <= 4096): node-parallel S2M / point-parallel L2T
# (kernels_far_gen.cu).  Blob data keeps the oracle's dense per-pair M2L cheap; rho = zeta = 1
# so that the few occupied boxes interact through the far field.
GEN_CASES = [  # D, P, gamma, extra
    (5, 4, 0.2, {}),
    (3, 6, 0.1, {}),
    (4, 4, 0.15, {}),
    (5, 3, 0.25, {}),
    (6, 3, 0.3, {}),
    (7, 3, 0.35, {"node_cap": 4096}),
    (2, 10, 0.05, {}),
    (1, 12, 0.01, {}),
]


@pytest.mark.parametrize("D,P,gamma,extra", GEN_CASES)
def test_parity_large_grids(f3m, D, P, gamma, extra):
    X = datagen.points("blobs", 2000, D, seed=0)
    b = datagen.weights(2000, seed=1)
    check_case(f3m, X, b, gamma, P=P, rho=1, zeta=1, **extra)


# The interaction division + classification on the device (kernels_tree.cu), forced at every
# depth (F3M_TREE_DEVICE=1): same pair lists, tags, stats, charges and v as the oracle.
DEVICE_TREE_CASES = [  # kind, n, D, ev-or-gamma, P, extra
    ("uniform", 10000, 3, 1.0, 4, {}),
    ("normal", 20000, 3, 1.0, 4, {}),                    # drops at depth 1, small pairs
    ("uniform", 30001, 3, 10.0, 4, {}),                  # four depths
    ("normal", 12000, 3, 1.0, 3, {"zeta": 16, "rho": 40}),  # near flush at loop exit
    ("uniform", 3000, 5, 1.0, 2, {}),
    ("normal", 2000, 7, 1.0, 2, {"max_depth": 1}),
    ("uniform", 8000, 3, 1.0, 4, {"flags": 2 | 4}),
    ("uniform", 3000, 3, ("gamma", 2.0), 5, {"eta": 0.01, "zeta": 8, "rho": 16}),  # P_far = 3 != P: split lists
    ("normal", 2000, 7, 1.0, 2, {"max_depth": 1, "flags": 32}),  # max-norm admissibility
]


@pytest.mark.parametrize("kind,n,D,ev,P,extra", DEVICE_TREE_CASES)
def test_parity_device_tree(f3m, monkeypatch, kind, n, D, ev, P, extra):
    monkeypatch.setenv("F3M_TREE_DEVICE", "1")
    X = datagen.points(kind, n, D, seed=0)
    b = datagen.weights(n, seed=1)
    gamma = ev[1] if isinstance(ev, tuple) else datagen.gamma_for_ev(kind, D, ev)
    check_case(f3m, X, b, gamma, P=P, **extra)


def test_parity_device_tree_k_xy(f3m, monkeypatch):
    monkeypatch.setenv("F3M_TREE_DEVICE", "1")
    test_parity_k_xy(f3m)


def check_case(f3m, X, b, gamma, **extra):
    g, r = run_both(f3m, X, b, gamma, **extra)
    st = g["st"]
    assert st.t_star == r.t_star and st.t_sort == r.T_sort and st.depth_reached == r.depth_reached
    assert st.E == r.E
    # bit-exact keys (sorted order) and permutations (Sec. 4.1-4.2, reading R12/R13)
    np.testing.assert_array_equal(g["perm"][0], r.perm[0])
    np.testing.assert_array_equal(g["keys"][0], r.keys[0][r.perm[0]])
    # bit-exact classified pair lists per depth (Fig. 6 order, tags)
    for t in range(1, r.depth_reached + 1):
        kp, kq, tg = g["pairs"][t]
        okp, okq, otg = r.pairs[t]
        np.testing.assert_array_equal(kp, okp)
        np.testing.assert_array_equal(kq, okq)
        np.testing.assert_array_equal(tg, otg)
    # stats (Thm. 2 counters)
    for name in ("M", "expanded", "m_far", "m_far_dropped", "m_smooth", "m_small", "m_near", "boxes_x", "empty_x"):
        np.testing.assert_array_equal(np.array(getattr(st, name))[: r.depth_reached + 1],
                                      r.stats[name][: r.depth_reached + 1], err_msg=name)
    # charges (stage 1) and locals (stage 2) per (depth, P')
    assert len(g["charges"]) == len(r.charges)
    for gc, oc in zip(g["charges"], r.charges):
        assert (gc["t"], gc["P"]) == (oc["t"], oc["P"])
        # the oracle lists source boxes in first-use order, the library in key order
        gs, os_ = np.argsort(gc["src_key"]), np.argsort(oc["src_key"])
        np.testing.assert_array_equal(gc["src_key"][gs], oc["src_key"][os_])
        np.testing.assert_array_equal(gc["tgt_key"], oc["tgt_key"])
        assert rel(gc["W"][gs], oc["W"][os_]) <= TOL_V
        assert rel(gc["U"], oc["U"]) <= TOL_V
        assert relmax(gc["W"][gs], oc["W"][os_]) <= TOL_MAX
        assert relmax(gc["U"], oc["U"]) <= TOL_MAX
    assert rel(g["v"], r.v) <= TOL_V
    assert relmax(g["v"], r.v) <= TOL_MAX


def test_parity_k_xy(f3m):
    X = datagen.points("uniform", 6000, 3, seed=0)
    Y = datagen.points("normal", 4000, 3, seed=7) * 0.4 + 0.5
    b = datagen.weights(4000, seed=1)
    g, r = run_both(f3m, X, b, 0.2, Y=Y)
    np.testing.assert_array_equal(g["perm"][1], r.perm[1])
    for t in range(1, r.depth_reached + 1):
        for a, o in zip(g["pairs"][t], r.pairs[t]):
            np.testing.assert_array_equal(a, o)
    assert rel(g["v"], r.v) <= TOL_V


def test_exact_mode_and_degenerate(f3m):
    X = datagen.points("normal", 3000, 3, seed=2)
    b = datagen.weights(3000, seed=3)
    ve = oracle.direct(X, b, 0.7)
    v = f3m.matvec(X.cuda(), b.cuda(), 0.7, flags=f3m.EXACT).cpu().numpy()
    assert rel(v, ve) <= TOL_V
    v2 = f3m.matvec(X.cuda(), b.cuda(), 0.7, zeta=3000).cpu().numpy()  # zeta >= n: no division
    assert rel(v2, ve) <= TOL_V
    # all points identical: E = 0 -> direct
    Z = torch.full((100, 2), 0.3)
    bz = datagen.weights(100, seed=4)
    vz = f3m.matvec(Z.cuda(), bz.cuda(), 1.0).cpu().numpy()
    np.testing.assert_allclose(vz, np.full(100, bz.double().sum().item()), rtol=1e-6)
    # n = 1
    v1 = f3m.matvec(X[:1].contiguous().cuda(), b[:1].contiguous().cuda(), 1.0).cpu().numpy()
    assert abs(v1[0] - b[0].item()) < 1e-6


def test_zero_weights_and_linearity(f3m):
    X = datagen.points("uniform", 20000, 3, seed=5).cuda()
    g = datagen.gamma_for_ev("uniform", 3, 1.0)
    b1 = datagen.weights(20000, seed=6).cuda()
    b2 = datagen.weights(20000, seed=8).cuda()
    assert torch.all(f3m.matvec(X, torch.zeros_like(b1), g) == 0)
    v = f3m.matvec(X, 2 * b1 + b2, g).double()
    lin = 2 * f3m.matvec(X, b1, g).double() + f3m.matvec(X, b2, g).double()
    assert (torch.linalg.norm(v - lin) / torch.linalg.norm(lin)).item() <= 1e-5


def test_direct_kernels(f3m):
    X = datagen.points("normal", 3000, 3, seed=9)
    Y = datagen.points("uniform", 2500, 3, seed=10)
    b = datagen.weights(2500, seed=11)
    ve = oracle.direct(X, b, 0.9, Y=Y)
    v32 = f3m.direct(X.cuda(), b.cuda(), 0.9, Y=Y.cuda()).cpu().numpy()
    v64 = f3m.direct(X.cuda(), b.cuda(), 0.9, Y=Y.cuda(), fp64=True).cpu().numpy()
    assert rel(v32, ve) <= 1e-5
    assert rel(v64, ve) <= 1e-12


def test_host_pointer_path(f3m):
    X = datagen.points("uniform", 50000, 3, seed=12).pin_memory()
    b = datagen.weights(50000, seed=13).pin_memory()
    g = datagen.gamma_for_ev("uniform", 3, 1.0)
    vh = f3m.matvec(X, b, g)
    vd = f3m.matvec(X.cuda(), b.cuda(), g).cpu()
    assert vh.device.type == "cpu"
    assert torch.equal(vh, vd)


def test_determinism(f3m):
    X = datagen.points("normal", 40000, 3, seed=14).cuda()
    b = datagen.weights(40000, seed=15).cuda()
    g = datagen.gamma_for_ev("normal", 3, 1.0)
    assert torch.equal(f3m.matvec(X, b, g), f3m.matvec(X, b, g))


@pytest.mark.parametrize("kind,ev", [("uniform", 1.0), ("normal", 1.0), ("uniform", 10.0)])
def test_accuracy_vs_exact(f3m, kind, ev):
    """F^3M vs exact at the paper defaults (P = 4, eta = 0.5): err^2 <= 1e-3."""
    n = 200000
    X = datagen.points(kind, n, 3, seed=0)
    b = datagen.weights(n, seed=1)
    g = datagen.gamma_for_ev(kind, 3, ev)
    v = f3m.matvec(X.cuda(), b.cuda(), g).cpu().numpy()
    m = 1000
    ve = oracle.direct(X[:m], b, g, Y=X)
    err2, err = oracle.subset_error(v[:m], ve)
    assert err2 <= 1e-3, (err2, err)


@pytest.mark.parametrize("gamma,T", [(0.4, 2), (0.1, 4)])
def test_keys_on_cell_boundaries(f3m, far_path, gamma, T):
    """Adversarial binning: coordinates exactly on (and one ulp around) the cell faces
    alpha + j E / 2^T, where the fp32 fast path must defer to the exact rule (reading R12)."""
    rng = np.random.default_rng(T)
    faces = np.arange(0, 2 ** T + 1, dtype=np.float64) / 2 ** T
    base = rng.choice(faces, size=(30000, 3)).astype(np.float32)
    bump = rng.integers(-1, 2, size=base.shape)
    X = np.where(bump > 0, np.nextafter(base, np.float32(2)), np.where(bump < 0, np.nextafter(base, np.float32(-1)), base))
    X[0] = 0.0
    X[1] = 1.0
    X = torch.from_numpy(np.clip(X, 0.0, 1.0).astype(np.float32))
    b = datagen.weights(len(X), seed=3)
    g, r = run_both(f3m, X, b, gamma, P=3)
    assert r.T_sort == T
    np.testing.assert_array_equal(g["perm"][0], r.perm[0])
    np.testing.assert_array_equal(g["keys"][0], r.keys[0][r.perm[0]])
    assert rel(g["v"], r.v) <= TOL_V


def test_parity_maxbox_over_near_boxes(f3m):
    """The constructed Alg. 1 stop of tests/test_oracle_pins_alg1.py (MaxBox over the boxes in
    I_near, reading R9): the library must stop at the same depth with the same lists and v."""
    rng = np.random.default_rng(0)
    A = rng.uniform(0.0, 0.1, 200)
    B = rng.uniform(0.9, 1.0, 20)
    A[0], B[-1] = 0.0, 1.0
    C = rng.uniform(0.85, 1.0, 200)
    X = torch.from_numpy(np.concatenate([A, B])[:, None].astype(np.float32))
    Y = torch.from_numpy(C[:, None].astype(np.float32))
    b = torch.from_numpy(rng.normal(size=200).astype(np.float32))
    g, r = run_both(f3m, X, b, 1.0, Y=Y, P=2, eta=1e-12, rho=60, zeta=50)
    assert g["st"].depth_reached == r.depth_reached == 2
    assert g["st"].n_near_flushed == r.n_near_flushed == 1
    for t in range(1, r.depth_reached + 1):
        for a, o in zip(g["pairs"][t], r.pairs[t]):
            np.testing.assert_array_equal(a, o)
    assert rel(g["v"], r.v) <= TOL_V
    assert relmax(g["v"], r.v) <= TOL_MAX


# App. A datasets: clustered data, Brownian motion and fractional
# Brownian motion paths (D = 1, 2, 3 in the paper) -- strongly non-uniform box occupancy, deep
# trees, empty-box removal, small and near fields.  EV from the sample variance.
@pytest.mark.parametrize("kind,n,D,ev", [("clustered", 30000, 3, 1.0), ("bm", 30000, 2, 1.0), ("fbm", 30000, 3, 1.0),
                                         ("fbm", 20000, 1, 10.0), ("clustered", 20000, 2, 0.1)])
def test_parity_appendix_a_datasets(f3m, far_path, kind, n, D, ev):
    X, _, b, gamma = datagen.problem(kind, n, D, seed=0, ev=ev)
    check_case(f3m, X, b, gamma, P=4)


# F3M_KEEP_EMPTY: no empty-box removal (FFM(GPU) of Tables 5-6): bit-exact pair
# lists including the empty-box pairs, v as the oracle; and the full FFM(GPU) flag set.
@pytest.mark.parametrize("flags", [64, 64 | 2 | 4 | 8], ids=["KEEP_EMPTY", "FFM_GPU"])
def test_parity_keep_empty(f3m, flags):
    X = datagen.points("normal", 12000, 3, seed=0)
    b = datagen.weights(12000, seed=1)
    check_case(f3m, X, b, datagen.gamma_for_ev("normal", 3, 1.0), P=3, flags=flags)
