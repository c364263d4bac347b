"""GPU parity of the operator API (plan reuse across right-hand sides).

The b-independent plan (cube, keys, counting-sort histogram and tile orders, tree, lists) is
built once; each apply runs S2M from the stored tile orders, M2L and L2T.  The applies must
give what a fresh f3m_matvec gives (the same sums; the moment accumulation may group the
points differently, so agreement is to fp32 rounding, 1e-6), and match the oracle for
several right-hand sides.
"""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def f3m():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2202_01085_b200 as m
    return m


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n,ev", [(200_003, 1.0), (100_000, 0.1), (300_000, 1.2)])
def test_operator_reuse_matches_matvec_and_oracle(f3m, n, ev):
    X = datagen.points("uniform", n, 3, seed=0)
    g = datagen.gamma_for_ev("uniform", 3, ev)
    Xd = X.cuda()
    op = f3m.Operator(Xd, g)
    assert op.reuses_plan
    for seed in (1, 2, 3):
        b = datagen.weights(n, seed=seed)
        bd = b.cuda()
        v = op.apply(bd)
        torch.cuda.synchronize()
        vm = f3m.matvec(Xd, bd, g)
        assert (torch.linalg.norm((v - vm).double()) / torch.linalg.norm(vm.double())).item() <= 1e-6
        if seed == 1:
            r = oracle.f3m(X, b, g, details=False, n_eval=2000)
            assert rel(v.cpu().numpy()[:2000], r.v[:2000]) <= 1e-5
    # linearity across applies of the same plan
    b1 = datagen.weights(n, seed=4).cuda()
    b2 = datagen.weights(n, seed=5).cuda()
    lin = 2 * op.apply(b1).double() + op.apply(b2).double()
    v3 = op.apply(2 * b1 + b2).double()
    assert (torch.linalg.norm(v3 - lin) / torch.linalg.norm(lin)).item() <= 1e-5
    op.close()


def test_operator_without_reuse_state(f3m):
    # normal data (near field and small pairs; a multi-pass tree keeps sorted-path reuse state,
    # a single-pass one none): either way an apply equals a fresh matvec
    X = datagen.points("normal", 20000, 3, seed=0).cuda()
    g = datagen.gamma_for_ev("normal", 3, 1.0)
    op = f3m.Operator(X, g)
    b = datagen.weights(20000, seed=1).cuda()
    v, vm = op.apply(b), f3m.matvec(X, b, g)
    assert (torch.linalg.norm((v - vm).double()) / torch.linalg.norm(vm.double())).item() <= 1e-6
    # k(X, Y)
    Y = datagen.points("uniform", 5000, 3, seed=3).cuda()
    op2 = f3m.Operator(X, 0.3, Y=Y)
    assert not op2.reuses_plan
    bY = datagen.weights(5000, seed=2).cuda()
    assert torch.equal(op2.apply(bY), f3m.matvec(X, bY, 0.3, Y=Y))


def test_operator_batch_of_right_hand_sides(f3m):
    n = 150_000
    X = datagen.points("uniform", n, 3, seed=0).cuda()
    g = datagen.gamma_for_ev("uniform", 3, 1.0)
    op = f3m.Operator(X, g)
    B = torch.stack([datagen.weights(n, seed=s) for s in (11, 12, 13)]).cuda().contiguous()
    V = op.apply(B)
    assert V.shape == (3, n)
    for r in range(3):
        assert torch.equal(V[r], op.apply(B[r].contiguous()))
    op.close()


# Multi-pass (LSD) trees: the operator keeps the sorted copies, pi, the LSD tile orders, the tree
# and the lists; each apply gathers b into the sorted order and runs S2M, M2L, the near field,
# L2T and the un-scatter.  Same sums as a fresh matvec (to fp32 rounding of the gathered b: none,
# the gather is exact) and the oracle.
SORTED_CASES = [  # kind, n, D, ev, P, extra, m (oracle rows)
    ("uniform", 300_000, 3, 10.0, 4, {}, 2000),        # 12-bit keys, exact multi-level M2M / L2L
    ("normal", 200_000, 3, 1.0, 4, {}, 2000),          # near field and small pairs on the sorted copies
    ("uniform", 200_000, 5, 1.0, 4, {}, 2),            # C5 D = 5: register-blocked S2M / L2T, grid M2L
    ("uniform", 300_000, 7, 1.0, 2, {}, 4),            # C5 D = 7
]


@pytest.mark.parametrize("kind,n,D,ev,P,extra,m", SORTED_CASES)
def test_operator_reuse_sorted_path(f3m, kind, n, D, ev, P, extra, m):
    X = datagen.points(kind, n, D, seed=0)
    g = datagen.gamma_for_ev(kind, D, ev)
    Xd = X.cuda()
    op = f3m.Operator(Xd, g, P=P, **extra)
    assert op.reuses_plan
    for seed in (1, 2):
        b = datagen.weights(n, seed=seed)
        bd = b.cuda()
        v, st = op.apply(bd, return_stats=True)
        vm, stm = f3m.matvec(Xd, bd, g, P=P, return_stats=True, **extra)
        torch.cuda.synchronize()
        assert st.num_sort_passes >= 2 and stm.num_sort_passes >= 2
        assert list(st.m_far) == list(stm.m_far) and list(st.m_near) == list(stm.m_near)
        assert (torch.linalg.norm((v - vm).double()) / torch.linalg.norm(vm.double())).item() <= 1e-6
        if seed == 1:
            r = oracle.f3m(X, b, g, P=P, details=False, n_eval=m, **extra)
            assert rel(v.cpu().numpy()[:m], r.v[:m]) <= 1e-5
    B = torch.stack([datagen.weights(n, seed=s) for s in (7, 8)]).cuda().contiguous()
    V = op.apply(B)
    for r_ in range(2):
        assert torch.equal(V[r_], op.apply(B[r_].contiguous()))
    op.close()
