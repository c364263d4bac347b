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
    # near field / small pairs (normal data): no reuse state, every apply is a full matvec
    X = datagen.points("normal", 20000, 3, seed=0).cuda()
    g = datagen.gamma_for_ev("normal", 3, 1.0)
    op = f3m.Operator(X, g)
    assert not op.reuses_plan
    b = datagen.weights(20000, seed=1).cuda()
    assert torch.equal(op.apply(b), f3m.matvec(X, b, g))
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
