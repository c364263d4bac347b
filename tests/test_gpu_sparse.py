"""GPU parity of the Smolyak sparse-grid far field (Sec. 4.2 "Sparse grids", PAPER.md:214;
reading R27) against the oracle's sparse grids (pinned in
test_oracle_sparse.py): bit-exact keys, permutations and pair lists, the nodal charges W and
locals U of every (depth, level) group and v within 1e-5 (relative L2) and 1e-4 (element-wise),
and the F^3M-vs-exact error of the sparse run."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.test_gpu_parity import check_case, f3m, rel  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n,D,q,ev,extra", [
    ("uniform", 20000, 3, 2, 1.0, {}),                      # 25 nodes, t* = 2
    ("uniform", 20000, 3, 3, 1.0, {}),                      # 69 nodes
    ("normal", 15000, 3, 2, 1.0, {}),                       # deep tree, small + near field
    ("uniform", 12000, 5, 2, 1.0, {}),                      # 61 nodes, corner-touching far pairs at t = 1
    # D = 7: zeta small enough to divide, depth 1 (8192 corner-touching far pairs; the rest small)
    ("uniform", 8000, 7, 1, 1.0, {"zeta": 16, "max_depth": 1}),   # 15 nodes
    ("uniform", 6000, 7, 2, 1.0, {"zeta": 16, "max_depth": 1}),   # 113 nodes
    # adaptive rule at t = 1 (q_1 <= 0.01): far pairs get P' = min(P, 3) -> the largest level with
    # |H| <= 3^4 (level 2, 41 nodes), smooth pairs keep level 3 (137 nodes): two groups
    ("uniform", 12000, 4, 3, 0.01, {}),
])
def test_sparse_parity(f3m, kind, n, D, q, ev, extra):
    X = datagen.points(kind, n, D, seed=0)
    b = datagen.weights(n, seed=1)
    check_case(f3m, X, b, datagen.gamma_for_ev(kind, D, ev), P=4, sparse_level=q, node_cap=4096, **extra)


def test_sparse_vs_exact(f3m):
    """Error of the sparse-grid F^3M against the exact sum decreases with the level (no dropped
    pairs at EV = 1 uniform, D = 3), and matches the oracle's error."""
    n = 20000
    X = datagen.points("uniform", n, 3, seed=0)
    b = datagen.weights(n, seed=1)
    gamma = datagen.gamma_for_ev("uniform", 3, 1.0)
    exact = oracle.direct(X.numpy()[:2000], b.numpy(), gamma, Y=X.numpy())
    errs = []
    for q in (1, 2, 3):
        v = f3m.matvec(X.cuda(), b.cuda(), gamma, P=4, sparse_level=q).cpu().double().numpy()[:2000]
        errs.append(rel(v, exact))
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 1e-2


def test_sparse_node_cap(f3m):
    X = datagen.points("uniform", 1000, 7, seed=0)
    b = datagen.weights(1000, seed=1)
    with pytest.raises(f3m.F3MError):
        f3m.matvec(X.cuda(), b.cuda(), 0.5, P=2, sparse_level=3, node_cap=500)  # |H| = 589 > 500
