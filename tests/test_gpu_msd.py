"""The two-digit (MSD) path for deep D = 3 trees (engine.cu msd_matvec; C4 with EV = 10 is
its headline): one counting-sort scatter by the top digit into tile-aligned buckets, then the
tile-local warp-specialised S2M / L2T per bucket, the exact multi-level form in between.  Its
v is compared with the oracle (subset-target mode: the whole tree and every charge, v for the
first rows, PAPER.md:286 error protocol), with the LSD path of the same call (debug runs take
the LSD path), and the Thm. 2 counters with the oracle's.  A normal cloud (near / small field)
makes the path decline after its tree and restart on the LSD path."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.test_gpu_parity import TOL_MAX, TOL_V, f3m, rel, relmax  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu
NE = 3000


def run_gpu(f3m, X, b, gamma, debug=False, **kw):
    f3m.debug.enable(debug)
    try:
        v, st = f3m.matvec(X.cuda(), b.cuda(), gamma, return_stats=True, **kw)
        torch.cuda.synchronize()
    finally:
        f3m.debug.enable(False)
    return v.cpu().double().numpy(), st


@pytest.mark.parametrize("kind,n,ev,msd", [
    ("uniform", 2_000_000, 10.0, True),   # T_sort = 4: 64 buckets x 64 leaves
    ("uniform", 1_000_003, 2.5, True),    # T_sort = 3: 8 buckets, ragged tail
    ("normal", 300_000, 1.0, False),      # small / near field: declines, LSD path
    ("clustered", 1_000_000, 1.0, False),  # unbalanced buckets (max > 1.5 x mean): declines
])
def test_msd_parity(f3m, kind, n, ev, msd):
    X = datagen.points(kind, n, 3, seed=0)
    b = datagen.weights(n, seed=1)
    gamma = datagen.gamma_for_ev_sample(X, ev) if kind == "clustered" else datagen.gamma_for_ev(kind, 3, ev)
    v, st = run_gpu(f3m, X, b, gamma, P=4)
    v_lsd, st_lsd = run_gpu(f3m, X, b, gamma, debug=True, P=4)
    assert st.t_sort >= 3 and st.num_sort_passes == 2
    assert (st.far_groups_local > 0) == msd and st_lsd.far_groups_local == 0
    r = oracle.f3m(X, b, gamma, P=4, n_eval=NE)
    assert st.t_star == r.t_star and st.depth_reached == r.depth_reached
    for name in ("M", "m_far", "m_far_dropped", "m_smooth", "m_small", "m_near", "boxes_x"):
        np.testing.assert_array_equal(np.array(getattr(st, name))[: r.depth_reached + 1],
                                      r.stats[name][: r.depth_reached + 1], err_msg=name)
    assert rel(v[:NE], r.v[:NE]) <= TOL_V
    assert relmax(v[:NE], r.v[:NE]) <= TOL_MAX
    assert rel(v, v_lsd) <= 1e-6  # the two paths: same method, fp32 summation order only
