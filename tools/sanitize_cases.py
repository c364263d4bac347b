"""Small F^3M calls that reach every kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py

Each case is one f3m_matvec on a seeded problem (datagen), sized so that the tile-local TMA /
warp-specialised kernels see several 4096-point tiles plus a ragged tail.  The script only
exercises the library; correctness is the parity tests' job.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2202_01085_b200 as f3m  # noqa: E402

CASES = [
    # (kind, n, D, ev, P, extra kwargs) -- which path it reaches
    ("uniform", 3 * 4096 + 77, 3, 1.0, 4, {}),                  # k_s2m_ws + k_l2t_fix (C4 shape)
    ("uniform", 3 * 4096 + 77, 3, 10.0, 4, {}),                 # LSD passes, sorted far, M2M/L2L
    ("normal", 20000, 3, 1.0, 4, {}),                           # small + near field, device division
    ("uniform", 9000, 5, 1.0, 4, {}),                           # large-grid S2M/L2T (m = 1024)
    ("uniform", 9000, 7, 1.0, 2, {}),                           # P = 2 shuffle M2L
    ("uniform", 9000, 2, 1.0, 6, {}),                           # k_s2m_ws <2,6,3>
    ("uniform", 200003, 3, 2.5, 4, {}),                         # two-digit path, T = 3 (8 buckets)
    ("uniform", 1100000, 3, 10.0, 4, {}),                       # two-digit path, T = 4: ranking-only +
                                                                # bucket-mode k_s2m_ws, k_scatter_msd
    ("uniform", 9000, 7, 1.0, 3, {"node_cap": 4096}),           # P = 3 register/shuffle M2L (k_m2l_p3)
    ("uniform", 20000, 3, 1.0, 4, {"sparse_level": 2}),         # sparse-grid kernels
    ("uniform", 12000, 5, 1.0, 4, {"sparse_level": 2}),
    ("uniform", 60000, 5, 1.0, 4, {}),                          # complete level: k_grid_col, multi-level
                                                                # M2M / L2L with k_s2m_blk / k_l2t_blk
    ("uniform", 300000, 7, 1.0, 2, {"flags": 32}),              # grid M2L, max norm (one degree)
    ("uniform", 300000, 7, 1.0, 3, {"node_cap": 4096}),         # D = 7 P = 3 blk kernels, M2M at m = 2187
]


def main():
    dev = torch.device("cuda:0")
    pick = [int(a) for a in sys.argv[1:]]  # optional case indices
    for i, (kind, n, D, ev, P, kw) in enumerate(CASES):
        if pick and i not in pick:
            continue
        X, _, b, g = datagen.problem(kind, n, D, seed=3, ev=ev)
        v = f3m.matvec(X.to(dev), b.to(dev), g, P=P, **kw)
        torch.cuda.synchronize()
        print(f"case {kind} n={n} D={D} ev={ev} P={P}: |v|={float(v.norm()):.6g}", flush=True)
    Xd = datagen.points("uniform", 5000, 3, seed=4, device="cpu").to(dev)
    bd = datagen.weights(5000, seed=5).to(dev)
    vd = f3m.direct(Xd, bd, 0.3)
    vd64 = f3m.direct(Xd, bd, 0.3, fp64=True)
    op = f3m.Operator(Xd, 0.35, P=4)
    vo = op.apply(bd)
    vb = op.apply(torch.stack([bd, 2 * bd]))
    torch.cuda.synchronize()
    print(f"direct/operator: {float(vd.norm()):.6g} {float(vd64.norm()):.6g} {float(vo.norm()):.6g} "
          f"{float(vb.norm()):.6g}", flush=True)
    op.close()
    X5 = datagen.points("uniform", 60000, 5, seed=6).to(dev)  # multi-pass tree: sorted-path operator
    op5 = f3m.Operator(X5, 0.45, P=4)
    v5 = op5.apply(datagen.weights(60000, seed=7).to(dev))
    torch.cuda.synchronize()
    print(f"sorted-path operator (reuse={op5.reuses_plan}): {float(v5.norm()):.6g}", flush=True)
    op5.close()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
