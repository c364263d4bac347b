import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import os, numpy as np, torch, datagen, oracle
import paper_2202_01085_b200 as f3m
X = datagen.points("uniform", 10000, 3, seed=0); b = datagen.weights(10000, seed=1)
g = datagen.gamma_for_ev("uniform", 3, 1.0)
for env in ("1", None):
    if env: os.environ["F3M_NO_THRESH"] = "1"
    else: os.environ.pop("F3M_NO_THRESH", None)
    f3m.debug.enable(True)
    v, st = f3m.matvec(X.cuda(), b.cuda(), g, return_stats=True)
    perm = f3m.debug.perm(0, 10000); keys = f3m.debug.keys(0, 10000)
    f3m.debug.enable(False)
    r = oracle.f3m(X, b, g)
    print("env", env, "depth", st.depth_reached, "perm ok", np.array_equal(perm, r.perm[0]), "keys ok", np.array_equal(keys, r.keys[0][r.perm[0]]), "v err", np.linalg.norm(v.cpu().numpy()-r.v)/np.linalg.norm(r.v))
    print(" gpu keys head", keys[:10], "oracle", r.keys[0][r.perm[0]][:10])
