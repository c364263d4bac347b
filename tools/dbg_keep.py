import sys, numpy as np
sys.path.insert(0, '.')
import datagen, oracle, torch
import paper_2202_01085_b200 as f3m
from tests.test_gpu_parity import run_both, rel, relmax
X = datagen.points("normal", 12000, 3, seed=0); b = datagen.weights(12000, seed=1)
for flags in (0, 64):
    g, r = run_both(f3m, X, b, datagen.gamma_for_ev("normal", 3, 1.0), P=3, flags=flags)
    for gc, oc in zip(g["charges"], r.charges):
        gs, os_ = np.argsort(gc["src_key"]), np.argsort(oc["src_key"])
        print(flags, gc["t"], gc["P"], len(gs), "W", rel(gc["W"][gs], oc["W"][os_]), relmax(gc["W"][gs], oc["W"][os_]), "U", rel(gc["U"], oc["U"]), relmax(gc["U"], oc["U"]))
    print("v", rel(g["v"], r.v))
