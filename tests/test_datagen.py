"""The App. A generators produce what the paper describes; CPU only.

datagen holds no arithmetic of the method; these checks pin the input recipe:
seeded determinism, fractional Gaussian increments with the fGn lag-1 correlation 2^(2H-1) - 1
(H = 0.75 -> 0.414; Brownian motion H = 0.5 -> 0), and the clustered data's multi-scale structure."""
import numpy as np
import torch

import datagen


def test_seeded_and_shaped():
    for kind in datagen.KINDS:
        a = datagen.points(kind, 5000, 3, seed=4)
        b = datagen.points(kind, 5000, 3, seed=4)
        assert a.shape == (5000, 3) and a.dtype == torch.float32 and a.is_contiguous()
        assert torch.equal(a, b)
        assert torch.isfinite(a).all()


def test_fbm_increment_correlation():
    for H, want in ((0.75, 2 ** (2 * 0.75 - 1) - 1), (0.5, 0.0)):
        kind = "fbm" if H == 0.75 else "bm"
        X = datagen.points(kind, 1 << 17, 2, seed=1).double()
        inc = X[1:] - X[:-1]
        for d in range(2):
            c = np.corrcoef(inc[:-1, d].numpy(), inc[1:, d].numpy())[0, 1]
            assert abs(c - want) < 0.02, (kind, d, c, want)
        # self-similarity: Var(X_t) ~ t^(2H) over the path (unit time scaling)
        v = inc.var(dim=0).mean().item()
        assert 0.5 < v * (1 << 17) ** (2 * H) < 2.0


def test_clustered_is_multiscale():
    X = datagen.points("clustered", 40000, 2, seed=3).double()
    # nearest-neighbour distances are far below the spread (recursive sub-clusters)
    sub = X[:2000]
    d = torch.cdist(sub, X)
    d[torch.arange(2000), torch.arange(2000)] = float("inf")
    nn = d.min(dim=1).values.median().item()
    assert nn < 0.01 * X.std(dim=0).mean().item()


def test_sample_ev_lengthscale():
    X = datagen.points("bm", 10000, 3, seed=0)
    g = datagen.gamma_for_ev_sample(X, 1.0)
    v = X.double().var(dim=0, unbiased=False).sum().item()
    assert abs(v / (2 * g * g) - 1.0) < 1e-12
