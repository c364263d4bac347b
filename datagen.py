"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

This module holds NO arithmetic of the F^3M method: it only draws the point clouds and
weights the paper's experiments describe, so that both sides of every parity test see
the same bytes.

* Datasets (Sec. 5 "KMVM experiments"; App. A): X uniform in
  [0,1)^D, X standard normal, the k(X,Y) case "uniformly distributed x and normal
  distributed y", and App. A's clustered data, Brownian motion (H = 0.5) and fractional
  Brownian motion (H = 0.75) paths.
* Weights b ~ N(0, I) (Sec. 5 "we fix b ~ N(0, I_n)").
* Effective-variance targeting ("We generate data such that the EV ... varies
  between 0.1, 1, 10"; EV defined in Sec. 4.3): the lengthscale is chosen as
  gamma = sqrt(sum_d Var_d / (2 EV)) using the *population* variance of the generating
  distribution (1/12 per uniform dimension, 1 per normal dimension), so gamma does not
  depend on n or the seed.

Seeds: X uses ``seed``, Y uses ``seed + 1000``, b uses ``seed + 1`` (torch.Generator,
Philox on CUDA / mt19937 on CPU).  CPU generation is used for every parity case; the
1e9-point bench generates on the device with the CUDA generator.
"""
from __future__ import annotations

import math

import torch

KINDS = ("uniform", "normal", "blobs", "clustered", "bm", "fbm")


def population_variance(kind: str) -> float:
    if kind == "uniform":
        return 1.0 / 12.0
    if kind == "normal":
        return 1.0
    raise ValueError(f"no population variance for dataset kind {kind!r} (use gamma_for_ev_sample)")


def gamma_for_ev_sample(X: torch.Tensor, ev: float) -> float:
    """gamma = sqrt(sum_d Var_d / (2 EV)) with the SAMPLE variance of X (the EV of Sec. 4.3 for
    the App. A datasets whose population variance has no closed form: clustered, BM, fBm)."""
    if ev <= 0:
        raise ValueError("EV must be > 0")
    v = X.double().var(dim=0, unbiased=False).sum().item()
    return math.sqrt(v / (2.0 * ev))


def gamma_for_ev(kind: str, D: int, ev: float) -> float:
    """gamma = sqrt(sum_d Var_d / (2 EV)) (EV of Sec. 4.3 / Sec. 5, population variance)."""
    if ev <= 0:
        raise ValueError("EV must be > 0")
    return math.sqrt(D * population_variance(kind) / (2.0 * ev))


def points(kind: str, n: int, D: int, seed: int = 0, device="cpu") -> torch.Tensor:
    """[n, D] float32 row-major point cloud."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if kind == "uniform":
        return torch.rand((n, D), generator=g, dtype=torch.float32, device=device)
    if kind == "normal":
        return torch.randn((n, D), generator=g, dtype=torch.float32, device=device)
    if kind == "blobs":
        # 4 cubes of edge 0.1 at random corners of [0, 1)^D: few occupied boxes per level, so
        # the oracle's dense per-pair far field stays cheap for large grids (P^D up to 4096)
        w = 0.1
        corners = (torch.rand((4, D), generator=g, device=device) < 0.5).float() * (1.0 - w)
        c = torch.randint(0, 4, (n,), generator=g, device=device)
        return (corners[c] + w * torch.rand((n, D), generator=g, device=device)).float()
    if kind == "clustered":
        return _clustered(n, D, g, device)
    if kind == "bm":
        return _fbm_path(n, D, 0.5, g, device)
    if kind == "fbm":
        return _fbm_path(n, D, 0.75, g, device)
    raise ValueError(f"unknown dataset kind {kind!r}")


def _clustered(n: int, D: int, g: torch.Generator, device) -> torch.Tensor:
    """App. A: cluster centres ~ N(0, I); recursively, sub-cluster centres ~ N(centre,
    (s / 4)^2 I) around each centre, 8 children per centre, until there are >= n leaves; the first
    n leaves (in a seeded random order) are the points."""
    centres = torch.randn((8, D), generator=g, dtype=torch.float64, device=device)
    s = 1.0
    while centres.shape[0] < n:
        s /= 4.0
        kids = centres.repeat_interleave(8, dim=0)
        centres = kids + s * torch.randn(kids.shape, generator=g, dtype=torch.float64, device=device)
    pick = torch.randperm(centres.shape[0], generator=g, device=device)[:n]
    return centres[pick].float().contiguous()


def _fbm_path(n: int, D: int, H: float, g: torch.Generator, device) -> torch.Tensor:
    """App. A: n samples of a D-dimensional fractional Brownian motion path with
    Hurst index H (0.5 = Brownian motion), independent coordinates, on t = 1..n scaled to unit
    time: exact fractional Gaussian noise by circulant embedding (Davies-Harte), cumulated."""
    if H == 0.5:
        inc = torch.randn((n, D), generator=g, dtype=torch.float64, device=device)
    else:
        k = torch.arange(0, n + 1, dtype=torch.float64, device=device)
        # autocovariance of fGn: 0.5 (|k+1|^2H - 2|k|^2H + |k-1|^2H)
        r = 0.5 * ((k + 1) ** (2 * H) - 2 * k ** (2 * H) + (k - 1).abs() ** (2 * H))
        circ = torch.cat([r, r[1:-1].flip(0)])  # length 2n
        lam = torch.fft.fft(circ).real.clamp_min(0.0)
        m = circ.shape[0]
        z = torch.complex(torch.randn((m, D), generator=g, dtype=torch.float64, device=device),
                          torch.randn((m, D), generator=g, dtype=torch.float64, device=device))
        w = torch.fft.fft(z * torch.sqrt(lam / m)[:, None], dim=0)
        inc = w.real[:n]
    path = torch.cumsum(inc, dim=0) * float(n) ** (-H)
    return path.float().contiguous()


def weights(n: int, seed: int = 1, device="cpu") -> torch.Tensor:
    """[n] float32, b ~ N(0, 1)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn((n,), generator=g, dtype=torch.float32, device=device)


def problem(kind: str, n: int, D: int, seed: int = 0, ev: float = 1.0, ykind: str | None = None,
            ny: int | None = None, device="cpu"):
    """A full KMVM problem: (X, Y or None for the k(X,X) case, b, gamma)."""
    X = points(kind, n, D, seed, device)
    if ykind is None:
        Y = None
        nb = n
        gamma = gamma_for_ev(kind, D, ev) if kind in ("uniform", "normal") else gamma_for_ev_sample(X, ev)
    else:
        nb = n if ny is None else ny
        Y = points(ykind, nb, D, seed + 1000, device)
        # EV of the union is dominated by the wider set; use the wider population variance.
        gamma = math.sqrt(D * max(population_variance(kind), population_variance(ykind)) / (2.0 * ev))
    b = weights(nb, seed + 1, device)
    return X, Y, b, gamma
