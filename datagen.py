"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

This module holds NO arithmetic of the F^3M method: it only draws the point clouds and
weights the paper's experiments describe, so that both sides of every parity test see
the same bytes.

* Datasets (Sec. 5 "KMVM experiments"; App. A): X uniform in
  [0,1)^D, X standard normal, and the k(X,Y) case "uniformly distributed x and normal
  distributed y".
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

KINDS = ("uniform", "normal", "blobs")


def population_variance(kind: str) -> float:
    if kind == "uniform":
        return 1.0 / 12.0
    if kind == "normal":
        return 1.0
    raise ValueError(f"no population variance for dataset kind {kind!r}")


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
    raise ValueError(f"unknown dataset kind {kind!r}")


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
        gamma = gamma_for_ev(kind, D, ev)
    else:
        nb = n if ny is None else ny
        Y = points(ykind, nb, D, seed + 1000, device)
        # EV of the union is dominated by the wider set; use the wider population variance.
        gamma = math.sqrt(D * max(population_variance(kind), population_variance(ykind)) / (2.0 * ev))
    b = weights(nb, seed + 1, device)
    return X, Y, b, gamma
