"""Targets sharded across ranks (one process per GPU), SURVEY.md 8(e).

Each rank owns a contiguous row slice of X (= Y, the k(X, X) case of App. G,
PAPER.md:740-745) as both its targets and its S2M sources.  Three collectives make every
rank build the identical tree and see the global node charges:

1. all_reduce MIN of [min_d, -max_d]             (enclosing cube)
2. all_gather of the sparse (key, count) leaf lists (box counts -> empty-box removal, zeta,
   rho; any D * T_sort, no dense 2^{D T} histogram)
3. all_reduce SUM of the fp64 node charges        (v1 = L_Y b is linear in the sources)

M2L is replicated (tiny); L2T runs on the local targets; the near / small field reads its
sources from the replicated full point set (Yfull, bfull: the library sorts it only when the
tree has such pairs); v comes back in the local row order.  The device work between the collectives runs in libf3m.so (plan API of
include/f3m.h); this module only marshals pointers and calls torch.distributed.

``ShardedPlan`` is the interface the driver needs from a plan; tests substitute a CPU
double of it to exercise the collective logic with the gloo backend.
"""
from __future__ import annotations

import ctypes as C
from typing import Protocol

import numpy as np
import torch
import torch.distributed as dist


class ShardedPlan(Protocol):
    def bbox(self) -> torch.Tensor: ...                          # fp64 [2D]: mins, maxs (local)
    def leaves(self, global_minmax: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]: ...  # local (keys, counts)
    def set_leaves(self, keys: torch.Tensor, counts: torch.Tensor) -> None: ...  # all ranks' lists
    def s2m(self) -> torch.Tensor: ...                           # fp64 charges (local partial)
    def evaluate(self, out: torch.Tensor) -> torch.Tensor: ...   # fp32 v (local rows)
    def close(self) -> None: ...


class _DevArray:
    """Zero-copy view of a library-owned device buffer as a torch tensor."""

    def __init__(self, ptr: int, n: int, typestr: str, device: torch.device):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}
        self.device = device


class DevicePlan:
    """libf3m.so plan over the local shard (device tensors)."""

    def __init__(self, X: torch.Tensor, b: torch.Tensor, gamma: float, Yfull: torch.Tensor | None = None,
                 bfull: torch.Tensor | None = None, **cfg):
        from . import _ffi, make_config
        self._ffi = _ffi
        self.X, self.b, self.Yfull, self.bfull = X, b, Yfull, bfull
        self.D = X.shape[1]
        self.dev = X.device
        for t, name in ((X, "X"), (b, "b"), (Yfull, "Yfull"), (bfull, "bfull")):
            if t is not None and (t.device != self.dev or t.dtype != torch.float32 or not t.is_contiguous()):
                raise ValueError(f"{name} must be a contiguous float32 tensor on {self.dev}")
        if (Yfull is None) != (bfull is None):
            raise ValueError("Yfull and bfull go together")
        ny = 0 if Yfull is None else Yfull.shape[0]
        if Yfull is not None and (Yfull.shape[1] != self.D or bfull.shape[0] != ny):
            raise ValueError("Yfull must be [ny, D] and bfull [ny]")
        self._k = _ffi.Kernel(0, float(gamma))
        self._cfg = make_config(self.D, **cfg)
        self._h = C.c_void_p()
        self._stream = torch.cuda.current_stream(self.dev).cuda_stream
        _ffi.check(_ffi.lib.f3m_plan_create(X.data_ptr(), X.shape[0], None, 0, b.data_ptr(),
                                            None if Yfull is None else Yfull.data_ptr(),
                                            None if bfull is None else bfull.data_ptr(), ny, self.D,
                                            C.byref(self._k), C.byref(self._cfg), None, self._stream,
                                            C.byref(self._h)))
        self.stats = _ffi.Stats()

    def bbox(self) -> torch.Tensor:
        mm = np.zeros(2 * self.D)
        self._ffi.check(self._ffi.lib.f3m_plan_bbox(self._h, mm.ctypes.data))
        return torch.from_numpy(mm)

    def leaves(self, global_minmax: torch.Tensor):
        mm = np.ascontiguousarray(global_minmax.double().cpu().numpy())
        kp, cp, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        self._ffi.check(self._ffi.lib.f3m_plan_leaves(self._h, mm.ctypes.data, C.byref(kp), C.byref(cp), C.byref(n)))
        if n.value == 0:
            return (torch.zeros(0, dtype=torch.int64, device=self.dev), torch.zeros(0, dtype=torch.int64, device=self.dev))
        keys = torch.as_tensor(_DevArray(kp.value, n.value, "<u8", self.dev), device=self.dev).view(torch.int64)
        counts = torch.as_tensor(_DevArray(cp.value, n.value, "<i8", self.dev), device=self.dev)
        return keys.clone(), counts.clone()

    def set_leaves(self, keys: torch.Tensor, counts: torch.Tensor) -> None:
        keys = keys.to(self.dev).contiguous()
        counts = counts.to(self.dev).contiguous()
        self._ffi.check(self._ffi.lib.f3m_plan_set_leaves(self._h, keys.data_ptr(), counts.data_ptr(), keys.numel()))

    def s2m(self) -> torch.Tensor:
        ptr, n = C.c_void_p(), C.c_int64()
        self._ffi.check(self._ffi.lib.f3m_plan_s2m(self._h, C.byref(ptr), C.byref(n)))
        if n.value == 0:
            return torch.zeros(0, dtype=torch.float64, device=self.dev)
        return torch.as_tensor(_DevArray(ptr.value, n.value, "<f8", self.dev), device=self.dev)

    def evaluate(self, out: torch.Tensor) -> torch.Tensor:
        self._ffi.check(self._ffi.lib.f3m_plan_evaluate(self._h, out.data_ptr(), C.byref(self.stats)))
        return out

    def close(self) -> None:
        if self._h:
            self._ffi.lib.f3m_plan_destroy(self._h)
            self._h = C.c_void_p()


def all_gather_varlen(x: torch.Tensor, group=None) -> torch.Tensor:
    """Concatenation over the ranks of 1-D tensors of different lengths (rank order)."""
    world = dist.get_world_size(group)
    n = torch.tensor([x.numel()], dtype=torch.int64, device=x.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    m = max(ns)
    pad = torch.zeros(m, dtype=x.dtype, device=x.device)
    pad[: x.numel()] = x
    parts = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:k] for p, k in zip(parts, ns)])


def run_sharded(plan: ShardedPlan, out: torch.Tensor, group=None) -> torch.Tensor:
    """The sharded flow: local bbox -> MIN/MAX -> local leaf lists -> all_gather -> local
    charges -> SUM -> evaluate.  Every rank must call it (collectives)."""
    mm = plan.bbox()
    D = mm.numel() // 2
    dev = out.device if out.device.type == "cuda" else torch.device("cpu")
    red = torch.cat([mm[:D], -mm[D:]]).to(dev)
    dist.all_reduce(red, op=dist.ReduceOp.MIN, group=group)
    gmm = torch.cat([red[:D], -red[D:]]).cpu()
    keys, counts = plan.leaves(gmm)
    plan.set_leaves(all_gather_varlen(keys.to(dev), group), all_gather_varlen(counts.to(dev), group))
    charges = plan.s2m()
    if charges.numel():
        dist.all_reduce(charges, op=dist.ReduceOp.SUM, group=group)
    return plan.evaluate(out)


def sharded_matvec(X_local: torch.Tensor, b_local: torch.Tensor, gamma: float, group=None,
                   Yfull: torch.Tensor | None = None, bfull: torch.Tensor | None = None, **cfg):
    """F^3M KMVM with targets (and S2M sources) sharded over the ranks of ``group``.
    X_local [n_local, D] fp32 (device), b_local [n_local]; Yfull / bfull: the replicated full
    point set and weights (needed when the tree has near / small pairs); returns v for the
    local rows."""
    plan = DevicePlan(X_local, b_local, gamma, Yfull=Yfull, bfull=bfull, **cfg)
    try:
        out = torch.empty(X_local.shape[0], dtype=torch.float32, device=X_local.device)
        return run_sharded(plan, out, group), plan.stats
    finally:
        plan.close()
