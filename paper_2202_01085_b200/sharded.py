"""Targets sharded across ranks (one process per GPU), SURVEY.md 8(e).

Each rank owns a contiguous row slice of X (= Y, the k(X, X) case of App. G,
PAPER.md:740-745) as both its targets and its S2M sources.  Three collectives make every
rank build the identical tree and see the global node charges:

1. all_reduce MIN of [min_d, -max_d]          (enclosing cube)
2. all_reduce SUM of the int64 leaf histogram (box counts -> empty-box removal, zeta, rho)
3. all_reduce SUM of the fp64 node charges     (v1 = L_Y b is linear in the sources)

M2L is replicated (tiny); L2T runs on the local targets; v comes back in the local row
order.  The device work between the collectives runs in libf3m.so (plan API of
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
    def counts(self, global_minmax: torch.Tensor) -> torch.Tensor: ...  # int64 leaf histogram (local)
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

    def __init__(self, X: torch.Tensor, b: torch.Tensor, gamma: float, **cfg):
        from . import _ffi, make_config
        self._ffi = _ffi
        self.X, self.b = X, b
        self.D = X.shape[1]
        self.dev = X.device
        self._k = _ffi.Kernel(0, float(gamma))
        self._cfg = make_config(self.D, **cfg)
        self._h = C.c_void_p()
        self._stream = torch.cuda.current_stream(self.dev).cuda_stream
        _ffi.check(_ffi.lib.f3m_plan_create(X.data_ptr(), X.shape[0], self.D, b.data_ptr(), C.byref(self._k),
                                            C.byref(self._cfg), self._stream, C.byref(self._h)))
        self.stats = _ffi.Stats()

    def bbox(self) -> torch.Tensor:
        mm = np.zeros(2 * self.D)
        self._ffi.check(self._ffi.lib.f3m_plan_bbox(self._h, mm.ctypes.data))
        return torch.from_numpy(mm)

    def counts(self, global_minmax: torch.Tensor) -> torch.Tensor:
        mm = np.ascontiguousarray(global_minmax.double().cpu().numpy())
        ptr, n = C.c_void_p(), C.c_int64()
        self._ffi.check(self._ffi.lib.f3m_plan_counts(self._h, mm.ctypes.data, C.byref(ptr), C.byref(n)))
        return torch.as_tensor(_DevArray(ptr.value, n.value, "<i8", self.dev), device=self.dev)

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


def run_sharded(plan: ShardedPlan, out: torch.Tensor, group=None) -> torch.Tensor:
    """The sharded flow: local bbox -> MIN/MAX -> local counts -> SUM -> local charges ->
    SUM -> evaluate.  Every rank must call it (collectives)."""
    mm = plan.bbox()
    D = mm.numel() // 2
    dev = out.device if out.device.type == "cuda" else torch.device("cpu")
    red = torch.cat([mm[:D], -mm[D:]]).to(dev)
    dist.all_reduce(red, op=dist.ReduceOp.MIN, group=group)
    gmm = torch.cat([red[:D], -red[D:]]).cpu()
    counts = plan.counts(gmm)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    charges = plan.s2m()
    if charges.numel():
        dist.all_reduce(charges, op=dist.ReduceOp.SUM, group=group)
    return plan.evaluate(out)


def sharded_matvec(X_local: torch.Tensor, b_local: torch.Tensor, gamma: float, group=None, **cfg):
    """F^3M KMVM with targets (and S2M sources) sharded over the ranks of ``group``.
    X_local [n_local, D] fp32 (device), b_local [n_local]; returns v for the local rows."""
    plan = DevicePlan(X_local, b_local, gamma, **cfg)
    try:
        out = torch.empty(X_local.shape[0], dtype=torch.float32, device=X_local.device)
        return run_sharded(plan, out, group), plan.stats
    finally:
        plan.close()
