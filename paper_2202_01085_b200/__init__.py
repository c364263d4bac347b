"""B200-native F^3M kernel matrix-vector product (arXiv 2202.01085).

Public API (thin marshalling over the C ABI of ``libf3m.so``, include/f3m.h):

* :func:`matvec` -- the F^3M approximate KMVM v = k(X, Y) b (App. F Algorithm 1).
* :func:`direct` -- the exact KMVM by a KeOps-style tiled map-reduce (fp32 or fp64).
* :mod:`paper_2202_01085_b200.sharded` -- targets sharded over ranks with
  torch.distributed (NCCL) all-reduces of bbox, counts and node charges.

PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _ffi
from ._ffi import (ADMISSIBLE_MAXNORM, EXACT, F25M, FFM_GPU, KEEP_EMPTY, NO_ADAPTIVE, NO_DROP, NO_SMALL, NO_SMOOTH,
                   F3MError, Stats, check)

__all__ = ["matvec", "direct", "Operator", "make_config", "F3MError", "Stats", "EXACT", "NO_SMOOTH", "NO_ADAPTIVE",
           "NO_SMALL", "NO_DROP", "ADMISSIBLE_MAXNORM", "KEEP_EMPTY", "FFM_GPU", "F25M", "debug"]


def _stream_handle(device) -> int:
    if device.type != "cuda":
        return torch.cuda.current_stream().cuda_stream
    return torch.cuda.current_stream(device).cuda_stream


def make_config(D: int, P: int = 4, eta: float = 0.5, rho: int | None = None, zeta: int | None = None,
                max_depth: int | None = None, flags: int = 0, node_cap: int = 2048,
                sparse_level: int = 0) -> _ffi.Config:
    c = _ffi.default_config(D)
    c.nodes_per_dim = P
    c.node_cap = node_cap
    c.eta = eta
    c.rho = -1 if rho is None else int(rho)
    c.zeta = 0 if zeta is None else int(zeta)
    c.max_depth = -1 if max_depth is None else int(max_depth)
    c.flags = int(flags)
    c.sparse_level = int(sparse_level)
    return c


def _check_points(X: torch.Tensor, name: str) -> torch.Tensor:
    if X.dtype != torch.float32 or X.dim() != 2:
        raise ValueError(f"{name} must be a float32 [n, D] tensor")
    if not X.is_contiguous():
        raise ValueError(f"{name} must be contiguous (row-major)")
    return X


def _check_vector(v: torch.Tensor, name: str, n: int, device, dtype=torch.float32, rows: int | None = None):
    """v must be a contiguous `dtype` tensor of shape [n] (or [rows, n]) on `device`."""
    shape = (n,) if rows is None else (rows, n)
    if v.dtype != dtype or tuple(v.shape) != shape or not v.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor of shape {list(shape)}")
    if v.device != device:
        raise ValueError(f"{name} must be on {device} (got {v.device})")
    return v


def _same_device(X: torch.Tensor, Y: torch.Tensor | None, D: int):
    if Y is None:
        return
    _check_points(Y, "Y")
    if Y.shape[1] != D:
        raise ValueError("X and Y must have the same D")
    if Y.device != X.device:
        raise ValueError(f"Y must be on X's device {X.device} (got {Y.device})")


def matvec(X: torch.Tensor, b: torch.Tensor, gamma: float, Y: torch.Tensor | None = None, *, P: int = 4,
           eta: float = 0.5, rho: int | None = None, zeta: int | None = None, max_depth: int | None = None,
           flags: int = 0, node_cap: int = 2048, sparse_level: int = 0, out: torch.Tensor | None = None,
           return_stats: bool = False):
    """F^3M approximation of v = k(X, Y) b with the Gaussian kernel of lengthscale gamma.

    X [nx, D], Y [ny, D] (None: Y = X), b [ny]: float32.  Tensors on a CUDA device use the
    device path; CPU tensors (ideally pinned) use the library's staged host path (the copies
    run on the current CUDA stream inside the call)."""
    _check_points(X, "X")
    nx, D = X.shape
    _same_device(X, Y, D)
    ny = nx if Y is None else Y.shape[0]
    dev = X.device
    _check_vector(b, "b", ny, dev)
    if out is None:
        out = torch.empty(nx, dtype=torch.float32, device=dev, pin_memory=(dev.type == "cpu" and X.is_pinned()))
    else:
        _check_vector(out, "out", nx, dev)
    k = _ffi.Kernel(0, float(gamma))
    cfg = make_config(D, P, eta, rho, zeta, max_depth, flags, node_cap, sparse_level)
    st = Stats()
    with torch.cuda.device(dev if dev.type == "cuda" else torch.cuda.current_device()):
        stream = _stream_handle(dev)
        check(_ffi.lib.f3m_matvec(X.data_ptr(), nx, None if Y is None else Y.data_ptr(), ny, D, b.data_ptr(),
                                  out.data_ptr(), C.byref(k), C.byref(cfg), None, stream, C.byref(st)))
    return (out, st) if return_stats else out


def direct(X: torch.Tensor, b: torch.Tensor, gamma: float, Y: torch.Tensor | None = None, *,
           fp64: bool = False) -> torch.Tensor:
    """Exact KMVM on the device (KeOps-style tiled map-reduce): fp32 evaluation with fp64
    cross-tile accumulation, or fully fp64 when fp64=True (returns float64)."""
    _check_points(X, "X")
    if X.device.type != "cuda":
        raise ValueError("direct() needs device tensors")
    nx, D = X.shape
    _same_device(X, Y, D)
    ny = nx if Y is None else Y.shape[0]
    _check_vector(b, "b", ny, X.device)
    v = torch.empty(nx, dtype=torch.float64 if fp64 else torch.float32, device=X.device)
    k = _ffi.Kernel(0, float(gamma))
    with torch.cuda.device(X.device):
        check(_ffi.lib.f3m_direct(X.data_ptr(), nx, None if Y is None else Y.data_ptr(), ny, D, b.data_ptr(),
                                  v.data_ptr(), 1 if fp64 else 0, C.byref(k), _stream_handle(X.device)))
    return v


class Operator:
    """F^3M operator k(X, Y) with its b-independent plan built once (f3m_op_*, plan reuse
    across right-hand sides, e.g. CG / KRR iterations).  X (and Y) are referenced by the
    library: this object keeps them alive until close()."""

    def __init__(self, X: torch.Tensor, gamma: float, Y: torch.Tensor | None = None, *, P: int = 4,
                 eta: float = 0.5, rho: int | None = None, zeta: int | None = None,
                 max_depth: int | None = None, flags: int = 0, node_cap: int = 2048):
        _check_points(X, "X")
        if X.device.type != "cuda":
            raise ValueError("Operator needs device tensors")
        self.X, self.Y = X, Y
        self.nx, self.D = X.shape
        _same_device(X, Y, self.D)
        self.ny = self.nx if Y is None else Y.shape[0]
        self._k = _ffi.Kernel(0, float(gamma))
        self._cfg = make_config(self.D, P, eta, rho, zeta, max_depth, flags, node_cap)
        h = C.c_void_p()
        self._h = None
        with torch.cuda.device(X.device):
            check(_ffi.lib.f3m_op_create(X.data_ptr(), self.nx, None if Y is None else Y.data_ptr(), self.ny, self.D,
                                         C.byref(self._k), C.byref(self._cfg), _stream_handle(X.device), C.byref(h)))
        self._h = h

    @property
    def reuses_plan(self) -> bool:
        return bool(_ffi.lib.f3m_op_reuses_plan(self._h))

    def apply(self, b: torch.Tensor, out: torch.Tensor | None = None, return_stats: bool = False):
        """v = F^3M(k(X, Y)) b.  b [ny] or, for several right-hand sides, [nrhs, ny] (row r is one
        b; the result is [nrhs, nx])."""
        dev = self.X.device
        if self._h is None:
            raise ValueError("operator is closed")
        if b.dim() == 2:
            R = b.shape[0]
            _check_vector(b, "b", self.ny, dev, rows=R)
            if out is None:
                out = torch.empty((R, self.nx), dtype=torch.float32, device=dev)
            else:
                _check_vector(out, "out", self.nx, dev, rows=R)
            st = Stats()
            with torch.cuda.device(dev):
                check(_ffi.lib.f3m_op_apply_batch(self._h, b.data_ptr(), self.ny, R, out.data_ptr(), self.nx,
                                                  _stream_handle(dev), C.byref(st)))
            return (out, st) if return_stats else out
        _check_vector(b, "b", self.ny, dev)
        if out is None:
            out = torch.empty(self.nx, dtype=torch.float32, device=dev)
        else:
            _check_vector(out, "out", self.nx, dev)
        st = Stats()
        with torch.cuda.device(dev):
            check(_ffi.lib.f3m_op_apply(self._h, b.data_ptr(), out.data_ptr(), _stream_handle(dev), C.byref(st)))
        return (out, st) if return_stats else out

    __matmul__ = apply

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _ffi.lib.f3m_op_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


class debug:
    """Introspection of the last call (parity tests)."""

    @staticmethod
    def enable(on: bool = True, level: int = 1):
        """level 1: everything; level 2 (full-size tests): pairs, charges and pi of X (int32)."""
        _ffi.lib.f3m_debug_enable(level if on else 0)

    @staticmethod
    def perm32(n: int) -> np.ndarray:
        a = np.zeros(n, dtype=np.int32)
        check(_ffi.lib.f3m_debug_last_perm32(a.ctypes.data, n))
        return a

    @staticmethod
    def perm(side: int, n: int) -> np.ndarray:
        a = np.zeros(n, dtype=np.int64)
        check(_ffi.lib.f3m_debug_last_perm(side, a.ctypes.data, n))
        return a

    @staticmethod
    def keys(side: int, n: int) -> np.ndarray:
        a = np.zeros(n, dtype=np.uint64)
        check(_ffi.lib.f3m_debug_last_keys(side, a.ctypes.data, n))
        return a

    @staticmethod
    def pairs(t: int):
        n = _ffi.lib.f3m_debug_num_pairs(t)
        kp = np.zeros(n, dtype=np.uint64)
        kq = np.zeros(n, dtype=np.uint64)
        tg = np.zeros(n, dtype=np.int32)
        if n:
            check(_ffi.lib.f3m_debug_pairs(t, kp.ctypes.data, kq.ctypes.data, tg.ctypes.data))
        return kp, kq, tg

    @staticmethod
    def charges(D: int):
        out = []
        for i in range(_ffi.lib.f3m_debug_num_charge_sets()):
            info = np.zeros(6, dtype=np.int64)
            check(_ffi.lib.f3m_debug_charge_info(i, info.ctypes.data))
            t, P, ns, nt, m, q = (int(x) for x in info)
            sk = np.zeros(ns, dtype=np.uint64)
            W = np.zeros(ns * m)
            tk = np.zeros(nt, dtype=np.uint64)
            U = np.zeros(nt * m)
            check(_ffi.lib.f3m_debug_charges(i, sk.ctypes.data, W.ctypes.data, tk.ctypes.data, U.ctypes.data))
            out.append(dict(t=t, P=P, q=q, src_key=sk, W=W.reshape(ns, m), tgt_key=tk, U=U.reshape(nt, m)))
        return out
