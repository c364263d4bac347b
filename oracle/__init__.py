"""F^3M oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/f3m_oracle.cpp``: a plain, single-threaded fp64 CPU
implementation of F^3M (App. F Algorithm 1) and of the exact direct
KMVM.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package; the product package
``paper_2202_01085_b200`` never does, and the two share no code.

Every function is pinned in ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "f3m_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

# flags (same meaning as include/f3m.h F3M_* flags; defined independently here)
EXACT, NO_SMOOTH, NO_ADAPTIVE, NO_SMALL, NO_DROP, MAXNORM, KEEP_EMPTY = 1, 2, 4, 8, 16, 32, 64
TAG_NEAR, TAG_FAR, TAG_FAR_DROPPED, TAG_SMOOTH, TAG_SMALL = 0, 1, 2, 3, 4
STAT_NAMES = ("M", "expanded", "m_far", "m_far_dropped", "m_smooth", "m_small", "m_near",
              "boxes_x", "boxes_y", "empty_x", "empty_y", "pfar")

BUILD_CMD = ["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17", "-shared", "-fPIC",
             "-o", _LIB, _SRC]


def build(force: bool = False) -> str:
    """Compile the oracle (plain g++, no OpenMP/SIMD flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(BUILD_CMD)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        i64, i32, dbl = C.c_int64, C.c_int, C.c_double
        L.orc_last_error.restype = C.c_char_p
        L.orc_cheb_nodes.argtypes = [i32, P]
        L.orc_bary_weights.argtypes = [i32, P]
        L.orc_basis.argtypes = [i32, dbl, P]
        L.orc_tensor_basis.argtypes = [i32, i32, P, P]
        L.orc_box_index.argtypes = [P, i32, i32, dbl, P]
        L.orc_box_index.restype = i64
        L.orc_direct.argtypes = [P, i64, P, i64, i32, P, dbl, P]
        L.orc_f3m_run.argtypes = [P, i64, P, i64, i32, P, dbl, i32, dbl, i64, i64, i32, C.c_uint, i64, i64, i32,
                                  C.POINTER(C.c_void_p)]
        L.orc_sparse_size.argtypes = [i32, i32]
        L.orc_sparse_size.restype = i64
        L.orc_sparse_nodes.argtypes = [i32, i32, P]
        L.orc_sparse_basis.argtypes = [i32, i32, P, P]
        L.orc_cube_f32.argtypes = [P, i64, i32, P, P]
        L.orc_keys_f32.argtypes = [P, i64, i32, i32, dbl, P, P]
        L.orc_s2m_box_f32.argtypes = [P, P, i64, i32, i32, i32, i32, dbl, P, P, P]
        L.orc_free.argtypes = [P]
        L.orc_free.restype = None
        L.orc_get_v.argtypes = [P, P]
        L.orc_get_scalars.argtypes = [P, P]
        L.orc_num_points.argtypes = [P, i32]
        L.orc_num_points.restype = i64
        L.orc_get_keys.argtypes = [P, i32, P]
        L.orc_get_perm.argtypes = [P, i32, P]
        L.orc_get_stats.argtypes = [P, P]
        L.orc_num_boxes.argtypes = [P, i32, i32]
        L.orc_num_boxes.restype = i64
        L.orc_get_boxes.argtypes = [P, i32, i32, P, P, P]
        L.orc_num_pairs.argtypes = [P, i32]
        L.orc_num_pairs.restype = i64
        L.orc_get_pairs.argtypes = [P, i32, P, P, P]
        L.orc_num_charge_sets.argtypes = [P]
        L.orc_charge_info.argtypes = [P, i32, P]
        L.orc_get_charges.argtypes = [P, i32, P, P, P, P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    """fp32 (or any) input -> contiguous fp64 (exact for fp32 inputs)."""
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


def _check(st: int):
    if st != 0:
        raise OracleError(st, lib().orc_last_error().decode())


def cheb_nodes(P: int) -> np.ndarray:
    s = np.zeros(P)
    _check(lib().orc_cheb_nodes(P, _ptr(s)))
    return s


def bary_weights(P: int) -> np.ndarray:
    w = np.zeros(P)
    _check(lib().orc_bary_weights(P, _ptr(w)))
    return w


def basis(P: int, t: float) -> np.ndarray:
    L = np.zeros(P)
    _check(lib().orc_basis(P, float(t), _ptr(L)))
    return L


def tensor_basis(D: int, P: int, tau) -> np.ndarray:
    tau = _f64(tau)
    out = np.zeros(P ** D)
    _check(lib().orc_tensor_basis(D, P, _ptr(tau), _ptr(out)))
    return out


def box_index(x, t: int, E: float, alpha) -> int:
    x = _f64(x)
    alpha = _f64(alpha)
    return int(lib().orc_box_index(_ptr(x), len(x), t, float(E), _ptr(alpha)))


def sparse_nodes(D: int, q: int) -> np.ndarray:
    """Nodes H of the level-q Smolyak sparse grid (reading R27) as finest-grid integer coordinates
    [|H| x D] (1-D finest grid: the 2^q + 1 Chebyshev points), ascending linear index."""
    L = lib()
    n = L.orc_sparse_size(D, q)
    if n < 0:
        raise OracleError(5, "bad sparse grid")
    out = np.zeros((n, D), dtype=np.int64)
    _check(L.orc_sparse_nodes(D, q, _ptr(out)))
    return out


def sparse_basis(D: int, q: int, tau) -> np.ndarray:
    """Phi_h(tau) for every node h of the level-q sparse grid, tau in [-1, 1]^D."""
    tau = _f64(np.atleast_1d(tau))
    L = lib()
    out = np.zeros(L.orc_sparse_size(D, q))
    _check(L.orc_sparse_basis(D, q, _ptr(tau), _ptr(out)))
    return out


def direct(X, b, gamma: float, Y=None) -> np.ndarray:
    """Exact fp64 KMVM v = k(X, Y) b; Y=None means Y = X."""
    X = _f64(X)
    b = _f64(b)
    nx, D = X.shape
    Yp = None
    ny = nx
    if Y is not None:
        Y = _f64(Y)
        ny = Y.shape[0]
        Yp = _ptr(Y)
    v = np.zeros(nx)
    _check(lib().orc_direct(_ptr(X), nx, Yp, ny, D, _ptr(b), float(gamma), _ptr(v)))
    return v


def subset_error(v_hat, v_exact) -> tuple[float, float]:
    """(err2, err): the paper's squared relative error ||v^-v||^2/||v||^2
    and the plain relative L2 error (reading R16)."""
    vh = np.asarray(v_hat, dtype=np.float64)
    ve = np.asarray(v_exact, dtype=np.float64)
    num = float(np.sum((vh - ve) ** 2))
    den = float(np.sum(ve ** 2))
    return num / den, (num / den) ** 0.5


@dataclass
class F3MResult:
    v: np.ndarray
    E: float
    t_star: int
    T_sort: int
    depth_reached: int
    alphaX: np.ndarray
    alphaY: np.ndarray
    n_near_flushed: int
    keys: list = field(default_factory=list)      # [X keys, Y keys] per original point (uint64)
    perm: list = field(default_factory=list)      # [pi_X, pi_Y] sorted position -> original index
    stats: dict = field(default_factory=dict)     # name -> int64[64] per depth
    boxes: dict = field(default_factory=dict)     # (side, t) -> (key, start, count)
    pairs: dict = field(default_factory=dict)     # t -> (key_p, key_q, tag)
    charges: list = field(default_factory=list)   # dicts t, P, src_key, W, tgt_key, U


def f3m(X, b, gamma: float, P: int = 4, eta: float = 0.5, rho: int | None = None,
        zeta: int | None = None, Y=None, max_depth: int = -1, flags: int = 0,
        node_cap: int = 2048, details: bool = True, n_eval: int = 0, sparse_level: int = 0) -> F3MResult:
    """Run the oracle F^3M (defaults per SURVEY 8: rho = 2 P^D, zeta = P^D).

    n_eval > 0: subset-target mode -- the whole tree and every charge as usual, v computed only
    for the first n_eval rows of X (the rest of v is 0)."""
    X = _f64(X)
    b = _f64(b)
    nx, D = X.shape
    m = P ** D
    rho = 2 * m if rho is None else rho
    zeta = m if zeta is None else zeta
    Yp = None
    ny = nx
    if Y is not None:
        Y = _f64(Y)
        ny = Y.shape[0]
        Yp = _ptr(Y)
    h = C.c_void_p()
    L = lib()
    _check(L.orc_f3m_run(_ptr(X), nx, Yp, ny, D, _ptr(b), float(gamma), P, float(eta), int(rho), int(zeta),
                         int(max_depth), flags, int(node_cap), int(n_eval), int(sparse_level), C.byref(h)))
    try:
        v = np.zeros(nx)
        L.orc_get_v(h, _ptr(v))
        sc = np.zeros(19)
        L.orc_get_scalars(h, _ptr(sc))
        res = F3MResult(v=v, E=sc[0], t_star=int(sc[1]), T_sort=int(sc[2]), depth_reached=int(sc[3]),
                        alphaX=sc[4:4 + D].copy(), alphaY=sc[11:11 + D].copy(), n_near_flushed=int(sc[18]))
        if details and res.T_sort >= 1 and not (flags & EXACT) and res.E > 0:
            st = np.zeros(12 * 64, dtype=np.int64)
            L.orc_get_stats(h, _ptr(st))
            res.stats = {k: st[i * 64:(i + 1) * 64].copy() for i, k in enumerate(STAT_NAMES)}
            for side in (0, 1):
                n = L.orc_num_points(h, side)
                k = np.zeros(n, dtype=np.uint64)
                p = np.zeros(n, dtype=np.int64)
                L.orc_get_keys(h, side, _ptr(k))
                L.orc_get_perm(h, side, _ptr(p))
                res.keys.append(k)
                res.perm.append(p)
                for t in range(res.T_sort + 1):
                    nb = L.orc_num_boxes(h, side, t)
                    bk = np.zeros(nb, dtype=np.uint64)
                    bs = np.zeros(nb, dtype=np.int64)
                    bc = np.zeros(nb, dtype=np.int64)
                    L.orc_get_boxes(h, side, t, _ptr(bk), _ptr(bs), _ptr(bc))
                    res.boxes[(side, t)] = (bk, bs, bc)
            for t in range(res.T_sort + 1):
                npairs = L.orc_num_pairs(h, t)
                kp = np.zeros(npairs, dtype=np.uint64)
                kq = np.zeros(npairs, dtype=np.uint64)
                tg = np.zeros(npairs, dtype=np.int32)
                if npairs:
                    L.orc_get_pairs(h, t, _ptr(kp), _ptr(kq), _ptr(tg))
                res.pairs[t] = (kp, kq, tg)
            for i in range(L.orc_num_charge_sets(h)):
                info = np.zeros(6, dtype=np.int64)
                L.orc_charge_info(h, i, _ptr(info))
                t, Pn, ns, nt, mm, q = (int(x) for x in info)
                sk = np.zeros(ns, dtype=np.uint64)
                W = np.zeros(ns * mm)
                tk = np.zeros(nt, dtype=np.uint64)
                U = np.zeros(nt * mm)
                L.orc_get_charges(h, i, _ptr(sk), _ptr(W), _ptr(tk), _ptr(U))
                res.charges.append(dict(t=t, P=Pn, q=q, src_key=sk, W=W.reshape(ns, mm), tgt_key=tk,
                                        U=U.reshape(nt, mm)))
        return res
    finally:
        L.orc_free(h)


def _f32c(a) -> np.ndarray:
    a = a.numpy() if hasattr(a, "numpy") else np.asarray(a)
    return np.ascontiguousarray(a, dtype=np.float32)


def cube_f32(X):
    """Step 2 on fp32 points without an fp64 copy: (alpha [D], E)."""
    X = _f32c(X)
    n, D = X.shape
    alpha = np.zeros(D)
    E = np.zeros(1)
    _check(lib().orc_cube_f32(_ptr(X), n, D, _ptr(alpha), _ptr(E)))
    return alpha, float(E[0])


def keys_f32(X, T: int, E: float, alpha) -> np.ndarray:
    """Order key (nested Morton, reading R13) of every point at depth T, uint32 (D T <= 32)."""
    X = _f32c(X)
    n, D = X.shape
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    k = np.zeros(n, dtype=np.uint32)
    _check(lib().orc_keys_f32(_ptr(X), n, D, int(T), float(E), _ptr(alpha), _ptr(k)))
    return k


def s2m_box_f32(X, b, P: int, T: int, t: int, E: float, alpha, cell) -> np.ndarray:
    """Stage-1 charges W [P^D] of the single depth-t source box with integer cell coords `cell`."""
    X = _f32c(X)
    b = _f32c(b)
    n, D = X.shape
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    cell = np.ascontiguousarray(cell, dtype=np.int64)
    W = np.zeros(P ** D)
    _check(lib().orc_s2m_box_f32(_ptr(X), _ptr(b), n, D, P, int(T), int(t), float(E), _ptr(alpha), _ptr(cell),
                                 _ptr(W)))
    return W
