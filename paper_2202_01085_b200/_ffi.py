"""ctypes binding of libf3m.so (include/f3m.h).  Argument marshalling only: every step of
the F^3M path runs in the library's sm_100a kernels.  There is no CPU fallback: if the
shared library is missing or cannot be loaded, importing this module raises."""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libf3m.so")

F3M_OK, F3M_ERR_INVALID_INPUT, F3M_ERR_RESOURCE, F3M_ERR_INTERNAL = 0, 2, 3, 4
F3M_ERR_INVALID_SPEC, F3M_ERR_GRID_TOO_LARGE, F3M_ERR_CUDA = 5, 6, 7
EXACT, NO_SMOOTH, NO_ADAPTIVE, NO_SMALL, NO_DROP, ADMISSIBLE_MAXNORM, KEEP_EMPTY = 1, 2, 4, 8, 16, 32, 64
# the FFM(GPU) / F^2.5M / F^3M ablations of Tables 5-6
FFM_GPU = KEEP_EMPTY | NO_SMOOTH | NO_ADAPTIVE | NO_SMALL
F25M = NO_SMOOTH | NO_ADAPTIVE
MAX_LEVELS = 64


class Kernel(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lengthscale", C.c_double)]


class Config(C.Structure):
    _fields_ = [("nodes_per_dim", C.c_int32), ("node_cap", C.c_int32), ("eta", C.c_double),
                ("rho", C.c_int64), ("zeta", C.c_int64), ("max_depth", C.c_int32), ("flags", C.c_uint32),
                ("sparse_level", C.c_int32)]


_L64 = C.c_int64 * MAX_LEVELS


class Stats(C.Structure):
    _fields_ = [("depth_reached", C.c_int32), ("t_star", C.c_int32), ("t_sort", C.c_int32),
                ("num_sort_passes", C.c_int32), ("E", C.c_double),
                ("M", _L64), ("expanded", _L64), ("m_far", _L64), ("m_far_dropped", _L64), ("m_smooth", _L64),
                ("m_small", _L64), ("m_near", _L64), ("boxes_x", _L64), ("boxes_y", _L64), ("empty_x", _L64),
                ("empty_y", _L64), ("pfar", _L64), ("n_near_flushed", C.c_int64), ("s2m_points", C.c_int64), ("l2t_points", C.c_int64),
                ("near_pairs", C.c_int64), ("far_groups_local", C.c_int32), ("far_groups_sorted", C.c_int32),
                ("kernel_launches", C.c_int32), ("m2l_grid_groups", C.c_int32), ("m2l_grid_fma", C.c_int64),
                ("m2l_grid_pairs", C.c_int64),
                ("ms_phase", C.c_float * 16)]

    def as_dict(self) -> dict:
        out = {}
        for name, _ in self._fields_:
            val = getattr(self, name)
            if isinstance(val, C.Array):
                val = list(val)
            out[name] = val
        return out


class Allocator(C.Structure):
    _fields_ = [("ctx", C.c_void_p),
                ("alloc", C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)),
                ("free", C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p))]


class F3MError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"f3m status {status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2202_01085_b200.build` "
                          "(nvcc, sm_100a).  There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    i64, i32 = C.c_int64, C.c_int32
    L.f3m_last_error.restype = C.c_char_p
    L.f3m_version.restype = C.c_char_p
    L.f3m_phase_name.restype = C.c_char_p
    L.f3m_phase_name.argtypes = [i32]
    L.f3m_default_config.argtypes = [i32, C.POINTER(Config)]
    L.f3m_matvec.argtypes = [P, i64, P, i64, i32, P, P, C.POINTER(Kernel), C.POINTER(Config), C.POINTER(Allocator),
                             P, C.POINTER(Stats)]
    L.f3m_direct.argtypes = [P, i64, P, i64, i32, P, P, i32, C.POINTER(Kernel), P]
    L.f3m_debug_enable.argtypes = [i32]
    L.f3m_debug_enable.restype = None
    L.f3m_debug_last_perm.argtypes = [i32, P, i64]
    L.f3m_debug_last_keys.argtypes = [i32, P, i64]
    L.f3m_debug_last_perm32.argtypes = [P, i64]
    L.f3m_debug_num_pairs.argtypes = [i32]
    L.f3m_debug_num_pairs.restype = i64
    L.f3m_debug_pairs.argtypes = [i32, P, P, P]
    L.f3m_debug_num_charge_sets.restype = i32
    L.f3m_debug_charge_info.argtypes = [i32, P]
    L.f3m_debug_charges.argtypes = [i32, P, P, P, P]
    if hasattr(L, "f3m_plan_create"):
        L.f3m_plan_create.argtypes = [P, i64, P, i64, P, P, P, i64, i32, C.POINTER(Kernel), C.POINTER(Config),
                                      C.POINTER(Allocator), P, C.POINTER(P)]
        L.f3m_plan_bbox.argtypes = [P, P]
        L.f3m_plan_leaves.argtypes = [P, P, C.POINTER(P), C.POINTER(P), C.POINTER(i64)]
        L.f3m_plan_set_leaves.argtypes = [P, P, P, i64]
        L.f3m_plan_s2m.argtypes = [P, C.POINTER(P), C.POINTER(i64)]
        L.f3m_plan_evaluate.argtypes = [P, P, C.POINTER(Stats)]
        L.f3m_plan_destroy.argtypes = [P]
        L.f3m_plan_destroy.restype = None
    L.f3m_op_create.argtypes = [P, i64, P, i64, i32, C.POINTER(Kernel), C.POINTER(Config), P, C.POINTER(P)]
    L.f3m_op_apply.argtypes = [P, P, P, P, C.POINTER(Stats)]
    L.f3m_op_apply_batch.argtypes = [P, P, i64, i32, P, i64, P, C.POINTER(Stats)]
    L.f3m_op_reuses_plan.argtypes = [P]
    L.f3m_op_reuses_plan.restype = i32
    L.f3m_op_destroy.argtypes = [P]
    L.f3m_op_destroy.restype = None
    return L


lib = _load()


def check(status: int):
    if status != F3M_OK:
        raise F3MError(status, lib.f3m_last_error().decode(errors="replace"))


def default_config(D: int) -> Config:
    c = Config()
    check(lib.f3m_default_config(D, C.byref(c)))
    return c


def phase_names() -> list[str]:
    return [lib.f3m_phase_name(i).decode() for i in range(16) if lib.f3m_phase_name(i)]
