"""CPU checks of the boundary: libf3m.so builds for sm_100a, loads, and exports every
symbol include/f3m.h declares; host-side config defaults; no compute calls (no GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "f3m.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"F3M_API\s+[\w\s\*]+?\b(f3m_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("f3m_matvec", "f3m_direct", "f3m_default_config", "f3m_plan_create", "f3m_plan_bbox",
              "f3m_plan_leaves", "f3m_plan_set_leaves", "f3m_plan_s2m", "f3m_plan_evaluate", "f3m_plan_destroy", "f3m_last_error"):
        assert s in syms


def test_library_builds_loads_and_exports_every_symbol():
    import importlib.util
    # by path: importing the package would need the library this test builds
    spec = importlib.util.spec_from_file_location("_f3m_build", os.path.join(ROOT, "paper_2202_01085_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    lib = b.build()
    L = ctypes.CDLL(lib)
    for s in declared_symbols():
        assert hasattr(L, s), f"{s} declared in include/f3m.h but not exported"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_config_and_errors_without_gpu():
    import paper_2202_01085_b200 as f3m
    from paper_2202_01085_b200 import _ffi
    c = _ffi.default_config(3)
    assert (c.nodes_per_dim, c.node_cap, c.eta, c.rho, c.zeta, c.max_depth, c.flags) == (4, 2048, 0.5, 128, 64, 21, 0)
    c7 = _ffi.default_config(7)
    assert c7.zeta == 4 ** 7 and c7.max_depth == 9
    with pytest.raises(f3m.F3MError) as e:
        _ffi.check(_ffi.lib.f3m_default_config(9, ctypes.byref(_ffi.Config())))
    assert e.value.status == 2
    # invalid spec is rejected before any device work
    k = _ffi.Kernel(0, -1.0)
    st = _ffi.lib.f3m_matvec(None, 10, None, 10, 3, None, None, ctypes.byref(k), None, None, None, None)
    assert st == 5


def test_product_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2202_01085_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "f3m_oracle" not in txt, f
