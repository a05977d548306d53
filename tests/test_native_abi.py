"""CPU checks of the C-ABI boundary: the in-tree library loads without a GPU
and exports every entry point include/pintoc_b200.h declares (no compute)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pintoc_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ptc_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("ptc_lqr_solve", "ptc_propagate", "ptc_solver_create", "ptc_solver_iterate",
                     "ptc_solver_read", "ptc_solver_expand"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2409_20027_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built (run python -m paper_2409_20027_b200._build)")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    # the ctypes binding covers exactly the declared surface
    assert set(_native.exported_symbols()) == set(declared_functions())


def test_library_reports_instantiated_kernel_sets():
    from paper_2409_20027_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    lib = _native.load_library()
    assert lib.ptc_version() >= 100
    for dt in (_native.PTC_F32, _native.PTC_F64):
        assert lib.ptc_supported(dt, _native.DYN_PENDULUM, 2, 1) == 1
        assert lib.ptc_supported(dt, _native.DYN_CARTPOLE, 4, 1) == 1
        for nx, nu in ((2, 1), (4, 2), (8, 4), (12, 6), (12, 4), (1, 3), (3, 3)):
            assert lib.ptc_supported(dt, -1, nx, nu) == 1, (dt, nx, nu)
            assert lib.ptc_supported(dt, _native.DYN_LINEAR, nx, nu) == 1
    assert lib.ptc_supported(_native.PTC_F64, _native.DYN_PENDULUM, 4, 1) == 0


def test_workspace_queries_without_gpu():
    from paper_2409_20027_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    lib = _native.load_library()
    small = lib.ptc_lqr_workspace_bytes(_native.PTC_F64, 1, 1 << 10, 4, 2, 0, 0)
    big = lib.ptc_lqr_workspace_bytes(_native.PTC_F64, 1, 1 << 16, 4, 2, 0, 0)
    assert 0 < small < big
    assert lib.ptc_lqr_workspace_bytes(_native.PTC_F64, 0, 10, 4, 2, 0, 0) < 0
    k0, k, lv = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert lib.ptc_lqr_plan(65536, 256, 0, 0, ctypes.byref(k0), ctypes.byref(k),
                            ctypes.byref(lv)) == 0
    assert k0.value == 256 and lv.value == 0          # big batch: one sweep per problem
    assert lib.ptc_lqr_plan(1, 1 << 16, 0, 0, ctypes.byref(k0), ctypes.byref(k),
                            ctypes.byref(lv)) == 0
    assert lv.value >= 3                              # long horizon: log-depth tree


def test_solver_path_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2409_20027_b200 as P
    dyn = P.LinearDynamics(np.eye(2), np.ones((2, 1)), horizon=4)
    with pytest.raises(P.NativeUnavailable):
        P.rollout(dyn, np.zeros(2), np.zeros((4, 1)))
