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
    assert lib.ptc_lqr_plan(65536, 256, 4, 0, 0, ctypes.byref(k0), ctypes.byref(k),
                            ctypes.byref(lv)) == 0
    assert k0.value == 256 and lv.value == 0          # big batch: one sweep per problem
    assert lib.ptc_lqr_plan(1, 1 << 16, 4, 0, 0, ctypes.byref(k0), ctypes.byref(k),
                            ctypes.byref(lv)) == 0
    assert lv.value >= 3 and k.value == 4             # long horizon: log-depth tree
    assert lib.ptc_lqr_plan(1, 1 << 16, 12, 0, 0, ctypes.byref(k0), ctypes.byref(k),
                            ctypes.byref(lv)) == 0
    assert (k0.value, k.value) == (16, 4)             # warp kernels: narrow tree


def test_solver_path_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2409_20027_b200 as P
    dyn = P.LinearDynamics(np.eye(2), np.ones((2, 1)), horizon=4)
    with pytest.raises(P.NativeUnavailable):
        P.rollout(dyn, np.zeros(2), np.zeros((4, 1)))


def test_argument_errors_are_reported_without_touching_the_device():
    """Invalid arguments come back as PTC_ERR_ARG / PTC_ERR_UNSUPPORTED with a
    message, before any device work (so this runs on a GPU-less host)."""
    from paper_2409_20027_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    lib = _native.load_library()
    F64 = _native.PTC_F64
    null = [None] * 15          # P..PT, alpha, S..du, flags
    # bad dims
    rc = lib.ptc_lqr_solve(F64, 0, 10, 4, 2, *null, None, 0, 0, 0, None)
    assert rc == -1 and b"bad dims" in lib.ptc_last_error()
    # unsupported kernel set
    rc = lib.ptc_lqr_solve(F64, 1, 10, 5, 5, *null, None, 0, 0, 0, None)
    assert rc == -2 and b"not instantiated" in lib.ptc_last_error()
    # unknown dtype
    rc = lib.ptc_lqr_solve(7, 1, 10, 4, 2, *null, None, 0, 0, 0, None)
    assert rc == -1
    # time-block phases
    vc, pc = ctypes.c_int(), ctypes.c_int()
    assert lib.ptc_lqr_block_comps(12, ctypes.byref(vc), ctypes.byref(pc)) == 0
    assert (vc.value, pc.value) == (3 * 144 + 24, 144 + 12)
    args = [None] * 16 + [None, None, 0, 0, 0, None]
    assert lib.ptc_lqr_block_solve(3, F64, 1, 10, 4, 2, 0, 1, 0, 1, *args) == -1   # phase
    assert lib.ptc_lqr_block_solve(0, F64, 1, 10, 4, 2, 0, 1, 2, 2, *args) == -1   # rank
    assert lib.ptc_lqr_block_solve(1, F64, 1, 10, 4, 2, 0, 0, 0, 2, *args) == -1   # blocks_in
    assert lib.ptc_lqr_block_solve(0, F64, 1, 10, 4, 2, 0, 1, 0, 1, *args) == -1   # PT on last
    assert lib.ptc_lqr_block_workspace_bytes(F64, 1, 1 << 12, 12, 4, 0, 0) > \
        lib.ptc_lqr_workspace_bytes(F64, 1, 1 << 12, 12, 4, 0, 0)   # + stage-major staging


def test_solver_descriptor_validation_without_gpu():
    """ptc_solver_workspace_bytes sizes the solver from the descriptor alone
    and rejects dimension / model combinations that are not compiled in."""
    import numpy as np
    from paper_2409_20027_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    lib = _native.load_library()
    d = _native.ProblemDesc()
    d.dtype, d.batch, d.horizon, d.nx, d.nu = _native.PTC_F64, 4, 64, 2, 1
    d.model = _native.DYN_PENDULUM
    Q = np.eye(2)
    R = np.eye(1)
    d.Q, d.R, d.Qf = Q.ctypes.data, R.ctypes.data, Q.ctypes.data
    d.max_iters, d.hist_cap, d.round_cap = 10, 10, 1
    small = lib.ptc_solver_workspace_bytes(ctypes.byref(d))
    d.batch = 400
    assert lib.ptc_solver_workspace_bytes(ctypes.byref(d)) > small > 0


def test_user_model_source_and_library():
    """The user-model hook's generated source (usermodel.model_source) and,
    when build() has compiled them, the test models' libraries exporting the
    one hook the main library binds (ptc_user_model_ops)."""
    import ctypes
    import os
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from user_models import PEND_HESS, PEND_JAC, PEND_STEP

    from paper_2409_20027_b200 import usermodel
    tag, src = usermodel.model_source(2, 1, PEND_STEP, PEND_JAC, PEND_HESS, "pendulum")
    assert "PTC_USER_MODEL_LIBRARY(2, 1, ptc::UmSrc_" + tag + ")" in src
    assert "kHess = true" in src and PEND_STEP.strip().splitlines()[0] in src
    so = os.path.join(usermodel.MODEL_DIR, f"um_{tag}.so")
    if os.path.exists(so):
        lib = ctypes.CDLL(so)
        assert hasattr(lib, "ptc_user_model_ops")


def test_solver_loop_argument_errors_without_gpu():
    """ptc_solver_loop validates its handle before touching the device."""
    from paper_2409_20027_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    lib = _native.load_library()
    assert lib.ptc_solver_loop(None, 1, 10, None, None) == -1   # PTC_ERR_ARG
    assert b"NULL" in lib.ptc_last_error()
