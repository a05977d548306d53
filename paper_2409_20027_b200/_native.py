"""ctypes binding of the C ABI in include/pintoc_b200.h.

This is the only place the shared library is loaded.  There is no fallback:
if ``_lib/libpintoc_b200.so`` is missing or no CUDA device is present, every
solver entry point raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libpintoc_b200.so")

PTC_F32, PTC_F64 = 0, 1
DYN_PENDULUM, DYN_CARTPOLE, DYN_LINEAR = 0, 1, 2
DYN_USER_BASE = 100
AUG_ZERO, AUG_BARRIER, AUG_ADMM = 0, 1, 2
METHOD_NEWTON, METHOD_BARRIER, METHOD_ADMM = 0, 1, 2
ST_RUNNING, ST_DONE, ST_ERR_STALLED, ST_ERR_INFEASIBLE = 0, 1, -1, -2
TERM_NAMES = {0: "none", 1: "converged_cost", 2: "converged_step", 3: "max_iters", 4: "stalled"}


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a CUDA device) is not available."""


class NativeError(RuntimeError):
    """A C ABI call returned an error code."""


class ProblemDesc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("batch", C.c_int32), ("horizon", C.c_int32),
        ("nx", C.c_int32), ("nu", C.c_int32),
        ("model", C.c_int32),
        ("dyn_params", C.c_double * 8),
        ("lin_a", C.c_void_p), ("lin_b", C.c_void_p), ("lin_c", C.c_void_p),
        ("lin_rows", C.c_int32), ("lin_batch", C.c_int32),
        ("Q", C.c_void_p), ("R", C.c_void_p), ("Qf", C.c_void_p), ("goal", C.c_void_p),
        ("state_lower", C.c_void_p), ("state_upper", C.c_void_p),
        ("control_lower", C.c_void_p), ("control_upper", C.c_void_p),
        ("method", C.c_int32), ("aug", C.c_int32), ("aug_mu", C.c_double),
        ("alpha0", C.c_double), ("nu0", C.c_double), ("inner_tol", C.c_double),
        ("max_iters", C.c_int32),
        ("mu0", C.c_double), ("zeta", C.c_double), ("mu_tol", C.c_double),
        ("rho", C.c_double), ("residual_tol", C.c_double),
        ("max_outer", C.c_int32),
        ("hist_cap", C.c_int32), ("round_cap", C.c_int32),
        ("keep_round_controls", C.c_int32),
        ("chunk0", C.c_int32), ("chunk", C.c_int32),
        ("rollout", C.c_int32),
        ("block_mode", C.c_int32), ("t_base", C.c_int32), ("block_last", C.c_int32),
        ("user_data", C.c_void_p),
        ("cost_params", C.c_double * 8), ("cost_data", C.c_void_p),
        ("con_rows_state", C.c_int32), ("con_rows_control", C.c_int32),
        ("con_params", C.c_double * 8), ("con_data", C.c_void_p),
    ]


_lib = None
_lock = threading.Lock()

_SIGS = {
    "ptc_last_error": (C.c_char_p, []),
    "ptc_version": (C.c_int, []),
    "ptc_supported": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "ptc_lqr_workspace_bytes": (C.c_int64, [C.c_int] * 7),
    "ptc_lqr_solve": (C.c_int, [C.c_int] * 5 + [C.c_void_p] * 7 + [C.c_void_p]
                      + [C.c_void_p] * 6 + [C.c_void_p, C.c_void_p, C.c_int64,
                                             C.c_int, C.c_int, C.c_void_p]),
    "ptc_lqr_plan": (C.c_int, [C.c_int] * 5 + [C.POINTER(C.c_int)] * 3),
    "ptc_propagate": (C.c_int, [C.c_int] * 5 + [C.c_void_p] * 7
                      + [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p]),
    "ptc_lqr_block_comps": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ptc_lqr_block_workspace_bytes": (C.c_int64, [C.c_int] * 7),
    "ptc_lqr_block_solve": (C.c_int, [C.c_int] * 10 + [C.c_void_p] * 16
                            + [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p]),
    "ptc_solver_workspace_bytes": (C.c_int64, [C.POINTER(ProblemDesc)]),
    "ptc_solver_create": (C.c_int, [C.POINTER(ProblemDesc), C.c_void_p, C.c_int64,
                                    C.POINTER(C.c_void_p)]),
    "ptc_solver_destroy": (C.c_int, [C.c_void_p]),
    "ptc_solver_load": (C.c_int, [C.c_void_p] * 5 + [C.c_int, C.c_void_p]),
    "ptc_solver_check_consistency": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ptc_lqr_host_workspace_bytes": (C.c_int64, [C.c_int] * 7),
    "ptc_lqr_solve_host": (C.c_int, [C.c_int] * 5 + [C.c_void_p] * 7 + [C.c_void_p]
                           + [C.c_void_p] * 4 + [C.c_void_p, C.c_void_p, C.c_int64, C.c_int,
                                                  C.c_int, C.c_void_p]),
    "ptc_lqr_host_stacked_workspace_bytes": (C.c_int64, [C.c_int] * 7),
    "ptc_lqr_solve_host_stacked": (C.c_int, [C.c_int] * 5 + [C.c_void_p] * 7 + [C.c_void_p]
                                   + [C.c_void_p] * 4 + [C.c_void_p, C.c_void_p, C.c_int64,
                                                          C.c_int, C.c_int, C.c_void_p]),
    "ptc_value_elements": (C.c_int, [C.c_int] * 4 + [C.c_void_p] * 7
                           + [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ptc_value_combine": (C.c_int, [C.c_int] * 3 + [C.c_void_p] * 5),
    "ptc_affine_combine": (C.c_int, [C.c_int] * 4 + [C.c_void_p] * 4),
    "ptc_lqr_block_solve_rows": (C.c_int, [C.c_int] * 9 + [C.c_void_p] * 3
                                 + [C.c_void_p] * 2 + [C.c_void_p] * 6
                                 + [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                    C.c_void_p]),
    "ptc_lqr_solve_rows": (C.c_int, [C.c_int] * 4 + [C.c_void_p] * 3 + [C.c_void_p] * 6
                           + [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p]),
    "ptc_solver_iterate": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "ptc_solver_block_phase": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "ptc_solver_running": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_void_p]),
    "ptc_solver_running_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ptc_solver_loop": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "ptc_solver_expand": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ptc_solver_lqr": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ptc_solver_rollout": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ptc_solver_total_cost": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ptc_solver_buffer_info": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int32)]),
    "ptc_solver_read": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64, C.c_int,
                                  C.c_void_p]),
    "ptc_solver_write": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64, C.c_int,
                                   C.c_void_p]),
    "ptc_model_load": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(C.c_int)]),
    "ptc_lqr_diagnose": (C.c_int, [C.c_int] * 5 + [C.c_void_p] * 7
                         + [C.c_void_p, C.c_void_p, C.c_void_p]),
}


def load_library(path: str = LIB_PATH):
    """Load (once) and return the ctypes handle; raises NativeUnavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"CUDA library {path} not built; run `python -m paper_2409_20027_b200._build`")
        try:
            lib = C.CDLL(path)
        except OSError as err:
            raise NativeUnavailable(f"cannot load {path}: {err}") from err
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(rc: int) -> None:
    if rc != 0:
        msg = load_library().ptc_last_error().decode()
        raise NativeError(f"pintoc_b200 error {rc}: {msg}")


def require_cuda():
    """Return torch with a CUDA device, or raise NativeUnavailable."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the pintoc_b200 solver runs on the GPU only")
    load_library()
    return torch


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
