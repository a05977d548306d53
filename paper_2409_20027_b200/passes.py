"""Pass-level API (mirror of reference ``pintoc/passes.py``).

``value_pass`` + ``propagation_pass`` together are the LQR-scan solve of
one Newton subproblem; on the device they are one call (``LqrSolver``) that
runs the blocked reverse scan over dual value elements, the gains, and the
blocked forward scan over closed-loop maps.  ``costate_pass`` and
``hamiltonian_expansion`` run the fused co-state / expansion kernels.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace
from typing import NamedTuple

import numpy as np

from . import _native as N
from ._device import DeviceSolver, SolveSettings
from .exceptions import ConditioningError, DefinitenessError
from .newton import aug_settings, plan_chunks
from .problem import Trajectory


class CostateElement(NamedTuple):
    """Adjoint segment (dl/dx, dc/dx, df/dx)  (passes.py:30-35)."""
    dl: np.ndarray  # (d_x,)
    dc: np.ndarray  # (d_x,)
    df: np.ndarray  # (d_x, d_x)


class ValueElement(NamedTuple):
    """Dual parameterisation (A, Y, C, eta, b)  (passes.py:38-45)."""
    A: np.ndarray
    Y: np.ndarray
    C: np.ndarray
    eta: np.ndarray
    b: np.ndarray


class RolloutElement(NamedTuple):
    """Affine map dx -> F dx + e  (passes.py:48-52)."""
    F: np.ndarray
    e: np.ndarray


class FeedbackLaw(NamedTuple):
    """du_t = Gamma_t dx_t + gamma_t  (passes.py:55-59)."""
    Gamma: np.ndarray  # (N, d_u, d_x)
    gamma: np.ndarray  # (N, d_u)


@dataclass(frozen=True)
class StageExpansion:
    """Second-order data of the subproblem (passes.py:62-97)."""
    P: np.ndarray
    R: np.ndarray
    M: np.ndarray
    d: np.ndarray
    Fx: np.ndarray
    Fu: np.ndarray
    P_terminal: np.ndarray
    alpha: float
    R_reg: np.ndarray

    @property
    def horizon(self) -> int:
        return self.P.shape[0]

    @property
    def d_x(self) -> int:
        return self.P.shape[1]

    @property
    def d_u(self) -> int:
        return self.R.shape[1]

    def with_alpha(self, alpha: float) -> "StageExpansion":
        if alpha < 0:
            raise ValueError("alpha must be nonnegative")
        return replace(self, alpha=alpha, R_reg=self.R + alpha * np.eye(self.d_u))

    @staticmethod
    def build(P, R, M, d, Fx, Fu, P_terminal, alpha=0.0) -> "StageExpansion":
        R = np.asarray(R, float)
        return StageExpansion(np.asarray(P, float), R, np.asarray(M, float),
                              np.asarray(d, float), np.asarray(Fx, float),
                              np.asarray(Fu, float), np.asarray(P_terminal, float),
                              float(alpha), R + alpha * np.eye(R.shape[1]))


FLAG_DEF_R, FLAG_DEF_Q, FLAG_COND = 1, 2, 4


class LqrSolver:
    """Batched LQR-scan solver on device tensors in SoA batch-minor layout.

    Inputs (torch, device, dtype float32/float64): P (nx*nx, T, B),
    R (nu*nu, T, B), M (nx*nu, T, B), d (nu, T, B), Fx (nx*nx, T, B),
    Fu (nx*nu, T, B), PT (nx*nx, 1, B), alpha (float64, B).
    """

    def __init__(self, batch, horizon, nx, nu, dtype=None, chunk0=0, chunk=0,
                 with_value=False, device=None):
        torch = N.require_cuda()
        self.torch = torch
        self.lib = N.load_library()
        self.B, self.T, self.nx, self.nu = int(batch), int(horizon), int(nx), int(nu)
        self.dtype = dtype or torch.float64
        self.code = N.PTC_F64 if self.dtype == torch.float64 else N.PTC_F32
        if not self.lib.ptc_supported(self.code, -1, self.nx, self.nu):
            raise N.NativeError(f"LQR kernels not compiled for nx={nx} nu={nu}")
        self.chunk0, self.chunk = int(chunk0), int(chunk)
        dev = torch.device(device or "cuda")
        self.device = dev
        nbytes = self.lib.ptc_lqr_workspace_bytes(self.code, self.B, self.T, self.nx, self.nu,
                                                  self.chunk0, self.chunk)
        N.check(0 if nbytes >= 0 else int(nbytes))
        self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
        B, T, nx_, nu_ = self.B, self.T, self.nx, self.nu
        mk = lambda *s: torch.empty(*s, dtype=self.dtype, device=dev)
        self.Gamma = mk(nu_ * nx_, T, B)
        self.gamma = mk(nu_, T, B)
        self.dx = mk(nx_, T + 1, B)
        self.du = mk(nu_, T, B)
        self.S = mk(nx_ * nx_, T + 1, B) if with_value else None
        self.s = mk(nx_, T + 1, B) if with_value else None
        self.flags = torch.zeros(B, dtype=torch.int32, device=dev)

    def plan(self):
        k0, k, lv = C.c_int(), C.c_int(), C.c_int()
        N.check(self.lib.ptc_lqr_plan(self.B, self.T, self.nx, self.chunk0, self.chunk, C.byref(k0),
                                      C.byref(k), C.byref(lv)))
        return k0.value, k.value, lv.value

    def solve_rows(self, rows, PT, alpha, stream=None):
        """One long problem (batch 1, nx >= 8, horizon >= 1024) from stage rows
        (T, SC): [P | R | M | d | Fx | Fu] per stage (ptc_lqr_solve_rows)."""
        self.flags.zero_()
        ptr = lambda t: None if t is None else t.data_ptr()
        N.check(self.lib.ptc_lqr_solve_rows(
            self.code, self.T, self.nx, self.nu, ptr(rows), ptr(PT), ptr(alpha), ptr(self.S),
            ptr(self.s), ptr(self.Gamma), ptr(self.gamma), ptr(self.dx), ptr(self.du),
            ptr(self.flags), ptr(self.workspace), self.workspace.numel(), self.chunk0,
            self.chunk, N.stream_ptr(stream)))

    def solve(self, P, R, M, d, Fx, Fu, PT, alpha, stream=None):
        self.flags.zero_()
        ptr = lambda t: None if t is None else t.data_ptr()
        N.check(self.lib.ptc_lqr_solve(
            self.code, self.B, self.T, self.nx, self.nu,
            ptr(P), ptr(R), ptr(M), ptr(d), ptr(Fx), ptr(Fu), ptr(PT), ptr(alpha),
            ptr(self.S), ptr(self.s), ptr(self.Gamma), ptr(self.gamma), ptr(self.dx),
            ptr(self.du), ptr(self.flags), ptr(self.workspace), self.workspace.numel(),
            self.chunk0, self.chunk, N.stream_ptr(stream)))


class HostLqrSolver:
    """The same batched LQR-scan solve on HOST tensors (``ptc_lqr_solve_host``):
    inputs and outputs are CPU tensors in the LqrSolver layouts (pin them
    for asynchronous copies, and keep them referenced until ``stream`` is
    synchronised: torch's pinned-memory cache does not see these copies);
    the host->device copies (only the parts the kernels read), the solve
    and the device->host copies are enqueued on ``stream``, so calls on
    several streams overlap PCIe with compute.

    ``stacked=True`` takes the reference's per-problem arrays stacked over
    the batch instead (``ptc_lqr_solve_host_stacked``): P (B, T, nx, nx),
    R (B, T, nu, nu), M (B, T, nx, nu), d (B, T, nu), Fx (B, T, nx, nx),
    Fu (B, T, nx, nu), PT (B, nx, nx); outputs Gamma (B, T, nu, nx),
    gamma (B, T, nu), dx (B, T + 1, nx), du (B, T, nu) -- restacked on the
    device, no host transpose."""

    def __init__(self, batch, horizon, nx, nu, dtype=None, chunk0=0, chunk=0, device=None,
                 stacked=False):
        self.stacked = bool(stacked)
        torch = N.require_cuda()
        self.torch = torch
        self.lib = N.load_library()
        self.B, self.T, self.nx, self.nu = int(batch), int(horizon), int(nx), int(nu)
        self.dtype = dtype or torch.float64
        self.code = N.PTC_F64 if self.dtype == torch.float64 else N.PTC_F32
        if not self.lib.ptc_supported(self.code, -1, self.nx, self.nu):
            raise N.NativeError(f"LQR kernels not compiled for nx={nx} nu={nu}")
        self.chunk0, self.chunk = int(chunk0), int(chunk)
        wsb = (self.lib.ptc_lqr_host_stacked_workspace_bytes if self.stacked
               else self.lib.ptc_lqr_host_workspace_bytes)
        nbytes = wsb(self.code, self.B, self.T, self.nx, self.nu, self.chunk0, self.chunk)
        N.check(0 if nbytes >= 0 else int(nbytes))
        self.workspace = torch.empty(int(nbytes), dtype=torch.uint8,
                                     device=torch.device(device or "cuda"))

    def outputs(self, pin=True):
        """Host output tensors Gamma, gamma, dx, du (pinned by default)."""
        torch = self.torch
        B, T, nx, nu = self.B, self.T, self.nx, self.nu
        mk = lambda *s: torch.empty(*s, dtype=self.dtype, pin_memory=pin)
        if self.stacked:
            return mk(B, T, nu, nx), mk(B, T, nu), mk(B, T + 1, nx), mk(B, T, nu)
        return mk(nu * nx, T, B), mk(nu, T, B), mk(nx, T + 1, B), mk(nu, T, B)

    def solve(self, P, R, M, d, Fx, Fu, PT, alpha, out, flags=None, stream=None):
        ins = (P, R, M, d, Fx, Fu, PT)
        if any(t.is_cuda for t in ins + tuple(out)) or alpha.is_cuda:
            raise ValueError("HostLqrSolver takes host tensors (use LqrSolver for device ones)")
        if not all(t.is_contiguous() for t in ins + tuple(out)):
            raise ValueError("HostLqrSolver takes contiguous tensors")
        B, T, nx, nu = self.B, self.T, self.nx, self.nu
        want = (nx * nx * T * B, nu * nu * T * B, nx * nu * T * B, nu * T * B, nx * nx * T * B,
                nx * nu * T * B, nx * nx * B, nu * nx * T * B, nu * T * B, nx * (T + 1) * B,
                nu * T * B)
        for name, t, n in zip(("P", "R", "M", "d", "Fx", "Fu", "PT", "Gamma", "gamma", "dx",
                               "du"), ins + tuple(out), want):
            if t.numel() != n or t.dtype != self.dtype:
                raise ValueError(f"{name}: {t.numel()} {t.dtype} elements, expected {n} "
                                 f"{self.dtype}")
        if alpha.numel() != B or alpha.dtype != self.torch.float64:
            raise ValueError("alpha: float64[batch]")
        ptr = lambda t: None if t is None else t.data_ptr()
        fn = self.lib.ptc_lqr_solve_host_stacked if self.stacked else self.lib.ptc_lqr_solve_host
        N.check(fn(
            self.code, self.B, self.T, self.nx, self.nu, *[ptr(t) for t in ins], ptr(alpha),
            *[ptr(t) for t in out], ptr(flags), ptr(self.workspace), self.workspace.numel(),
            self.chunk0, self.chunk, N.stream_ptr(stream)))


def _soa(torch, a, dtype, device, comps):
    """(T, *comp) numpy -> (prod comp, T, 1) device."""
    t = torch.as_tensor(np.asarray(a, float), dtype=dtype).reshape(a.shape[0], comps)
    return t.t().contiguous().unsqueeze(-1).to(device)


def _raise_gate(solver, exp, dtype, dev):
    """The reference's exception for a flagged solve, with the stage its gates
    name (passes.py:231-241): R + alpha I first, then a singular combine,
    then Q_t (ptc_lqr_diagnose re-runs the exact dual-form recursion)."""
    torch = solver.torch
    n, nx, nu = exp.horizon, exp.d_x, exp.d_u
    args = [_soa(torch, a, dtype, dev, c) for a, c in
            ((exp.P, nx * nx), (exp.R, nu * nu), (exp.M, nx * nu), (exp.d, nu),
             (exp.Fx, nx * nx), (exp.Fu, nx * nu))]
    PT = _soa(torch, exp.P_terminal[None], dtype, dev, nx * nx)
    alpha = torch.full((1,), float(exp.alpha), dtype=torch.float64, device=dev)
    out = torch.empty(3, dtype=torch.int32, device=dev)
    N.check(solver.lib.ptc_lqr_diagnose(solver.code, 1, n, nx, nu,
                                        *[a.data_ptr() for a in args], PT.data_ptr(),
                                        alpha.data_ptr(), out.data_ptr(), N.stream_ptr()))
    first_r, first_q, cond = (int(v) for v in out.cpu())
    if first_r >= 0:
        raise DefinitenessError(first_r, "R + alpha*I")
    if cond:
        raise ConditioningError("singular I + C*Y while combining value elements")
    if first_q >= 0:
        raise DefinitenessError(first_q, "Q")
    # the fused sweep flagged what the exact recursion does not: report the kind
    fl = int(solver.flags[0])
    if fl & FLAG_COND:
        raise ConditioningError("singular I + C*Y while combining value elements")
    raise DefinitenessError(-1, "R + alpha*I" if fl & FLAG_DEF_R else "Q")


def lqr_solve(exp: StageExpansion, executor: str = "auto", dtype=None):
    """value_pass + propagation_pass of one expansion on the device.
    Returns S, s, FeedbackLaw, dxs, dus as numpy (reference shapes)."""
    torch = N.require_cuda()
    dtype = dtype or torch.float64
    n, nx, nu = exp.horizon, exp.d_x, exp.d_u
    c0, c1 = plan_chunks(executor, n)
    solver = LqrSolver(1, n, nx, nu, dtype=dtype, chunk0=c0, chunk=c1, with_value=True)
    dev = solver.device
    alpha = torch.full((1,), float(exp.alpha), dtype=torch.float64, device=dev)
    PT = _soa(torch, exp.P_terminal[None], dtype, dev, nx * nx)
    if nx >= 8 and n >= 1024:
        # the reference's per-stage arrays side by side are the stage rows
        # the wide kernels read: no transpose on either side
        rows = np.concatenate([np.asarray(a, float).reshape(n, -1)
                               for a in (exp.P, exp.R, exp.M, exp.d, exp.Fx, exp.Fu)], axis=1)
        solver.solve_rows(torch.as_tensor(rows, dtype=dtype).to(dev), PT, alpha)
    else:
        args = [_soa(torch, exp.P, dtype, dev, nx * nx), _soa(torch, exp.R, dtype, dev, nu * nu),
                _soa(torch, exp.M, dtype, dev, nx * nu), _soa(torch, exp.d, dtype, dev, nu),
                _soa(torch, exp.Fx, dtype, dev, nx * nx), _soa(torch, exp.Fu, dtype, dev, nx * nu)]
        solver.solve(*args, PT, alpha)
    fl = int(solver.flags[0])
    if fl & (FLAG_DEF_R | FLAG_DEF_Q | FLAG_COND):
        _raise_gate(solver, exp, dtype, dev)
    host = lambda t, shape: t[..., 0].t().reshape(shape).cpu().numpy()
    S = host(solver.S, (n + 1, nx, nx))
    s = host(solver.s, (n + 1, nx))
    law = FeedbackLaw(host(solver.Gamma, (n, nu, nx)), host(solver.gamma, (n, nu)))
    return S, s, law, host(solver.dx, (n + 1, nx)), host(solver.du, (n, nu))


def value_pass(exp: StageExpansion, executor: str = "auto", dtype=None):
    """Cost-to-go (S, s) and the affine control law (passes.py:291-323)."""
    S, s, law, _, _ = lqr_solve(exp, executor, dtype)
    return S, s, law


def propagation_pass(law: FeedbackLaw, exp: StageExpansion, executor: str = "auto",
                     dtype=None):
    """Closed-loop deviations from dx_1 = 0 (passes.py:338-361): the device
    forward scan of ``law`` on the expansion's Jacobians (ptc_propagate)."""
    return propagate(law, exp, dtype=dtype)


def propagate(law: FeedbackLaw, exp: StageExpansion, dtype=None):
    """Forward scan of an arbitrary feedback law (device)."""
    from ._device import propagate_law
    return propagate_law(law, exp, dtype)


def _pass_solver(traj: Trajectory, cost, aug, dyn, alpha, dtype, executor="auto"):
    st = aug_settings(aug)
    con = getattr(aug, "constraints", None)
    c0, c1 = plan_chunks(executor, len(traj.controls))
    settings = SolveSettings(method=N.METHOD_NEWTON, alpha0=float(alpha), chunk0=c0, chunk=c1,
                             **st)
    solver = DeviceSolver(dyn, cost, con, 1, settings, dtype=dtype)
    z = v = None
    if st["aug"] == N.AUG_ADMM:
        z, v = np.asarray(aug.z, float)[None], np.asarray(aug.v, float)[None]
    solver.load(traj.states[None], traj.controls[None], z, v)
    solver.expand()
    return solver


def costate_pass(traj: Trajectory, cost, aug, dyn, executor: str = "auto", dtype=None):
    """Adjoint vectors lambda_{1:N+1} (passes.py:122-148) on the device."""
    solver = _pass_solver(traj, cost, aug, dyn, 0.0, dtype, executor)
    return solver.field("lam", solver.T + 1, (solver.nx,))[0].cpu().numpy()


def hamiltonian_expansion(traj: Trajectory, costates, cost, aug, dyn, alpha: float = 0.0,
                          dtype=None, executor: str = "auto") -> StageExpansion:
    """P, R, M, d, Fx, Fu of the augmented Lagrangian (passes.py:155-185).
    The device kernel fuses the co-state sweep with the expansion, so the
    co-states are recomputed on the fly (``costates`` is accepted for API
    compatibility and must be the output of ``costate_pass``)."""
    if alpha < 0:
        raise ValueError("alpha must be nonnegative")
    solver = _pass_solver(traj, cost, aug, dyn, alpha, dtype, executor)
    T, nx, nu = solver.T, solver.nx, solver.nu
    f = lambda name, shape: solver.field(name, T, shape)[0].cpu().numpy()
    PT = solver.read("PT").view(nx, nx).cpu().numpy()
    return StageExpansion.build(f("P", (nx, nx)), f("R", (nu, nu)), f("M", (nx, nu)),
                                f("d", (nu,)), f("Fx", (nx, nx)), f("Fu", (nx, nu)), PT,
                                alpha)


# ------------------------------------------------------------------ elements
#
# The element-level functions of the reference (one combine at a time) run
# the same device functions the scans use (elements.cuh: velem_from_stage,
# vcombine, aff_compose), batched over items: pass elements whose arrays
# carry a leading item axis to combine many pairs in one launch.

def _items(torch, dtype, dev, fields, dims):
    """Fields with shape (*lead, *dims[k]) -> one device (sum comps, n) tensor."""
    lead = np.asarray(fields[0]).shape[:len(np.asarray(fields[0]).shape) - len(dims[0])]
    n = int(np.prod(lead)) if lead else 1
    parts = [torch.as_tensor(np.asarray(f, dtype=float)).reshape(n, -1) for f in fields]
    return torch.cat(parts, 1).t().contiguous().to(device=dev, dtype=dtype), lead, n


def _split(t, lead, dims):
    out, c0 = [], 0
    host = t.t().double().cpu().numpy()
    for dm in dims:
        c = int(np.prod(dm)) if dm else 1
        out.append(host[:, c0:c0 + c].reshape(tuple(lead) + tuple(dm)))
        c0 += c
    return out


def _ctx(dtype):
    torch = N.require_cuda()
    return torch, N.load_library(), dtype or torch.float64, torch.device("cuda")


def _code(torch, dtype):
    return N.PTC_F64 if dtype == torch.float64 else N.PTC_F32


def costate_boundary(cost, x_final, dtype=None) -> np.ndarray:
    """Terminal adjoint: the terminal cost's gradient Qf (x - goal) (passes.py:106-110)."""
    torch, _, dtype, dev = _ctx(dtype)
    spec = cost._device_spec()
    Qf = torch.as_tensor(np.asarray(spec["Qf"], float), dtype=dtype, device=dev)
    e = torch.as_tensor(np.asarray(x_final, float) - np.asarray(spec["goal"], float),
                        dtype=dtype, device=dev)
    return (Qf @ e).double().cpu().numpy()


def value_element_init(exp: StageExpansion, t: int, dtype=None) -> ValueElement:
    """Dual-form value element of stage t (t == N: the boundary element)
    (passes.py:192-228).  Raises DefinitenessError if R_t + alpha I is not
    positive definite."""
    torch, lib, dtype, dev = _ctx(dtype)
    n, nx, nu = exp.horizon, exp.d_x, exp.d_u
    if not 0 <= t <= n:
        raise IndexError(f"stage {t} outside 0..{n}")
    soa = lambda a, c: _soa(torch, np.asarray(a)[None] if np.ndim(a) == 2 else a, dtype, dev, c)
    PT = soa(exp.P_terminal, nx * nx)
    alpha = torch.full((1,), float(exp.alpha), dtype=torch.float64, device=dev)
    vc = 3 * nx * nx + 2 * nx
    if t == n:
        out = torch.empty(vc, 1, dtype=dtype, device=dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        N.check(lib.ptc_value_elements(_code(torch, dtype), 0, nx, nu, None, None, None, None,
                                       None, None, PT.data_ptr(), alpha.data_ptr(),
                                       out.data_ptr(), flags.data_ptr(), N.stream_ptr()))
        col = out[:, :1]
    else:
        sl = lambda a, c: soa(np.asarray(a)[t:t + 1], c)
        ins = [sl(exp.P, nx * nx), sl(exp.R, nu * nu), sl(exp.M, nx * nu), sl(exp.d, nu),
               sl(exp.Fx, nx * nx), sl(exp.Fu, nx * nu)]
        out = torch.empty(vc, 2, dtype=dtype, device=dev)
        flags = torch.zeros(2, dtype=torch.int32, device=dev)
        N.check(lib.ptc_value_elements(_code(torch, dtype), 1, nx, nu,
                                       *[x.data_ptr() for x in ins], PT.data_ptr(),
                                       alpha.data_ptr(), out.data_ptr(), flags.data_ptr(),
                                       N.stream_ptr()))
        if int(flags[0]) & FLAG_DEF_R:
            raise DefinitenessError(t, "R + alpha*I")
        col = out[:, :1]
    return ValueElement(*_split(col, (), [(nx, nx), (nx, nx), (nx, nx), (nx,), (nx,)]))


def value_combine(left: ValueElement, right: ValueElement, dtype=None) -> ValueElement:
    """Merge adjacent conditional value functions, ``left`` covering the
    earlier stages (passes.py:264-288).  Raises ConditioningError if
    I + C_left Y_right is singular."""
    torch, lib, dtype, dev = _ctx(dtype)
    nx = np.asarray(left.A).shape[-1]
    dims = [(nx, nx), (nx, nx), (nx, nx), (nx,), (nx,)]
    L, lead, n = _items(torch, dtype, dev, list(left), dims)
    Rt, _, _ = _items(torch, dtype, dev, list(right), dims)
    out = torch.empty_like(L)
    flags = torch.zeros(n, dtype=torch.int32, device=dev)
    N.check(lib.ptc_value_combine(_code(torch, dtype), n, nx, L.data_ptr(), Rt.data_ptr(),
                                  out.data_ptr(), flags.data_ptr(), N.stream_ptr()))
    if bool((flags & FLAG_COND).any()):
        raise ConditioningError("singular I + C*Y while combining value elements")
    return ValueElement(*_split(out, lead, dims))


def costate_combine(left: CostateElement, right: CostateElement, dtype=None) -> CostateElement:
    """Compose two adjoint segments, ``left`` covering the earlier stages
    (passes.py:113-119)."""
    torch, lib, dtype, dev = _ctx(dtype)
    nx = np.asarray(left.dl).shape[-1]
    dims = [(nx, nx), (nx,), (nx,)]
    A, lead, n = _items(torch, dtype, dev, [left.df, left.dl, left.dc], dims)
    B, _, _ = _items(torch, dtype, dev, [right.df, right.dl, right.dc], dims)
    out = torch.empty_like(A)
    N.check(lib.ptc_affine_combine(_code(torch, dtype), n, nx, 1, A.data_ptr(), B.data_ptr(),
                                   out.data_ptr(), N.stream_ptr()))
    df, dl, dc = _split(out, lead, dims)
    return CostateElement(dl, dc, df)


def rollout_combine(first: RolloutElement, second: RolloutElement, dtype=None) -> RolloutElement:
    """Compose affine maps, applying ``first`` then ``second`` (passes.py:330-335)."""
    torch, lib, dtype, dev = _ctx(dtype)
    nx = np.asarray(first.e).shape[-1]
    dims = [(nx, nx), (nx,)]
    A, lead, n = _items(torch, dtype, dev, list(first), dims)
    B, _, _ = _items(torch, dtype, dev, list(second), dims)
    out = torch.empty_like(A)
    N.check(lib.ptc_affine_combine(_code(torch, dtype), n, nx, 0, A.data_ptr(), B.data_ptr(),
                                   out.data_ptr(), N.stream_ptr()))
    return RolloutElement(*_split(out, lead, dims))
