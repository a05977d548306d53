"""Constrained outer loops (mirror of reference ``pintoc/outer.py``).

Both loops run entirely on the device: when a problem's Newton solve
finishes, a per-stage kernel records the round (barrier) or performs the
ADMM projection / dual update with fused residual maxima, and a per-problem
kernel shrinks mu or tests the ADMM residuals and restarts Newton.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._device import DeviceSolver, SolveSettings
from .exceptions import InfeasibleError
from .newton import (NewtonOptions, NewtonReport, check_consistent_result, history_records,
                     plan_chunks, raise_status, rollout_mode)
from .problem import AugmentedCost, ConstraintModel, ControlProblem, Trajectory


class BarrierAugmentation(AugmentedCost):
    """-mu * sum(log(-g) + log(-h))  (outer.py:30-157), evaluated on device."""

    variant = "barrier"

    def __init__(self, constraints: ConstraintModel, mu: float):
        if mu <= 0:
            raise ValueError("barrier parameter mu must be > 0")
        self.constraints = constraints
        self.mu = float(mu)


def barrier_augmentation(constraints, mu):
    return BarrierAugmentation(constraints, mu)


class AdmmAugmentation(AugmentedCost):
    """(rho/2) ||w(x,u) - z_t + v_t/rho||^2  (outer.py:252-333), on device."""

    variant = "admm"

    def __init__(self, constraints: ConstraintModel, rho: float, z, v):
        if rho <= 0:
            raise ValueError("penalty parameter rho must be > 0")
        self.constraints = constraints
        self.rho = float(rho)
        self.z = np.asarray(z, dtype=float)
        self.v = np.asarray(v, dtype=float)
        if self.z.shape != self.v.shape:
            raise ValueError("z and v must have matching shapes")


def admm_augmentation(constraints, rho, z, v):
    return AdmmAugmentation(constraints, rho, z, v)


def project_box(point, constraints=None):
    """Projection onto {y <= 0}: componentwise clamp (outer.py:341-348)."""
    return np.minimum(np.asarray(point, dtype=float), 0.0)


def assert_strictly_feasible(constraints: ConstraintModel, traj: Trajectory) -> None:
    """Input validation of outer.py:163-177 (host check of the caller's data).
    Constraints that only evaluate on the device (DeviceConstraint) are
    checked there instead: the barrier solve's first cost evaluation raises
    InfeasibleError(stage, component, value) at the first violated row."""
    from .usermodel import DeviceConstraint
    if isinstance(constraints, DeviceConstraint):
        return
    w = constraints.w_batch(traj.states[:-1], traj.controls)
    st, comp = np.nonzero(w >= 0)
    if len(st):
        items = [f"stage {t} component {c}: {w[t, c]:.6g}" for t, c in zip(st[:10], comp[:10])]
        listing = "; ".join(items)
        if len(st) > 10:
            listing += f"; ... ({len(st)} total)"
        raise InfeasibleError(int(st[0]), int(comp[0]), float(w[st[0], comp[0]]),
                              f"trajectory is not strictly feasible: {listing}")


@dataclass(frozen=True)
class BarrierOptions:
    mu0: float = 0.1
    zeta: float = 0.2
    mu_tol: float = 1e-4
    newton: NewtonOptions = field(default_factory=NewtonOptions)

    def __post_init__(self):
        if self.mu0 <= 0:
            raise ValueError("mu0 must be > 0")
        if not 0 < self.zeta < 1:
            raise ValueError("zeta must lie in (0, 1)")
        if self.mu_tol <= 0:
            raise ValueError("mu_tol must be > 0")

    def rounds(self) -> int:
        mu, n = self.mu0, 0
        while mu > self.mu_tol:
            n += 1
            mu *= self.zeta
        return n


@dataclass(frozen=True)
class BarrierRound:
    mu: float
    cost: float
    controls: np.ndarray
    newton: NewtonReport


@dataclass(frozen=True)
class BarrierReport:
    rounds: tuple

    @property
    def outer_iterations(self) -> int:
        return len(self.rounds)

    @property
    def inner_iterations(self) -> int:
        return sum(r.newton.iterations for r in self.rounds)

    @property
    def converged(self) -> bool:
        return all(r.newton.converged for r in self.rounds)


@dataclass(frozen=True)
class AdmmOptions:
    rho: float = 1.0
    residual_tol: float = 1e-2
    max_outer: int = 200
    newton: NewtonOptions = field(default_factory=NewtonOptions)

    def __post_init__(self):
        if self.rho <= 0:
            raise ValueError("rho must be > 0")
        if self.residual_tol <= 0:
            raise ValueError("residual_tol must be > 0")
        if self.max_outer < 1:
            raise ValueError("max_outer must be >= 1")


@dataclass(frozen=True)
class AdmmState:
    z: np.ndarray
    v: np.ndarray
    primal_residual: float
    dual_residual: float


@dataclass(frozen=True)
class AdmmReport:
    outer_iterations: int
    converged: bool
    state: AdmmState
    residual_history: tuple
    newton_reports: tuple

    @property
    def inner_iterations(self) -> int:
        return sum(r.iterations for r in self.newton_reports)


def _newton_reports(solver: DeviceSolver, b: int, n_rounds: int, hist_cap: int):
    iters = solver.rounds("round_iters")[:, b].cpu().numpy()
    terms = solver.rounds("round_term")[:, b].cpu().numpy()
    costs = solver.rounds("round_cost")[:, b].cpu().numpy()
    hist = solver.history()[:, :, b].cpu().numpy() if hist_cap else np.zeros((0, 5))
    out, start = [], 0
    for r in range(n_rounds):
        k = int(iters[r])
        avail = max(0, min(k, hist.shape[0] - start))
        out.append(NewtonReport(iterations=k, final_cost=float(costs[r]),
                                history=history_records(hist, start, avail),
                                termination=N.TERM_NAMES[int(terms[r])]))
        start += k
    return out


def barrier_solve(problem: ControlProblem, initial: Trajectory,
                  opts: BarrierOptions | None = None, dtype=None,
                  keep_history: bool = True) -> tuple[Trajectory, BarrierReport]:
    """Primal log-barrier method (outer.py:221-245), every round on device."""
    if problem.constraints is None:
        raise ValueError("barrier_solve needs a ConstraintModel on the problem")
    opts = opts or BarrierOptions()
    assert_strictly_feasible(problem.constraints, initial)
    n_rounds = opts.rounds()
    if n_rounds == 0:
        return initial, BarrierReport(())
    nw = opts.newton
    c0, c1 = plan_chunks(nw.executor, problem.horizon)
    hist_cap = n_rounds * nw.max_iters if keep_history else 0
    settings = SolveSettings(method=N.METHOD_BARRIER, alpha0=nw.alpha0, nu0=nw.nu0,
                             inner_tol=nw.inner_tol, max_iters=nw.max_iters, mu0=opts.mu0,
                             zeta=opts.zeta, mu_tol=opts.mu_tol, hist_cap=hist_cap,
                             round_cap=n_rounds, keep_round_controls=True, chunk0=c0, chunk=c1,
                             rollout=rollout_mode(nw.executor))
    solver = DeviceSolver(problem.dynamics, problem.cost, problem.constraints, 1, settings,
                          dtype=dtype)
    solver.load(initial.states[None], initial.controls[None])
    check_consistent_result(solver.check_consistency())
    solver.run()
    raise_status(solver, solver.read("status").cpu().numpy())
    done = int(solver.read("round")[0])
    mus = solver.rounds("round_mu")[:, 0].cpu().numpy()
    ctrl = solver.read("round_controls").view(n_rounds, solver.nu, solver.T, 1)
    ctrl = ctrl[..., 0].permute(0, 2, 1).cpu().numpy()
    reports = _newton_reports(solver, 0, done, hist_cap)
    rounds = tuple(BarrierRound(float(mus[r]), reports[r].final_cost, ctrl[r].copy(), reports[r])
                   for r in range(done))
    xs = solver.states()[0].cpu().numpy()
    us = solver.controls()[0].cpu().numpy()
    return Trajectory(xs, us), BarrierReport(rounds)


def admm_solve(problem: ControlProblem, initial: Trajectory, opts: AdmmOptions | None = None,
               dtype=None, keep_history: bool = False) -> tuple[Trajectory, AdmmReport]:
    """ADMM operator splitting (outer.py:392-435), every outer step on device."""
    if problem.constraints is None:
        raise ValueError("admm_solve needs a ConstraintModel on the problem")
    opts = opts or AdmmOptions()
    nw = opts.newton
    c0, c1 = plan_chunks(nw.executor, problem.horizon)
    hist_cap = opts.max_outer * nw.max_iters if keep_history else 0
    settings = SolveSettings(method=N.METHOD_ADMM, alpha0=nw.alpha0, nu0=nw.nu0,
                             inner_tol=nw.inner_tol, max_iters=nw.max_iters, rho=opts.rho,
                             residual_tol=opts.residual_tol, max_outer=opts.max_outer,
                             hist_cap=hist_cap, round_cap=opts.max_outer, chunk0=c0, chunk=c1,
                             rollout=rollout_mode(nw.executor))
    solver = DeviceSolver(problem.dynamics, problem.cost, problem.constraints, 1, settings,
                          dtype=dtype)
    solver.load(initial.states[None], initial.controls[None])
    check_consistent_result(solver.check_consistency())
    solver.run()
    raise_status(solver, solver.read("status").cpu().numpy())
    done = int(solver.read("round")[0])
    rp = solver.rounds("round_rp")[:done, 0].cpu().numpy()
    rd = solver.rounds("round_rd")[:done, 0].cpu().numpy()
    residuals = tuple((float(a), float(b)) for a, b in zip(rp, rd))
    reports = tuple(_newton_reports(solver, 0, done, hist_cap))
    W = solver.W
    z = solver.field("z", solver.T, (W,))[0].cpu().numpy() if W else np.zeros((solver.T, 0))
    v = solver.field("v", solver.T, (W,))[0].cpu().numpy() if W else np.zeros((solver.T, 0))
    converged = bool(done and rp[-1] <= opts.residual_tol and rd[-1] <= opts.residual_tol)
    state = AdmmState(z, v, residuals[-1][0] if done else 0.0, residuals[-1][1] if done else 0.0)
    xs = solver.states()[0].cpu().numpy()
    us = solver.controls()[0].cpu().numpy()
    return Trajectory(xs, us), AdmmReport(done, converged, state, residuals, reports)
