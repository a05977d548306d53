"""Iterative parallel Newton method (mirror of reference ``pintoc/newton.py``).

``newton_solve`` keeps the reference signature and report types; the loop
itself (co-states, expansion, value and propagation scans, rollout, cost,
Levenberg-Marquardt trust-region control) runs on the device, one
``ptc_solver_iterate`` per iteration with no host round trip inside it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._device import DeviceSolver, SolveSettings
from .exceptions import InfeasibleError, SolverStalledError
from .problem import AugmentedCost, CostModel, DynamicsModel, Trajectory, ZeroAugmentation

ALPHA_MAX = 1e12

TERM_COST = "converged_cost"
TERM_STEP = "converged_step"
TERM_MAX_ITERS = "max_iters"
TERM_STALLED = "stalled"

SEQUENTIAL = "sequential"   # one device thread sweeps each horizon
PARALLEL = "parallel"       # blocked scan tree over the horizon
AUTO = "auto"               # plan chosen from (batch, horizon)
EXECUTORS = (SEQUENTIAL, PARALLEL, AUTO)


@dataclass(frozen=True)
class NewtonOptions:
    alpha0: float = 1.0
    nu0: float = 2.0
    inner_tol: float = 1e-8
    max_iters: int = 100
    executor: str = AUTO

    def __post_init__(self):
        if self.alpha0 < 0:
            raise ValueError("alpha0 must be >= 0")
        if self.nu0 <= 1:
            raise ValueError("nu0 must be > 1")
        if self.inner_tol <= 0:
            raise ValueError("inner_tol must be > 0")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.executor not in EXECUTORS:
            raise ValueError(f"executor must be one of {EXECUTORS}")


@dataclass(frozen=True)
class IterationRecord:
    cost: float
    alpha: float
    gain_ratio: float
    step_norm: float
    accepted: bool


@dataclass(frozen=True)
class NewtonReport:
    iterations: int
    final_cost: float
    history: tuple
    termination: str

    @property
    def converged(self) -> bool:
        return self.termination in (TERM_COST, TERM_STEP)

    @property
    def accepted_steps(self) -> int:
        return sum(1 for r in self.history if r.accepted)


def gain_ratio(actual_reduction: float, predicted_reduction: float) -> float:
    """newton.py:93-97 (host helper; the device applies the same rule)."""
    if predicted_reduction <= 0:
        return -math.inf
    return actual_reduction / predicted_reduction


def regularization_update(alpha: float, nu: float, ratio: float):
    """newton.py:100-110 (host helper; the device applies the same rule)."""
    if ratio > 0:
        return alpha * max(1.0 / 3.0, 1.0 - (2.0 * ratio - 1.0) ** 3), 2.0, True
    return alpha * nu, 2.0 * nu, False


def predicted_reduction(dus, d, alpha: float) -> float:
    dus = np.asarray(dus, float)
    d = np.asarray(d, float)
    return 0.5 * float(alpha * np.sum(dus * dus) - np.sum(dus * d))


def rollout_mode(executor: str) -> int:
    """Candidate-rollout schedule of an executor: the parallel executor uses
    the log-depth Newton rollout on tree plans, the sequential one the plain
    recurrence, auto decides by horizon (see ptc_problem_desc.rollout)."""
    return {SEQUENTIAL: 1, PARALLEL: 2}.get(executor, 0)


def plan_chunks(executor: str, horizon: int) -> tuple[int, int]:
    if executor == SEQUENTIAL:
        return horizon, 0
    if executor == PARALLEL:
        return 4, 8
    return 0, 0


def aug_settings(aug: AugmentedCost | None) -> dict:
    """Device tag + parameters of an augmentation object."""
    if aug is None or isinstance(aug, ZeroAugmentation) or aug.variant == "zero":
        return dict(aug=N.AUG_ZERO)
    if aug.variant == "barrier":
        return dict(aug=N.AUG_BARRIER, aug_mu=float(aug.mu))
    if aug.variant == "admm":
        return dict(aug=N.AUG_ADMM, rho=float(aug.rho))
    raise ValueError(f"unsupported augmentation {aug!r}")


def _traj_arrays(initial: Trajectory):
    return initial.states[None], initial.controls[None]


def history_records(hist: np.ndarray, start: int, count: int) -> tuple:
    """hist: (cap, 5) numpy for one problem."""
    out = []
    for k in range(start, start + count):
        c, a, r, s, acc = hist[k]
        out.append(IterationRecord(float(c), float(a), float(r), float(s), bool(acc > 0.5)))
    return tuple(out)


def check_consistent_result(bad: np.ndarray) -> None:
    for b, t in enumerate(bad):
        if t >= 0:
            raise ValueError(
                f"initial trajectory is not dynamically consistent at step {int(t)}"
                + (f" (problem {b})" if len(bad) > 1 else "") + "; build it with rollout()")


def raise_status(solver: DeviceSolver, status: np.ndarray, states=None, controls=None) -> None:
    """Turn device error codes into the reference exceptions."""
    for b, st in enumerate(status):
        if st == N.ST_ERR_STALLED:
            alpha = float(solver.read("alpha")[b])
            raise SolverStalledError(f"subproblem unsolvable with alpha={alpha:.3e}")
        if st == N.ST_ERR_INFEASIBLE:
            bad = int(solver.read("bad_index")[b])
            W = max(1, solver.W)
            stage, comp = divmod(bad, W)
            raise InfeasibleError(stage, comp, float(solver.read("bad_value")[b]))


def newton_solve(dyn: DynamicsModel, cost: CostModel, aug: AugmentedCost | None,
                 initial: Trajectory, opts: NewtonOptions | None = None,
                 dtype=None, constraints=None) -> tuple[Trajectory, NewtonReport]:
    """Minimise the augmented objective over controls from ``initial``
    (newton.py:129-215).  Raises SolverStalledError / InfeasibleError /
    ValueError exactly where the reference does."""
    opts = opts or NewtonOptions()
    st = aug_settings(aug)
    con = constraints if constraints is not None else getattr(aug, "constraints", None)
    c0, c1 = plan_chunks(opts.executor, dyn.horizon)
    settings = SolveSettings(method=N.METHOD_NEWTON, alpha0=opts.alpha0, nu0=opts.nu0,
                             inner_tol=opts.inner_tol, max_iters=opts.max_iters,
                             hist_cap=opts.max_iters, round_cap=1, chunk0=c0, chunk=c1,
                             rollout=rollout_mode(opts.executor), **st)
    solver = DeviceSolver(dyn, cost, con, 1, settings, dtype=dtype)
    X, U = _traj_arrays(initial)
    z = v = None
    if st["aug"] == N.AUG_ADMM:
        z = np.asarray(aug.z, float)[None]
        v = np.asarray(aug.v, float)[None]
    solver.load(X, U, z, v)
    check_consistent_result(solver.check_consistency())
    solver.run()
    status = solver.read("status").cpu().numpy()
    raise_status(solver, status)
    xs = solver.states()[0].cpu().numpy()
    us = solver.controls()[0].cpu().numpy()
    it = int(solver.read("iters")[0])
    hist = solver.history()[:, :, 0].cpu().numpy()
    term = N.TERM_NAMES[int(solver.rounds("round_term")[0, 0])]
    cost_v = float(solver.read("cur_cost")[0])
    report = NewtonReport(iterations=it, final_cost=cost_v,
                          history=history_records(hist, 0, min(it, hist.shape[0])),
                          termination=term)
    return Trajectory(xs, us), report
