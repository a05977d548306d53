"""Trajectory-level operations on the device (reference problem.py:449-486)."""

from __future__ import annotations

import numpy as np

from . import _native as N
from ._device import DeviceSolver, SolveSettings
from .exceptions import DimensionError, DivergenceError, InfeasibleError
from .newton import aug_settings
from .problem import AugmentedCost, CostModel, DynamicsModel, Trajectory
from .systems import QuadraticCost


def _zero_cost(dyn: DynamicsModel) -> QuadraticCost:
    return QuadraticCost(np.zeros((dyn.d_x, dyn.d_x)), np.zeros((dyn.d_u, dyn.d_u)),
                         np.zeros((dyn.d_x, dyn.d_x)))


def rollout(model: DynamicsModel, x1, controls, dtype=None) -> Trajectory:
    """States from x1 under ``controls`` (problem.py:449-473), on the device.

    Raises DivergenceError at the first non-finite state, DimensionError on
    shape mismatch."""
    x1 = np.asarray(x1, dtype=float).reshape(-1)
    controls = np.atleast_2d(np.asarray(controls, dtype=float))
    if x1.shape[0] != model.d_x:
        raise DimensionError(f"x1 has dimension {x1.shape[0]}, model wants {model.d_x}")
    if controls.shape != (model.horizon, model.d_u):
        raise DimensionError(f"controls shape {controls.shape} does not match "
                             f"(N, d_u) = ({model.horizon}, {model.d_u})")
    solver = DeviceSolver(model, _zero_cost(model), None, 1, SolveSettings(), dtype=dtype)
    states = np.zeros((model.horizon + 1, model.d_x))
    states[0] = x1
    solver.load(states[None], controls[None])
    solver.rollout()
    bad = int(solver.read("bad_index")[0])
    if bad >= 0:
        raise DivergenceError(bad)
    xs = solver.field("states", solver.T + 1, (solver.nx,))[0].cpu().numpy()
    return Trajectory(xs, controls)


def total_cost(cost: CostModel, aug: AugmentedCost | None, traj: Trajectory, dyn=None,
               dtype=None) -> float:
    """Augmented objective (problem.py:476-486), on the device.  ``dyn`` is any
    built-in model with the trajectory's dimensions (only used for shapes)."""
    from .systems import LinearDynamics
    if dyn is None:
        dyn = LinearDynamics(np.eye(traj.d_x), np.zeros((traj.d_x, traj.d_u)), traj.horizon)
    st = aug_settings(aug)
    con = getattr(aug, "constraints", None)
    solver = DeviceSolver(dyn, cost, con, 1, SolveSettings(method=N.METHOD_NEWTON, **st),
                          dtype=dtype)
    z = v = None
    if st["aug"] == N.AUG_ADMM:
        z, v = np.asarray(aug.z, float)[None], np.asarray(aug.v, float)[None]
    solver.load(traj.states[None], traj.controls[None], z, v)
    solver.total_cost()
    if st["aug"] == N.AUG_BARRIER:
        bad = int(solver.read("bad_index")[0])
        if bad >= 0:
            stage, comp = divmod(bad, max(1, solver.W))
            w = con.w_batch(traj.states[:-1], traj.controls)
            raise InfeasibleError(stage, comp, float(w[stage, comp]))
    return float(solver.read("cur_cost")[0])
