"""Problem data model (mirror of reference ``pintoc/problem.py``).

Models here are *descriptions*: each built-in dynamics / cost / constraint
class knows how to describe itself to the CUDA library (``_device_spec``),
where the fused kernels evaluate it.  The per-stage numpy evaluators (``f``,
``fx`` ...) are kept for API compatibility and for simulating a plant; the
solver never calls them.
"""

from __future__ import annotations

import abc
from dataclasses import dataclass

import numpy as np

from .exceptions import DimensionError


def _frozen(a) -> np.ndarray:
    out = np.array(a, dtype=float)
    out.setflags(write=False)
    return out


@dataclass(frozen=True)
class Trajectory:
    """A state sequence of length N+1 paired with N controls
    (reference problem.py:26-56)."""

    states: np.ndarray    # (N+1, d_x)
    controls: np.ndarray  # (N, d_u)

    def __post_init__(self):
        object.__setattr__(self, "states", _frozen(np.atleast_2d(self.states)))
        object.__setattr__(self, "controls", _frozen(np.atleast_2d(self.controls)))
        if self.states.shape[0] != self.controls.shape[0] + 1:
            raise DimensionError(
                f"need len(states) == len(controls) + 1, got {self.states.shape[0]} states "
                f"and {self.controls.shape[0]} controls")
        if not np.all(np.isfinite(self.states)):
            raise DimensionError("trajectory states contain non-finite values")
        if not np.all(np.isfinite(self.controls)):
            raise DimensionError("trajectory controls contain non-finite values")

    @property
    def horizon(self) -> int:
        return self.controls.shape[0]

    @property
    def d_x(self) -> int:
        return self.states.shape[1]

    @property
    def d_u(self) -> int:
        return self.controls.shape[1]


class DynamicsModel(abc.ABC):
    """Discrete map x_{t+1} = f_t(x_t, u_t) (reference problem.py:59-112)."""

    def __init__(self, horizon: int, d_x: int, d_u: int):
        if horizon < 1 or d_x < 1 or d_u < 1:
            raise DimensionError("horizon, d_x and d_u must all be positive")
        self.horizon = horizon
        self.d_x = d_x
        self.d_u = d_u

    @abc.abstractmethod
    def f(self, t: int, x: np.ndarray, u: np.ndarray) -> np.ndarray: ...

    def _device_spec(self) -> dict:
        raise NotImplementedError(
            f"{type(self).__name__} has no device implementation; the B200 solver runs "
            "PendulumDynamics, CartPoleDynamics, LinearDynamics and "
            "TimeVaryingLinearDynamics")


class CostModel(abc.ABC):
    """Stage and terminal cost (reference problem.py:115-164)."""

    @abc.abstractmethod
    def l(self, t: int, x: np.ndarray, u: np.ndarray) -> float: ...

    @abc.abstractmethod
    def terminal(self, x: np.ndarray) -> float: ...


class ConstraintModel(abc.ABC):
    """Stage inequality constraints w = [g(x); h(u)] <= 0
    (reference problem.py:167-230)."""

    n_state: int
    n_control: int

    @property
    def n_total(self) -> int:
        return self.n_state + self.n_control


class BoxConstraint(ConstraintModel):
    """Componentwise bounds stacked as one-sided rows (problem.py:233-340):
    h(u) = [u - ub; lb - u] (likewise for states), infinite bounds dropped."""

    def __init__(self, d_x: int, d_u: int, control_lower=None, control_upper=None,
                 state_lower=None, state_upper=None):
        self.d_x, self.d_u = d_x, d_u
        self.control_lower = self._bound(control_lower, d_u, -np.inf)
        self.control_upper = self._bound(control_upper, d_u, np.inf)
        self.state_lower = self._bound(state_lower, d_x, -np.inf)
        self.state_upper = self._bound(state_upper, d_x, np.inf)
        if np.any(self.control_lower >= self.control_upper) or np.any(
                self.state_lower >= self.state_upper):
            raise DimensionError("box bounds must satisfy lower < upper")
        self._rows = ([(0, i, 1.0, self.state_upper[i]) for i in range(d_x)
                       if np.isfinite(self.state_upper[i])]
                      + [(0, i, -1.0, self.state_lower[i]) for i in range(d_x)
                         if np.isfinite(self.state_lower[i])])
        self.n_state = len(self._rows)
        self._rows += ([(1, i, 1.0, self.control_upper[i]) for i in range(d_u)
                        if np.isfinite(self.control_upper[i])]
                       + [(1, i, -1.0, self.control_lower[i]) for i in range(d_u)
                          if np.isfinite(self.control_lower[i])])
        self.n_control = len(self._rows) - self.n_state

    @staticmethod
    def _bound(value, dim, default):
        if value is None:
            return _frozen(np.full(dim, default))
        return _frozen(np.broadcast_to(np.asarray(value, dtype=float), (dim,)))

    def w_batch(self, xs: np.ndarray, us: np.ndarray) -> np.ndarray:
        """Stacked constraint values (N, n_total) -- input validation helper."""
        n = len(us)
        out = np.empty((n, self.n_total))
        for k, (var, i, s, b) in enumerate(self._rows):
            src = xs[:n, i] if var == 0 else us[:, i]
            out[:, k] = src - b if s > 0 else b - src
        return out

    def max_violation(self, traj: Trajectory) -> float:
        if self.n_total == 0:
            return -np.inf
        return float(self.w_batch(traj.states[:-1], traj.controls).max())

    def clamp_controls(self, controls: np.ndarray, margin: float = 0.0) -> np.ndarray:
        lo, hi = self.control_lower, self.control_upper
        if margin:
            center = np.where(np.isfinite(lo) & np.isfinite(hi), 0.5 * (lo + hi), 0.0)
            lo = np.where(np.isfinite(lo), center + (1 - margin) * (lo - center), lo)
            hi = np.where(np.isfinite(hi), center + (1 - margin) * (hi - center), hi)
        return np.clip(controls, lo, hi)

    def _device_spec(self) -> dict:
        return dict(state_lower=self.state_lower, state_upper=self.state_upper,
                    control_lower=self.control_lower, control_upper=self.control_upper)


class AugmentedCost(abc.ABC):
    """Outer-solver augmentation c_t(x, u) (reference problem.py:343-389).
    On the device it is a tag plus parameters, not a callable."""

    variant: str = "zero"


class ZeroAugmentation(AugmentedCost):
    variant = "zero"


@dataclass(frozen=True)
class ControlProblem:
    """Bundle of the models describing one constrained control problem."""

    dynamics: DynamicsModel
    cost: CostModel
    constraints: ConstraintModel | None = None

    @property
    def horizon(self) -> int:
        return self.dynamics.horizon
