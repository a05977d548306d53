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
    arr = np.asarray(a, dtype=np.float64).copy()
    arr.flags.writeable = False
    return arr


@dataclass(frozen=True)
class Trajectory:
    """A state sequence of length N+1 paired with N controls
    (reference problem.py:26-56)."""

    states: np.ndarray    # (N+1, d_x)
    controls: np.ndarray  # (N, d_u)

    def __post_init__(self):
        for name in ("states", "controls"):
            object.__setattr__(self, name, _frozen(np.atleast_2d(getattr(self, name))))
        n_x, n_u = len(self.states), len(self.controls)
        if n_x != n_u + 1:
            raise DimensionError(
                f"need len(states) == len(controls) + 1, got {n_x} states "
                f"and {n_u} controls")
        for name in ("states", "controls"):
            if not np.isfinite(getattr(self, name)).all():
                raise DimensionError(f"trajectory {name} contain non-finite values")

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
        if min(horizon, d_x, d_u) < 1:
            raise DimensionError("horizon, d_x and d_u must all be positive")
        self.horizon, self.d_x, self.d_u = horizon, d_x, d_u

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
        for name, given, dim, sign in (("control_lower", control_lower, d_u, -1),
                                       ("control_upper", control_upper, d_u, 1),
                                       ("state_lower", state_lower, d_x, -1),
                                       ("state_upper", state_upper, d_x, 1)):
            setattr(self, name, self._bound(given, dim, sign * np.inf))
        if any((lo >= hi).any() for lo, hi in ((self.control_lower, self.control_upper),
                                               (self.state_lower, self.state_upper))):
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
        given = default if value is None else np.asarray(value, dtype=float)
        return _frozen(np.broadcast_to(given, (dim,)))

    def w_batch(self, xs: np.ndarray, us: np.ndarray) -> np.ndarray:
        """Stacked constraint values (N, n_total) -- input validation helper."""
        n = len(us)
        out = np.empty((n, self.n_total))
        for k, (var, i, s, b) in enumerate(self._rows):
            src = xs[:n, i] if var == 0 else us[:, i]
            out[:, k] = src - b if s > 0 else b - src
        return out

    def max_violation(self, traj: Trajectory) -> float:
        w = self.w_batch(traj.states[:-1], traj.controls)
        return float(w.max()) if w.size else -np.inf

    def clamp_controls(self, controls: np.ndarray, margin: float = 0.0) -> np.ndarray:
        """Clip to the control box shrunk by `margin` about its centre
        (problem.py:326-340; one-sided boxes shrink about 0)."""
        bounds = [self.control_lower, self.control_upper]
        if margin:
            two_sided = np.isfinite(bounds[0]) & np.isfinite(bounds[1])
            mid = np.where(two_sided, 0.5 * (bounds[0] + bounds[1]), 0.0)
            bounds = [np.where(np.isfinite(b), mid + (1 - margin) * (b - mid), b)
                      for b in bounds]
        return np.clip(controls, bounds[0], bounds[1])

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
