"""Benchmark systems (mirror of reference ``pintoc/systems.py``).

Conventions match the reference: pendulum state (theta, omega) with the
upright goal at the origin; cart-pole state (pos, theta, vel, omega) with
theta = 0 the pole-down equilibrium.  The device kernels implementing these
models are in csrc/models.cuh; the numpy ``f`` methods here simulate a plant
on the host (MPC loop) and are never used by the solver.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from ._native import DYN_CARTPOLE, DYN_LINEAR, DYN_PENDULUM
from .exceptions import DimensionError
from .problem import BoxConstraint, ControlProblem, CostModel, DynamicsModel, _frozen

SYSTEMS = ("pendulum", "cartpole")


@dataclass(frozen=True)
class PendulumParams:
    gravity: float = 9.81
    length: float = 1.0
    mass: float = 1.0
    damping: float = 1e-3
    dt: float = 0.01
    torque_limit: float = 5.0

    def __post_init__(self):
        for name in ("gravity", "length", "mass", "damping", "dt", "torque_limit"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")


def pendulum_step(state, control, params: PendulumParams) -> np.ndarray:
    """One Euler step of the damped torque-driven pendulum (systems.py:161)."""
    theta, omega = float(state[0]), float(state[1])
    tau = float(np.asarray(control, dtype=float).reshape(-1)[0])
    p = params
    acc = -(p.gravity / p.length) * math.sin(theta) + (tau - p.damping * omega) / (
        p.mass * p.length ** 2)
    return np.array([theta + p.dt * omega, omega + p.dt * acc])


def pendulum_energy(state, params: PendulumParams) -> float:
    theta, omega = state
    return 0.5 * omega ** 2 + (params.gravity / params.length) * (1.0 - math.cos(theta))


class PendulumDynamics(DynamicsModel):
    def __init__(self, horizon: int, params: PendulumParams | None = None):
        super().__init__(horizon, 2, 1)
        self.params = params if params is not None else PendulumParams()

    def f(self, t, x, u):
        return pendulum_step(x, u, self.params)

    def _device_spec(self):
        p = self.params
        return dict(model=DYN_PENDULUM,
                    dyn_params=[p.gravity, p.length, p.mass, p.damping, p.dt])


@dataclass(frozen=True)
class CartPoleParams:
    gravity: float = 9.81
    pole_length: float = 0.5
    cart_mass: float = 10.0
    pole_mass: float = 1.0
    dt: float = 0.01
    force_limit: float = 60.0

    def __post_init__(self):
        for name in ("gravity", "pole_length", "cart_mass", "pole_mass", "dt", "force_limit"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")


def cartpole_step(state, control, params: CartPoleParams) -> np.ndarray:
    """One Euler step of the force-driven cart-pole (systems.py:330)."""
    pos, theta, vel, omega = (float(v) for v in state)
    force = float(np.asarray(control, dtype=float).reshape(-1)[0])
    p = params
    s, c = math.sin(theta), math.cos(theta)
    den = p.cart_mass + p.pole_mass * s * s
    cart = (force + p.pole_mass * s * (p.pole_length * omega + p.gravity * c)) / den
    pole = (-force * c - p.pole_mass * p.pole_length * omega ** 2 * c * s
            - (p.cart_mass + p.pole_mass) * p.gravity * s) / (p.pole_length * den)
    return np.array([pos + p.dt * vel, theta + p.dt * omega, vel + p.dt * cart,
                     omega + p.dt * pole])


class CartPoleDynamics(DynamicsModel):
    def __init__(self, horizon: int, params: CartPoleParams | None = None):
        super().__init__(horizon, 4, 1)
        self.params = params if params is not None else CartPoleParams()

    def f(self, t, x, u):
        return cartpole_step(x, u, self.params)

    def _device_spec(self):
        p = self.params
        return dict(model=DYN_CARTPOLE,
                    dyn_params=[p.gravity, p.pole_length, p.cart_mass, p.pole_mass, p.dt])


class LinearDynamics(DynamicsModel):
    """Affine time-invariant map x' = A x + B u + c (systems.py:32-77)."""

    def __init__(self, A, B, horizon: int, offset=None):
        self.A, self.B = (np.asarray(m, dtype=np.float64) for m in (A, B))
        super().__init__(horizon, self.A.shape[0], self.B.shape[1])
        nx, nu = self.d_x, self.d_u
        if (self.A.shape, self.B.shape) != ((nx, nx), (nx, nu)):
            raise DimensionError("A must be (d_x, d_x) and B (d_x, d_u)")
        self.offset = np.asarray(np.zeros(nx) if offset is None else offset, dtype=np.float64)

    def f(self, t, x, u):
        return self.A.dot(x) + self.B.dot(u) + self.offset

    def _device_spec(self):
        return dict(model=DYN_LINEAR, lin_a=self.A.reshape(1, -1), lin_b=self.B.reshape(1, -1),
                    lin_c=self.offset.reshape(1, -1), lin_rows=1)


class TimeVaryingLinearDynamics(DynamicsModel):
    """x_{t+1} = A_t x_t + B_t u_t + c_t with per-stage matrices
    (the configs' random time-varying systems; a user DynamicsModel in the
    reference)."""

    def __init__(self, A, B, offset=None):
        # read-only copies: the device keeps a cached transposed upload
        self.A, self.B = _frozen(A), _frozen(B)
        super().__init__(self.A.shape[0], self.A.shape[1], self.B.shape[2])
        self.offset = _frozen(np.zeros((self.horizon, self.d_x)) if offset is None else offset)

    def f(self, t, x, u):
        return self.A[t] @ x + self.B[t] @ u + self.offset[t]

    def _device_spec(self):
        T, nx, nu = self.horizon, self.d_x, self.d_u
        # stage-major (rows, comps); the device upload transposes on the GPU
        return dict(model=DYN_LINEAR, lin_a=self.A.reshape(T, nx * nx),
                    lin_b=self.B.reshape(T, nx * nu), lin_c=self.offset.reshape(T, nx),
                    lin_rows=T)


class QuadraticCost(CostModel):
    """0.5 (x - g)^T Q (x - g) + 0.5 u^T R u, terminal 0.5 (x - g)^T Qf (x - g)
    (systems.py:80-139)."""

    def __init__(self, Q, R, Q_terminal, x_goal=None):
        self.Q, self.R, self.Qf = (np.atleast_2d(np.asarray(m, dtype=np.float64))
                                   for m in (Q, R, Q_terminal))
        goal = np.zeros(len(self.Q)) if x_goal is None else x_goal
        self.x_goal = np.asarray(goal, dtype=np.float64)

    @staticmethod
    def _half_form(M, v) -> float:
        return 0.5 * float(v @ M @ v)

    def l(self, t, x, u):
        return self._half_form(self.Q, x - self.x_goal) + self._half_form(self.R, u)

    def terminal(self, x):
        return self._half_form(self.Qf, x - self.x_goal)

    def _device_spec(self):
        return dict(Q=self.Q, R=self.R, Qf=self.Qf, goal=self.x_goal)


DEFAULT_WEIGHTS = {
    "pendulum": (np.array([10.0, 1.0]), np.array([0.1])),
    "cartpole": (np.array([10.0, 10.0, 1.0, 1.0]), np.array([0.1])),
}
DEFAULT_TERMINAL_SCALE = 10.0


def swingup_start(system: str) -> np.ndarray:
    starts = {"pendulum": [math.pi, 0.0], "cartpole": [0.0] * 4}
    if system not in starts:
        raise ValueError(f"unknown system {system!r}")
    return np.array(starts[system])


def swingup_goal(system: str, target_position: float = 0.0) -> np.ndarray:
    goals = {"pendulum": [0.0, 0.0], "cartpole": [target_position, math.pi, 0.0, 0.0]}
    if system not in goals:
        raise ValueError(f"unknown system {system!r}")
    return np.array(goals[system])


def make_swingup_problem(system: str, horizon: int, dt: float, q=None, r=None,
                         terminal_scale: float = DEFAULT_TERMINAL_SCALE,
                         target_position: float = 0.0) -> ControlProblem:
    """Swing-up benchmark bundle (systems.py:470-498)."""
    if system not in SYSTEMS:
        raise ValueError(f"unknown system {system!r}; expected one of {SYSTEMS}")
    if horizon < 1:
        raise ValueError("horizon must be >= 1")
    weights = [np.diag(np.asarray(dflt if given is None else given, dtype=np.float64))
               for given, dflt in zip((q, r), DEFAULT_WEIGHTS[system])]
    cost = QuadraticCost(weights[0], weights[1], terminal_scale * weights[0],
                         x_goal=swingup_goal(system, target_position))
    if system == "pendulum":
        dyn: DynamicsModel = PendulumDynamics(horizon, PendulumParams(dt=dt))
        limit = dyn.params.torque_limit
    else:
        dyn = CartPoleDynamics(horizon, CartPoleParams(dt=dt))
        limit = dyn.params.force_limit
    return ControlProblem(dynamics=dyn, cost=cost, constraints=BoxConstraint(
        dyn.d_x, dyn.d_u, control_lower=-limit, control_upper=limit))
