"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py            # all fast cases
    python tests/golden/make_golden.py --slow     # + full config-2 ADMM run

Each case stores its inputs and the reference outputs in ``<case>.npz`` so
that tests (CPU oracle checks and GPU parity checks) never need the reference
at run time.  The reference is imported read-only from
``/root/reference/pkg/src``; nothing of it is copied into this repository.
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))

import pintoc  # noqa: E402  (the reference)
from pintoc import (  # noqa: E402
    AdmmOptions, BarrierOptions, BoxConstraint, CartPoleDynamics, CartPoleParams,
    ControlProblem, DynamicsModel, LinearDynamics, NewtonOptions,
    PendulumDynamics, PendulumParams, QuadraticCost, StageExpansion, ZeroAugmentation,
    admm_solve, barrier_solve, costate_pass, hamiltonian_expansion, newton_solve,
    propagation_pass, rollout, total_cost, value_pass,
)
from pintoc.outer import AdmmAugmentation, BarrierAugmentation  # noqa: E402

from oracle.pintoc_oracle import random_lqr_expansion  # noqa: E402  (input generator only)


class TVLinear(DynamicsModel):
    """User-defined time-varying affine model plugged into the reference API."""

    def __init__(self, A, B, c):
        super().__init__(A.shape[0], A.shape[1], B.shape[2])
        self.A, self.B, self.c = A, B, c

    def f(self, t, x, u):
        return self.A[t] @ x + self.B[t] @ u + self.c[t]

    def fx(self, t, x, u):
        return self.A[t]

    def fu(self, t, x, u):
        return self.B[t]

    def fxx(self, t, x, u):
        return np.zeros((self.d_x, self.d_x, self.d_x))

    def fuu(self, t, x, u):
        return np.zeros((self.d_x, self.d_u, self.d_u))

    def fxu(self, t, x, u):
        return np.zeros((self.d_x, self.d_x, self.d_u))

    def fx_batch(self, xs, us):
        return self.A[:len(us)]

    def fu_batch(self, xs, us):
        return self.B[:len(us)]


class CosineCost(pintoc.CostModel):
    """User-defined, non-quadratic cost plugged into the reference API: a
    periodic angle penalty w0 (1 - cos theta) + w1 omega^2 / 2 + r u^2 / 2,
    terminal W0 (1 - cos theta) + W1 omega^2 / 2."""

    def __init__(self, w0, w1, r, W0, W1):
        self.w0, self.w1, self.r, self.W0, self.W1 = w0, w1, r, W0, W1

    def l(self, t, x, u):
        return self.w0 * (1.0 - np.cos(x[0])) + 0.5 * self.w1 * x[1] ** 2 + 0.5 * self.r * u[0] ** 2

    def lx(self, t, x, u):
        return np.array([self.w0 * np.sin(x[0]), self.w1 * x[1]])

    def lu(self, t, x, u):
        return np.array([self.r * u[0]])

    def lxx(self, t, x, u):
        return np.diag([self.w0 * np.cos(x[0]), self.w1])

    def luu(self, t, x, u):
        return np.array([[self.r]])

    def lxu(self, t, x, u):
        return np.zeros((2, 1))

    def terminal(self, x):
        return self.W0 * (1.0 - np.cos(x[0])) + 0.5 * self.W1 * x[1] ** 2

    def terminal_x(self, x):
        return np.array([self.W0 * np.sin(x[0]), self.W1 * x[1]])

    def terminal_xx(self, x):
        return np.diag([self.W0 * np.cos(x[0]), self.W1])


class NormConstraints(pintoc.ConstraintModel):
    """User-defined, nonlinear constraint rows plugged into the reference API:
    g(x) = [omega^2 - wmax^2] <= 0, h(u) = [u^2 - umax^2] <= 0 (curved rows,
    nonzero gxx / huu)."""

    n_state = 1
    n_control = 1

    def __init__(self, wmax, umax):
        self.wmax, self.umax = wmax, umax

    def g(self, t, x):
        return np.array([x[1] ** 2 - self.wmax ** 2])

    def gx(self, t, x):
        return np.array([[0.0, 2.0 * x[1]]])

    def gxx(self, t, x):
        return np.array([[[0.0, 0.0], [0.0, 2.0]]])

    def h(self, t, u):
        return np.array([u[0] ** 2 - self.umax ** 2])

    def hu(self, t, u):
        return np.array([[2.0 * u[0]]])

    def huu(self, t, u):
        return np.array([[[2.0]]])


def rand_spd(rng, n, scale=1.0):
    a = rng.normal(size=(n, n))
    return scale * (a @ a.T + n * np.eye(n))


def exp_arrays(exp):
    return dict(P=exp.P, R=exp.R, M=exp.M, d=exp.d, Fx=exp.Fx, Fu=exp.Fu,
                PT=exp.P_terminal, alpha=np.array(exp.alpha))


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def ulp_nudges(x0, u0):
    """Two copies of the inputs moved by one ulp (up / down)."""
    return [(np.nextafter(x0, np.inf), np.nextafter(u0, np.inf)),
            (np.nextafter(x0, -np.inf), np.nextafter(u0, -np.inf))]


def noise_floor(solve, x0, u0, traj, counts):
    """The reference's own reproducibility: rerun it with the inputs moved by
    one ulp and record how far its final trajectory moves and whether its
    iteration counts change.  GPU parity is judged against this floor."""
    fu = fx = 0.0
    stable = True
    for xp, up in ulp_nudges(x0, u0):
        t2, c2 = solve(xp, up)
        fu = max(fu, float(np.abs(t2.controls - traj.controls).max()
                           / max(1.0, np.abs(traj.controls).max())))
        fx = max(fx, float(np.abs(t2.states - traj.states).max()
                           / max(1.0, np.abs(traj.states).max())))
        stable = stable and list(c2) == list(counts)
    return dict(floor_u=np.array(fu), floor_x=np.array(fx), stable=np.array(stable))


def newton_hist(rep):
    h = np.array([(r.cost, r.alpha, r.gain_ratio, r.step_norm, float(r.accepted))
                  for r in rep.history]).reshape(-1, 5)
    return h


# ---------------------------------------------------------------------------

def case_lqr_small():
    rng = np.random.default_rng(101)
    out = {}
    for i in range(16):
        n = int(rng.integers(1, 41))
        dx = int(rng.integers(1, 4))
        du = int(rng.integers(1, 4))
        alpha = float(rng.uniform(0, 2))
        P = np.stack([rand_spd(rng, dx, 0.5) for _ in range(n)])
        R = np.stack([rand_spd(rng, du, 0.5) for _ in range(n)])
        M = 0.3 * rng.normal(size=(n, dx, du))
        d = rng.normal(size=(n, du))
        Fx = 0.7 * rng.normal(size=(n, dx, dx))
        Fu = rng.normal(size=(n, dx, du))
        PT = rand_spd(rng, dx, 0.5)
        exp = StageExpansion(P=P, R=R, M=M, d=d, Fx=Fx, Fu=Fu, P_terminal=PT,
                             alpha=alpha, R_reg=R + alpha * np.eye(du))
        S, s, law = value_pass(exp)
        dxs, dus = propagation_pass(law, exp)
        for k, v in exp_arrays(exp).items():
            out[f"{i}_{k}"] = v
        out[f"{i}_S"], out[f"{i}_s"] = S, s
        out[f"{i}_Gamma"], out[f"{i}_gamma"] = law.Gamma, law.gamma
        out[f"{i}_dxs"], out[f"{i}_dus"] = dxs, dus
    save("lqr_small", count=np.array(16), **out)


def case_lqr_config1():
    out = {}
    for nx in (2, 4, 8, 12):
        nu = nx // 2
        rng = np.random.default_rng(1000 + nx)
        e = random_lqr_expansion(rng, 64, nx, nu)
        exp = StageExpansion(P=e.P, R=e.R, M=e.M, d=e.d, Fx=e.Fx, Fu=e.Fu,
                             P_terminal=e.PT, alpha=0.0, R_reg=e.R.copy())
        S, s, law = value_pass(exp)
        dxs, dus = propagation_pass(law, exp)
        for k, v in exp_arrays(exp).items():
            out[f"{nx}_{k}"] = v
        out[f"{nx}_S"], out[f"{nx}_s"] = S, s
        out[f"{nx}_Gamma"], out[f"{nx}_gamma"] = law.Gamma, law.gamma
        out[f"{nx}_dxs"], out[f"{nx}_dus"] = dxs, dus
    save("lqr_config1", **out)


def _models():
    pend = PendulumDynamics(24, PendulumParams(damping=0.1, dt=0.05))
    pend_cost = QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]),
                              np.diag([100.0, 10.0]), x_goal=np.zeros(2))
    pend_box = BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0)
    cp = CartPoleDynamics(24, CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                             pole_length=0.5, dt=0.02))
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    cp_cost = QuadraticCost(Q, np.diag([0.01]), 10 * Q,
                            x_goal=np.array([0.0, math.pi, 0.0, 0.0]))
    cp_box = BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0,
                           state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                           state_upper=[1.5, np.inf, np.inf, np.inf])
    return {"pendulum": (pend, pend_cost, pend_box, np.array([math.pi, 0.0])),
            "cartpole": (cp, cp_cost, cp_box, np.array([0.1, 0.3, -0.2, 0.1]))}


def case_passes_models():
    """co-state pass, expansion and total cost on nonlinear models."""
    rng = np.random.default_rng(202)
    out = {}
    for name, (dyn, cost, box, x0) in _models().items():
        us = rng.uniform(-3.0, 3.0, size=(dyn.horizon, 1))
        traj = rollout(dyn, x0, us)
        out[f"{name}_x0"], out[f"{name}_us"], out[f"{name}_xs"] = x0, us, traj.states
        z = np.minimum(box.w_batch(traj.states[:-1], us) + 0.1 * rng.normal(size=(dyn.horizon, box.n_total)), 0)
        v = 0.2 * rng.normal(size=z.shape)
        augs = {"zero": ZeroAugmentation(), "barrier": BarrierAugmentation(box, 0.1),
                "admm": AdmmAugmentation(box, 0.7, z, v)}
        out[f"{name}_z"], out[f"{name}_v"] = z, v
        for an, aug in augs.items():
            lam = costate_pass(traj, cost, aug, dyn)
            exp = hamiltonian_expansion(traj, lam, cost, aug, dyn, alpha=0.5)
            key = f"{name}_{an}"
            out[f"{key}_lam"] = lam
            for k, val in exp_arrays(exp).items():
                out[f"{key}_{k}"] = val
            out[f"{key}_cost"] = np.array(total_cost(cost, aug, traj))
    save("passes_models", **out)


def case_newton_lq():
    rng = np.random.default_rng(303)
    out = {}
    for i in range(6):
        n, dx, du = int(rng.integers(4, 30)), int(rng.integers(1, 4)), int(rng.integers(1, 4))
        A = np.eye(dx) + 0.3 * rng.normal(size=(dx, dx)) / np.sqrt(dx)
        B = rng.normal(size=(dx, du))
        Q, R, Qf = rand_spd(rng, dx, 0.3), rand_spd(rng, du, 0.3), rand_spd(rng, dx, 1.0)
        goal = rng.normal(size=dx)
        x0 = rng.normal(size=dx)
        dyn = LinearDynamics(A, B, horizon=n)
        cost = QuadraticCost(Q, R, Qf, x_goal=goal)
        init = rollout(dyn, x0, np.zeros((n, du)))
        alpha0 = [0.0, 1.0][i % 2]
        traj, rep = newton_solve(dyn, cost, None, init, NewtonOptions(alpha0=alpha0))

        def solve(xp, up, dyn=dyn, cost=cost, alpha0=alpha0, n=n, du=du):
            t, r = newton_solve(dyn, cost, None, rollout(dyn, xp, up),
                                NewtonOptions(alpha0=alpha0))
            return t, [r.iterations]
        fl = noise_floor(solve, x0, np.zeros((n, du)), traj, [rep.iterations])
        for k, v in fl.items():
            out[f"{i}_{k}"] = v
        for k, v in dict(A=A, B=B, Q=Q, R=R, Qf=Qf, goal=goal, x0=x0,
                         alpha0=np.array(alpha0), xs=traj.states, us=traj.controls,
                         hist=newton_hist(rep),
                         term=np.array(rep.termination)).items():
            out[f"{i}_{k}"] = v
    save("newton_lq", count=np.array(6), **out)


def _barrier_record(prefix, traj, rep, out):
    out[f"{prefix}_xs"], out[f"{prefix}_us"] = traj.states, traj.controls
    out[f"{prefix}_mus"] = np.array([r.mu for r in rep.rounds])
    out[f"{prefix}_round_iters"] = np.array([r.newton.iterations for r in rep.rounds])
    out[f"{prefix}_round_term"] = np.array([r.newton.termination for r in rep.rounds])
    out[f"{prefix}_round_cost"] = np.array([r.cost for r in rep.rounds])
    for k, r in enumerate(rep.rounds):
        out[f"{prefix}_hist{k}"] = newton_hist(r.newton)


def case_barrier_pendulum_cfg0():
    """BASELINE config 0: pendulum swing-up, T=100, b=0.1, dt=0.05,
    Q=diag(10,0.1), R=0.01, Qf=diag(100,10), |u|<=5, mu 1e-1 -> 1e-6."""
    T = 100
    dyn = PendulumDynamics(T, PendulumParams(damping=0.1, dt=0.05))
    cost = QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]),
                         x_goal=np.zeros(2))
    box = BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0)
    prob = ControlProblem(dyn, cost, box)
    rng = np.random.default_rng(0)
    u0 = np.clip(rng.standard_normal((T, 1)), -4.5, 4.5)
    x0 = np.array([math.pi, 0.0])
    init = rollout(dyn, x0, u0)
    opts = BarrierOptions(mu0=0.1, zeta=0.1, mu_tol=5e-7, newton=NewtonOptions(max_iters=100))
    t0 = time.perf_counter()
    traj, rep = barrier_solve(prob, init, opts)
    wall = time.perf_counter() - t0
    out = dict(x0=x0, u0=u0, wall_s=np.array(wall))
    _barrier_record("sol", traj, rep, out)

    def solve(xp, up):
        t, r = barrier_solve(prob, rollout(dyn, xp, up), opts)
        return t, [q.newton.iterations for q in r.rounds]
    out.update({"sol_" + k: v for k, v in noise_floor(
        solve, x0, u0, traj, [q.newton.iterations for q in rep.rounds]).items()})
    save("barrier_pendulum_cfg0", **out)


def case_barrier_pendulum_conv():
    """A converging swing-up (reference defaults, N=40, dt=0.05, 300 max
    iterations): every round terminates on the cost test."""
    T = 40
    prob = pintoc.make_swingup_problem("pendulum", T, 0.05)
    rng = np.random.default_rng(42)
    u0 = np.clip(rng.standard_normal((T, 1)), -4.5, 4.5)
    x0 = np.array([math.pi, 0.0])
    opts = BarrierOptions(newton=NewtonOptions(max_iters=300))
    traj, rep = barrier_solve(prob, rollout(prob.dynamics, x0, u0), opts)
    out = dict(x0=x0, u0=u0)
    _barrier_record("sol", traj, rep, out)

    def solve(xp, up):
        t, r = barrier_solve(prob, rollout(prob.dynamics, xp, up), opts)
        return t, [q.newton.iterations for q in r.rounds]
    out.update({"sol_" + k: v for k, v in noise_floor(
        solve, x0, u0, traj, [q.newton.iterations for q in rep.rounds]).items()})
    save("barrier_pendulum_conv", **out)


def case_barrier_tvlinear():
    """config-4 shaped (small T): time-varying linear nx=4, nu=2, |u|<=2."""
    rng = np.random.default_rng(404)
    T, nx, nu = 48, 4, 2
    F = 0.2 * rng.normal(size=(T, nx, nx))
    A = np.eye(nx)[None] + 0.01 * F
    B = np.sqrt(0.1) * rng.normal(size=(T, nx, nu))
    c = np.zeros((T, nx))
    dyn = TVLinear(A, B, c)
    Q = np.diag(rng.uniform(0.1, 10.0, size=nx))
    cost = QuadraticCost(Q, 0.1 * np.eye(nu), Q, x_goal=np.zeros(nx))
    box = BoxConstraint(nx, nu, control_lower=-2.0, control_upper=2.0)
    x0 = rng.normal(size=nx) * 3.0
    u0 = np.clip(0.5 * rng.normal(size=(T, nu)), -1.8, 1.8)
    init = rollout(dyn, x0, u0)
    traj, rep = barrier_solve(ControlProblem(dyn, cost, box), init, BarrierOptions())
    out = dict(A=A, B=B, c=c, Q=Q, x0=x0, u0=u0)
    _barrier_record("sol", traj, rep, out)

    def solve(xp, up):
        t, r = barrier_solve(ControlProblem(dyn, cost, box), rollout(dyn, xp, up),
                             BarrierOptions())
        return t, [q.newton.iterations for q in r.rounds]
    out.update({"sol_" + k: v for k, v in noise_floor(
        solve, x0, u0, traj, [q.newton.iterations for q in rep.rounds]).items()})
    save("barrier_tvlinear", **out)


def case_barrier_pendulum_cosine():
    """A user-defined cost (CosineCost) on the pendulum swing-up (T=40,
    dt 0.05, reference default barrier, 300 iterations per round)."""
    T = 40
    dyn = PendulumDynamics(T, PendulumParams(damping=0.1, dt=0.05))
    cost = CosineCost(10.0, 0.1, 0.01, 100.0, 10.0)
    box = BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0)
    rng = np.random.default_rng(77)
    u0 = np.clip(rng.standard_normal((T, 1)), -4.5, 4.5)
    x0 = np.array([math.pi - 0.3, 0.0])
    opts = BarrierOptions(newton=NewtonOptions(max_iters=300))
    prob = ControlProblem(dyn, cost, box)
    traj, rep = barrier_solve(prob, rollout(dyn, x0, u0), opts)
    out = dict(x0=x0, u0=u0, weights=np.array([10.0, 0.1, 0.01, 100.0, 10.0]))
    _barrier_record("sol", traj, rep, out)

    def solve(xp, up):
        t, r = barrier_solve(prob, rollout(dyn, xp, up), opts)
        return t, [q.newton.iterations for q in r.rounds]
    out.update({"sol_" + k: v for k, v in noise_floor(
        solve, x0, u0, traj, [q.newton.iterations for q in rep.rounds]).items()})
    save("barrier_pendulum_cosine", **out)


def case_pendulum_norm_constraints():
    """User-defined constraints (NormConstraints: |omega| < 8, |u| < 5 as
    curved rows) on the T=40 pendulum swing-up, barrier and ADMM."""
    T = 40
    dyn = PendulumDynamics(T, PendulumParams(damping=0.1, dt=0.05))
    cost = QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]),
                         x_goal=np.zeros(2))
    con = NormConstraints(8.0, 5.0)
    prob = ControlProblem(dyn, cost, con)
    rng = np.random.default_rng(91)
    u0 = np.clip(0.5 * rng.standard_normal((T, 1)), -2.0, 2.0)
    x0 = np.array([math.pi - 0.2, 0.0])
    init = rollout(dyn, x0, u0)
    out = dict(x0=x0, u0=u0, limits=np.array([8.0, 5.0]))
    bopts = BarrierOptions(newton=NewtonOptions(max_iters=300))
    traj, rep = barrier_solve(prob, init, bopts)
    _barrier_record("bar", traj, rep, out)

    def solve(xp, up):
        t, r = barrier_solve(prob, rollout(dyn, xp, up), bopts)
        return t, [q.newton.iterations for q in r.rounds]
    out.update({"bar_" + k: v for k, v in noise_floor(
        solve, x0, u0, traj, [q.newton.iterations for q in rep.rounds]).items()})
    aopts = AdmmOptions(rho=1.0, max_outer=40)
    traj, rep = admm_solve(prob, init, aopts)
    _admm_record("admm", traj, rep, out)

    def solve2(xp, up):
        t, r = admm_solve(prob, rollout(dyn, xp, up), aopts)
        return t, [q.iterations for q in r.newton_reports]
    out.update({"admm_" + k: v for k, v in noise_floor(
        solve2, x0, u0, traj, [q.iterations for q in rep.newton_reports]).items()})
    save("pendulum_norm_constraints", **out)


def _admm_record(prefix, traj, rep, out):
    out[f"{prefix}_xs"], out[f"{prefix}_us"] = traj.states, traj.controls
    out[f"{prefix}_z"], out[f"{prefix}_v"] = rep.state.z, rep.state.v
    out[f"{prefix}_residuals"] = np.array(rep.residual_history)
    out[f"{prefix}_newton_iters"] = np.array([r.iterations for r in rep.newton_reports])
    out[f"{prefix}_converged"] = np.array(rep.converged)


def case_admm_small():
    """pendulum (reference default params) and config-2 cart-pole at T=60."""
    out = {}
    # pendulum, reference defaults, rho = 1
    T = 30
    prob = pintoc.make_swingup_problem("pendulum", T, 0.05)
    rng = np.random.default_rng(505)
    u0 = rng.standard_normal((T, 1))
    x0 = np.array([math.pi, 0.0])
    init = rollout(prob.dynamics, x0, u0)
    traj, rep = admm_solve(prob, init, AdmmOptions(rho=1.0, max_outer=150))
    out.update(pend_x0=x0, pend_u0=u0)
    _admm_record("pend", traj, rep, out)

    def solve(xp, up):
        t, r = admm_solve(prob, rollout(prob.dynamics, xp, up), AdmmOptions(rho=1.0, max_outer=150))
        return t, [q.iterations for q in r.newton_reports]
    out.update({"pend_" + k: v for k, v in noise_floor(
        solve, x0, u0, traj, [q.iterations for q in rep.newton_reports]).items()})
    # cart-pole, config-2 parameters, short horizon
    T = 60
    dyn = CartPoleDynamics(T, CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                             pole_length=0.5, dt=0.02))
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    cost = QuadraticCost(Q, np.diag([0.01]), 10 * Q, x_goal=np.array([0.0, math.pi, 0.0, 0.0]))
    box = BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0,
                        state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                        state_upper=[1.5, np.inf, np.inf, np.inf])
    u0 = 0.1 * rng.standard_normal((T, 1))
    x0 = np.zeros(4)
    init = rollout(dyn, x0, u0)
    traj, rep = admm_solve(ControlProblem(dyn, cost, box), init, AdmmOptions(rho=1.0, max_outer=40))
    out.update(cp_x0=x0, cp_u0=u0)
    _admm_record("cp", traj, rep, out)

    def solve2(xp, up):
        t, r = admm_solve(ControlProblem(dyn, cost, box), rollout(dyn, xp, up),
                          AdmmOptions(rho=1.0, max_outer=40))
        return t, [q.iterations for q in r.newton_reports]
    out.update({"cp_" + k: v for k, v in noise_floor(
        solve2, x0, u0, traj, [q.iterations for q in rep.newton_reports]).items()})
    save("admm_small", **out)


def case_admm_cartpole_cfg2():
    """BASELINE config 2 at full size (T=500, rho=1, 200 outer): slow (~16 min)."""
    T = 500
    dyn = CartPoleDynamics(T, CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                             pole_length=0.5, dt=0.02))
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    cost = QuadraticCost(Q, np.diag([0.01]), 10 * Q, x_goal=np.array([0.0, math.pi, 0.0, 0.0]))
    box = BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0,
                        state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                        state_upper=[1.5, np.inf, np.inf, np.inf])
    rng = np.random.default_rng(0)
    u0 = 0.1 * rng.standard_normal((T, 1))
    x0 = np.zeros(4)
    init = rollout(dyn, x0, u0)
    t0 = time.perf_counter()
    traj, rep = admm_solve(ControlProblem(dyn, cost, box), init, AdmmOptions(rho=1.0, max_outer=200))
    wall = time.perf_counter() - t0
    out = dict(x0=x0, u0=u0, wall_s=np.array(wall))
    _admm_record("sol", traj, rep, out)
    save("admm_cartpole_cfg2", **out)


def case_admm_cartpole_cfg2_nudge():
    """Reproducibility of config 2's Newton iteration counts in the reference
    itself: the first three ADMM outer steps from the config-2 start and from
    the start moved by one ulp either way (~1.5 min)."""
    T = 500
    dyn = CartPoleDynamics(T, CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                             pole_length=0.5, dt=0.02))
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    cost = QuadraticCost(Q, np.diag([0.01]), 10 * Q, x_goal=np.array([0.0, math.pi, 0.0, 0.0]))
    box = BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0,
                        state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                        state_upper=[1.5, np.inf, np.inf, np.inf])
    rng = np.random.default_rng(0)
    u0 = 0.1 * rng.standard_normal((T, 1))
    x0 = np.zeros(4)
    rows = []
    for xp, up in [(x0, u0)] + ulp_nudges(x0, u0):
        _, rep = admm_solve(ControlProblem(dyn, cost, box), rollout(dyn, xp, up),
                            AdmmOptions(rho=1.0, max_outer=3))
        rows.append([r.iterations for r in rep.newton_reports])
    save("admm_cartpole_cfg2_nudge", iters=np.array(rows))


def case_criterion5_pendulum():
    """Reference acceptance criterion 5 setup (harness draw, N = 20/100/500):
    the reference's per-round iteration counts and terminations (N = 500
    does not converge in its first round), their stability under one-ulp
    control nudges, and the final controls."""
    from pintoc.bench import RunConfig, draw_initial_controls
    from pintoc import swingup_start
    out = {}
    for n in (20, 100, 500):
        cfg = RunConfig(system="pendulum", solver="barrier", seed=0, horizons=(n,),
                        total_time=2.0)
        problem = cfg.build_problem(n, cfg.step_size(n))
        u0 = draw_initial_controls(problem, cfg, n, 0)
        x0 = swingup_start("pendulum")

        def solve(xp, up):
            traj, rep = barrier_solve(problem, rollout(problem.dynamics, xp, up),
                                      cfg.barrier_options())
            return traj, [r.newton.iterations for r in rep.rounds]

        traj, rep = barrier_solve(problem, rollout(problem.dynamics, x0, u0),
                                  cfg.barrier_options())
        counts = [r.newton.iterations for r in rep.rounds]
        out[f"n{n}_u0"] = u0
        out[f"n{n}_iters"] = np.array(counts)
        out[f"n{n}_terms"] = np.array([r.newton.termination for r in rep.rounds])
        out[f"n{n}_us"] = traj.controls
        out.update({f"n{n}_{k}": v for k, v in noise_floor(solve, x0, u0, traj, counts).items()})
    save("criterion5_pendulum", **out)


FAST = [case_lqr_small, case_lqr_config1, case_passes_models, case_newton_lq,
        case_barrier_pendulum_cfg0, case_barrier_pendulum_conv, case_barrier_tvlinear, case_admm_small,
        case_barrier_pendulum_cosine, case_pendulum_norm_constraints]

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--slow", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    cases = FAST + ([case_admm_cartpole_cfg2, case_admm_cartpole_cfg2_nudge,
                     case_criterion5_pendulum] if args.slow else [])
    for fn in cases:
        if args.only and args.only not in fn.__name__:
            continue
        t0 = time.perf_counter()
        fn()
        print(f"  {fn.__name__}: {time.perf_counter() - t0:.1f}s")
