"""Behavioural properties the reference's own suite asserts for the Newton
loop and the outer loops (reference pkg/tests/test_newton.py, test_outer.py),
checked on the CUDA path:

* LQ problems: at most two accepted steps to the Riccati optimum, an
  optimal start ends after one iteration on the step criterion, the first
  gain ratio of a quadratic problem is 1 (newton.py:93-110);
* accepted costs never increase, iterates stay dynamically consistent,
  barrier iterates stay strictly feasible, one history record per
  iteration, first-order optimality (d ~ 0) at a converged barrier
  subproblem;
* barrier: far bounds reproduce the unconstrained solve, a vacuous mu
  schedule returns the initial trajectory, every round strictly feasible;
* ADMM: a feasible unconstrained optimum is a fixed point (one outer
  iteration), an exhausted budget is reported, not raised.
Tolerances as in the reference tests.
"""

import numpy as np
import pytest

from oracle import pintoc_oracle as O

pytestmark = pytest.mark.gpu


def _lq(rng, n, nx, nu):
    import paper_2409_20027_b200 as P
    A = np.eye(nx) + 0.1 * rng.standard_normal((nx, nx))
    B = rng.standard_normal((nx, nu))
    Mq = rng.standard_normal((nx, nx))
    Q = Mq @ Mq.T + 0.5 * np.eye(nx)
    R = np.eye(nu) * 0.5
    goal = rng.standard_normal(nx)
    dyn = P.LinearDynamics(A, B, horizon=n)
    cost = P.QuadraticCost(Q, R, 2.0 * Q, x_goal=goal)
    x0 = rng.standard_normal(nx)
    init = P.rollout(dyn, x0, np.zeros((n, nu)))
    # the optimum: the oracle's Newton solve of the LQ problem (exact)
    ref = O.newton_solve(O.Linear(A, B), O.Quadratic(Q, R, 2.0 * Q, goal), ("zero",),
                         init.states, init.controls, alpha0=0.0)
    return dyn, cost, init, ref


def test_lq_converges_in_at_most_two_accepted_steps():
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(40)
    for _ in range(5):
        n = int(rng.integers(4, 20))
        dyn, cost, init, ref = _lq(rng, n, 2, 1)
        traj, rep = P.newton_solve(dyn, cost, None, init, P.NewtonOptions(alpha0=0.0))
        assert rep.converged and rep.accepted_steps <= 2
        scale = max(1.0, np.abs(ref.us).max())
        assert np.abs(traj.controls - ref.us).max() / scale < 1e-6


def test_optimal_start_terminates_on_the_step_criterion():
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(41)
    dyn, cost, init, ref = _lq(rng, 10, 2, 1)
    opt = P.Trajectory(ref.xs, ref.us)
    traj, rep = P.newton_solve(dyn, cost, None, opt, P.NewtonOptions(alpha0=0.0))
    assert rep.iterations == 1
    assert rep.history[0].step_norm <= 1e-8
    assert rep.termination == "converged_step"


def test_quadratic_problem_first_gain_ratio_is_one():
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(42)
    dyn, cost, init, _ = _lq(rng, 8, 2, 2)
    _, rep = P.newton_solve(dyn, cost, None, init, P.NewtonOptions(alpha0=0.5))
    first = rep.history[0]
    assert first.accepted and abs(first.gain_ratio - 1.0) < 1e-9


def _pendulum(n, rng, scale):
    import paper_2409_20027_b200 as P
    prob = P.make_swingup_problem("pendulum", n, 0.05)
    init = P.rollout(prob.dynamics, np.array([np.pi, 0.0]), scale * rng.standard_normal((n, 1)))
    return prob, init


def test_accepted_costs_never_increase():
    import paper_2409_20027_b200 as P
    prob, init = _pendulum(25, np.random.default_rng(43), 0.5)
    aug = P.BarrierAugmentation(prob.constraints, 0.1)
    _, rep = P.newton_solve(prob.dynamics, prob.cost, aug, init, P.NewtonOptions(max_iters=60))
    costs = [r.cost for r in rep.history if r.accepted]
    assert all(b <= a + 1e-12 for a, b in zip(costs, costs[1:]))
    assert rep.final_cost <= P.total_cost(prob.cost, aug, init, dyn=prob.dynamics)


def test_iterates_stay_dynamically_consistent():
    import paper_2409_20027_b200 as P
    prob, init = _pendulum(15, np.random.default_rng(44), 0.3)
    traj, _ = P.newton_solve(prob.dynamics, prob.cost, None, init, P.NewtonOptions(max_iters=40))
    odyn = O.Pendulum(dt=0.05)
    for t in range(traj.horizon):
        nxt = odyn.step(t, traj.states[t], traj.controls[t])
        assert np.abs(nxt - traj.states[t + 1]).max() < 1e-10


def test_barrier_newton_iterates_stay_strictly_feasible():
    import paper_2409_20027_b200 as P
    prob, init = _pendulum(20, np.random.default_rng(45), 0.5)
    aug = P.BarrierAugmentation(prob.constraints, 0.05)
    traj, _ = P.newton_solve(prob.dynamics, prob.cost, aug, init, P.NewtonOptions(max_iters=80))
    assert prob.constraints.max_violation(traj) < 0.0


def test_history_has_one_record_per_iteration():
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(46)
    dyn, cost, init, _ = _lq(rng, 6, 2, 1)
    _, rep = P.newton_solve(dyn, cost, None, init, P.NewtonOptions())
    assert len(rep.history) == rep.iterations


def test_first_order_optimality_at_converged_barrier_subproblem():
    import paper_2409_20027_b200 as P
    prob, init = _pendulum(30, np.random.default_rng(47), 0.5)
    aug = P.BarrierAugmentation(prob.constraints, 0.1)
    traj, rep = P.newton_solve(prob.dynamics, prob.cost, aug, init, P.NewtonOptions(max_iters=200))
    assert rep.converged
    lam = P.costate_pass(traj, prob.cost, aug, prob.dynamics)
    exp = P.hamiltonian_expansion(traj, lam, prob.cost, aug, prob.dynamics)
    assert np.abs(exp.d).max() <= 1e-4


def test_barrier_with_far_bounds_matches_unconstrained():
    import paper_2409_20027_b200 as P
    n = 12
    prob, init = _pendulum(n, np.random.default_rng(48), 0.3)
    wide = P.BoxConstraint(2, 1, control_lower=-1e6, control_upper=1e6)
    free, _ = P.newton_solve(prob.dynamics, prob.cost, None, init, P.NewtonOptions(max_iters=100))
    con, rep = P.barrier_solve(P.ControlProblem(prob.dynamics, prob.cost, wide), init,
                               P.BarrierOptions())
    assert rep.converged
    assert np.abs(con.controls - free.controls).max() < 1e-3


def test_barrier_vacuous_schedule_returns_initial():
    import paper_2409_20027_b200 as P
    dyn = P.LinearDynamics(np.eye(1), np.zeros((1, 1)), horizon=1)
    cost = P.QuadraticCost(np.zeros((1, 1)), 2.0 * np.eye(1), np.zeros((1, 1)))
    box = P.BoxConstraint(1, 1, control_lower=1.0)
    init = P.rollout(dyn, np.zeros(1), np.array([[2.0]]))
    traj, rep = P.barrier_solve(P.ControlProblem(dyn, cost, box), init,
                                P.BarrierOptions(mu0=1e-5, mu_tol=1e-4))
    assert rep.outer_iterations == 0
    assert np.array_equal(traj.controls, init.controls)


def test_barrier_every_round_strictly_feasible():
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200.harness import draw_initial_controls
    prob = P.make_swingup_problem("pendulum", 20, 0.05)
    cfg = P.RunConfig(system="pendulum", solver="barrier", horizons=(20,))
    init = P.rollout(prob.dynamics, np.array([np.pi, 0.0]),
                     draw_initial_controls(prob, cfg, 20, 0))
    _, rep = P.barrier_solve(prob, init, P.BarrierOptions())
    assert rep.outer_iterations > 0
    for rnd in rep.rounds:
        assert np.abs(rnd.controls).max() < 5.0


def test_admm_feasible_optimum_is_a_fixed_point():
    import paper_2409_20027_b200 as P
    n = 8
    dyn = P.LinearDynamics(np.eye(2) * 0.9, np.array([[0.0], [1.0]]), horizon=n)
    cost = P.QuadraticCost(np.eye(2), np.eye(1), np.eye(2))
    box = P.BoxConstraint(2, 1, control_lower=-50.0, control_upper=50.0)
    init = P.rollout(dyn, np.array([0.5, -0.5]), np.zeros((n, 1)))
    free, _ = P.newton_solve(dyn, cost, None, init, P.NewtonOptions())
    _, rep = P.admm_solve(P.ControlProblem(dyn, cost, box), free, P.AdmmOptions(rho=1.0))
    assert rep.converged and rep.outer_iterations == 1


def test_admm_budget_exhaustion_is_reported_not_raised():
    import paper_2409_20027_b200 as P
    prob, init = _pendulum(20, np.random.default_rng(49), 0.5)
    _, rep = P.admm_solve(prob, init, P.AdmmOptions(rho=1.0, max_outer=2))
    assert not rep.converged and rep.outer_iterations == 2
