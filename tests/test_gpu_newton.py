"""GPU parity of the full solver path against the reference's own runs.

Criterion: Newton iteration counts identical to the
reference wherever the reference's own counts are stable under one-ulp
input nudges, and final fp64 trajectories within max(1e-9, 10 x floor),
where `floor` is the reference's own reproducibility -- how far its final
trajectory moves when its inputs move by one ulp (recorded in the golden
fixture by tests/golden/make_golden.py).  For well-conditioned problems the
floor is ~1e-15 and the bound is the north-star 1e-9; for the chaotic
config-0 swing-up (100 non-converged LM iterations per round on an
unstable pendulum) the reference itself only reproduces to ~6e-3.
Per-iteration histories are compared while the floor is below 1e-9.
"""

import math

import numpy as np
import pytest
from conftest import golden, rel_gap

from oracle import pintoc_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-9


def tol(g, p):
    return max(TOL, 10.0 * float(g[p + "floor_u"]), 10.0 * float(g[p + "floor_x"]))


def well_posed(g, p):
    return float(g[p + "floor_u"]) < 1e-10 and bool(g[p + "stable"])


def _hist(report):
    return np.array([(r.cost, r.alpha, r.gain_ratio, r.step_norm, float(r.accepted))
                     for r in report.history]).reshape(-1, 5)


def _check_hist(hist, ref):
    assert hist.shape == ref.shape
    assert np.array_equal(hist[:, 4], ref[:, 4])
    # the gain ratio (cur - new) / pred is a quotient of two cancellations; once
    # the relative cost change falls to rounding level (< 1e-9) its digits are
    # noise in the reference too, so only its sign is compared there
    prev = np.concatenate([[np.inf], ref[:-1, 0]])
    noisy = np.abs(prev - ref[:, 0]) <= 1e-9 * np.maximum(1.0, np.abs(ref[:, 0]))
    for col, tol in ((0, 1e-9), (1, 1e-6), (2, 1e-6), (3, 1e-7)):
        a, b = hist[:, col], ref[:, col]
        fin = np.isfinite(b)
        assert np.array_equal(np.isfinite(a), fin), col
        check = fin & ~noisy if col == 2 else fin
        if col == 2:
            assert np.array_equal(np.sign(a[fin]), np.sign(b[fin]))
        if check.any():
            scale = np.maximum(1.0, np.abs(b[check]))
            assert np.max(np.abs(a[check] - b[check]) / scale) < tol, col


def test_newton_lq_matches_reference():
    import paper_2409_20027_b200 as P
    g = golden("newton_lq")
    for i in range(int(g["count"])):
        p = f"{i}_"
        n, du = g[p + "us"].shape
        dyn = P.LinearDynamics(g[p + "A"], g[p + "B"], horizon=n)
        cost = P.QuadraticCost(g[p + "Q"], g[p + "R"], g[p + "Qf"], x_goal=g[p + "goal"])
        init = P.rollout(dyn, g[p + "x0"], np.zeros((n, du)))
        traj, rep = P.newton_solve(dyn, cost, None, init,
                                   P.NewtonOptions(alpha0=float(g[p + "alpha0"])))
        assert rep.termination == str(g[p + "term"])
        assert rep.iterations == len(g[p + "hist"])
        if well_posed(g, p):
            _check_hist(_hist(rep), g[p + "hist"])
        assert rel_gap(traj.controls, g[p + "us"]) < tol(g, p), i
        assert rel_gap(traj.states, g[p + "xs"]) < tol(g, p), i


def _pend_cfg0(P, T=100):
    dyn = P.PendulumDynamics(T, P.PendulumParams(damping=0.1, dt=0.05))
    cost = P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
    box = P.BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0)
    return P.ControlProblem(dyn, cost, box)


@pytest.mark.parametrize("executor", ["auto", "sequential", "parallel"])
def test_barrier_pendulum_config0_matches_reference(executor):
    import paper_2409_20027_b200 as P
    g = golden("barrier_pendulum_cfg0")
    prob = _pend_cfg0(P)
    init = P.rollout(prob.dynamics, g["x0"], g["u0"])
    opts = P.BarrierOptions(mu0=0.1, zeta=0.1, mu_tol=5e-7,
                            newton=P.NewtonOptions(max_iters=100, executor=executor))
    traj, rep = P.barrier_solve(prob, init, opts)
    assert [r.newton.iterations for r in rep.rounds] == list(g["sol_round_iters"])
    assert [r.newton.termination for r in rep.rounds] == list(g["sol_round_term"])
    assert np.allclose([r.mu for r in rep.rounds], g["sol_mus"], rtol=1e-15)
    if well_posed(g, "sol_"):
        for k, r in enumerate(rep.rounds):
            _check_hist(_hist(r.newton), g[f"sol_hist{k}"])
    assert rel_gap(traj.controls, g["sol_us"]) < tol(g, "sol_")
    assert rel_gap(traj.states, g["sol_xs"]) < tol(g, "sol_")
    assert np.abs(traj.controls).max() < 5.0


def test_barrier_tvlinear_matches_reference():
    import paper_2409_20027_b200 as P
    g = golden("barrier_tvlinear")
    dyn = P.TimeVaryingLinearDynamics(g["A"], g["B"], g["c"])
    nu = dyn.d_u
    cost = P.QuadraticCost(g["Q"], 0.1 * np.eye(nu), g["Q"])
    box = P.BoxConstraint(dyn.d_x, nu, control_lower=-2.0, control_upper=2.0)
    init = P.rollout(dyn, g["x0"], g["u0"])
    traj, rep = P.barrier_solve(P.ControlProblem(dyn, cost, box), init, P.BarrierOptions())
    assert [r.newton.iterations for r in rep.rounds] == list(g["sol_round_iters"])
    assert well_posed(g, "sol_")
    for k, r in enumerate(rep.rounds):
        _check_hist(_hist(r.newton), g[f"sol_hist{k}"])
    assert rel_gap(traj.controls, g["sol_us"]) < TOL
    assert rel_gap(traj.states, g["sol_xs"]) < TOL


def test_admm_small_matches_reference():
    import paper_2409_20027_b200 as P
    g = golden("admm_small")
    prob = P.make_swingup_problem("pendulum", 30, 0.05)
    init = P.rollout(prob.dynamics, g["pend_x0"], g["pend_u0"])
    traj, rep = P.admm_solve(prob, init, P.AdmmOptions(rho=1.0, max_outer=150))
    assert rep.converged == bool(g["pend_converged"])
    assert [r.iterations for r in rep.newton_reports] == list(g["pend_newton_iters"])
    assert rel_gap(np.array(rep.residual_history), g["pend_residuals"]) < 1e-7
    assert rel_gap(traj.controls, g["pend_us"]) < TOL
    assert rel_gap(rep.state.z, g["pend_z"]) < 1e-8

    T = 60
    dyn = P.CartPoleDynamics(T, P.CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                                 pole_length=0.5, dt=0.02))
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    cost = P.QuadraticCost(Q, np.diag([0.01]), 10 * Q, x_goal=np.array([0.0, math.pi, 0.0, 0.0]))
    box = P.BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0,
                          state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                          state_upper=[1.5, np.inf, np.inf, np.inf])
    init = P.rollout(dyn, g["cp_x0"], g["cp_u0"])
    traj, rep = P.admm_solve(P.ControlProblem(dyn, cost, box), init,
                             P.AdmmOptions(rho=1.0, max_outer=40))
    assert rep.converged == bool(g["cp_converged"])
    assert [r.iterations for r in rep.newton_reports] == list(g["cp_newton_iters"])
    assert rel_gap(traj.controls, g["cp_us"]) < TOL
    assert rel_gap(traj.states, g["cp_xs"]) < TOL


def test_barrier_rejects_infeasible_start():
    import paper_2409_20027_b200 as P
    dyn = P.LinearDynamics(np.eye(1), np.zeros((1, 1)), horizon=1)
    cost = P.QuadraticCost(np.zeros((1, 1)), 2.0 * np.eye(1), np.zeros((1, 1)))
    box = P.BoxConstraint(1, 1, control_lower=1.0)
    init = P.rollout(dyn, np.zeros(1), np.array([[0.5]]))
    with pytest.raises(P.InfeasibleError, match="not strictly feasible"):
        P.barrier_solve(P.ControlProblem(dyn, cost, box), init, P.BarrierOptions())


def test_one_dim_barrier_tracks_closed_form():
    import paper_2409_20027_b200 as P
    dyn = P.LinearDynamics(np.eye(1), np.zeros((1, 1)), horizon=1)
    cost = P.QuadraticCost(np.zeros((1, 1)), 2.0 * np.eye(1), np.zeros((1, 1)))
    box = P.BoxConstraint(1, 1, control_lower=1.0)
    init = P.rollout(dyn, np.zeros(1), np.array([[2.0]]))
    traj, rep = P.barrier_solve(P.ControlProblem(dyn, cost, box), init, P.BarrierOptions())
    assert rep.outer_iterations == 5
    for rnd in rep.rounds:
        assert abs(rnd.controls[0, 0] - 0.5 * (1.0 + math.sqrt(1.0 + 2.0 * rnd.mu))) < 1e-6
    assert abs(traj.controls[0, 0] - 1.0) < 1e-3


def test_inconsistent_initial_rejected():
    import paper_2409_20027_b200 as P
    dyn = P.LinearDynamics(np.eye(2) * 0.9, np.array([[0.0], [1.0]]), horizon=6)
    cost = P.QuadraticCost(np.eye(2), np.eye(1), np.eye(2))
    init = P.rollout(dyn, np.array([0.5, -0.5]), np.zeros((6, 1)))
    bad = init.states.copy()
    bad[3] += 1.0
    with pytest.raises(ValueError, match="dynamically consistent"):
        P.newton_solve(dyn, cost, None, P.Trajectory(bad, init.controls))


def test_rollout_and_total_cost_match_oracle(rng):
    import paper_2409_20027_b200 as P
    g = golden("passes_models")
    prob = _pend_cfg0(P, 24)
    us = g["pendulum_us"]
    traj = P.rollout(prob.dynamics, g["pendulum_x0"], us)
    assert rel_gap(traj.states, g["pendulum_xs"]) < 1e-12
    aug = P.BarrierAugmentation(prob.constraints, 0.1)
    c = P.total_cost(prob.cost, aug, traj, dyn=prob.dynamics)
    assert abs(c - float(g["pendulum_barrier_cost"])) < 1e-11 * max(1.0, abs(c))


def test_barrier_pendulum_converging_matches_reference():
    """Nonlinear, converging swing-up: counts identical, trajectory 1e-9."""
    import paper_2409_20027_b200 as P
    g = golden("barrier_pendulum_conv")
    prob = P.make_swingup_problem("pendulum", 40, 0.05)
    init = P.rollout(prob.dynamics, g["x0"], g["u0"])
    for executor in ("auto", "sequential", "parallel"):
        opts = P.BarrierOptions(newton=P.NewtonOptions(max_iters=300, executor=executor))
        traj, rep = P.barrier_solve(prob, init, opts)
        assert well_posed(g, "sol_")
        assert [r.newton.iterations for r in rep.rounds] == list(g["sol_round_iters"])
        assert [r.newton.termination for r in rep.rounds] == list(g["sol_round_term"])
        for k, r in enumerate(rep.rounds):
            _check_hist(_hist(r.newton), g[f"sol_hist{k}"])
        assert rel_gap(traj.controls, g["sol_us"]) < TOL
        assert rel_gap(traj.states, g["sol_xs"]) < TOL


def test_admm_cartpole_config2_full_size():
    """BASELINE config 2 at full size (T=500, 200 outer iterations, ~17k
    Newton iterations; the reference needs ~16 min on one core)."""
    import paper_2409_20027_b200 as P
    g = golden("admm_cartpole_cfg2")
    T = 500
    dyn = P.CartPoleDynamics(T, P.CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                                 pole_length=0.5, dt=0.02))
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    cost = P.QuadraticCost(Q, np.diag([0.01]), 10 * Q, x_goal=np.array([0.0, math.pi, 0.0, 0.0]))
    box = P.BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0,
                          state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                          state_upper=[1.5, np.inf, np.inf, np.inf])
    init = P.rollout(dyn, g["x0"], g["u0"])
    traj, rep = P.admm_solve(P.ControlProblem(dyn, cost, box), init,
                             P.AdmmOptions(rho=1.0, max_outer=200))
    ref_iters = list(g["sol_newton_iters"])
    got = [r.iterations for r in rep.newton_reports]
    first_diff = next((k for k, (a, b) in enumerate(zip(got, ref_iters)) if a != b), None)
    print(f"cfg2: outer {rep.outer_iterations} vs {len(ref_iters)}, inner {sum(got)} vs "
          f"{sum(ref_iters)}, first differing outer step {first_diff}, "
          f"u gap {rel_gap(traj.controls, g['sol_us']):.3e}")
    assert rep.outer_iterations == len(ref_iters)
    assert rep.converged == bool(g["sol_converged"])
    # Iteration counts must match wherever the REFERENCE reproduces its own
    # counts under one-ulp input nudges (fixture admm_cartpole_cfg2_nudge:
    # the reference gives 100, {35, 37, 34}, 17 for the first three outer
    # steps -- outer step 0 ends in 100 non-converged LM iterations, so
    # step 1's count is rounding noise in the reference itself).
    nudge = golden("admm_cartpole_cfg2_nudge")["iters"]
    for k in range(nudge.shape[1]):
        if np.all(nudge[:, k] == nudge[0, k]):
            assert got[k] == ref_iters[k] == nudge[0, k], k
