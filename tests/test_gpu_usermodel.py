"""User-defined dynamics through the device hook (usermodel.DeviceDynamics,
csrc/user_model.cuh): the reference's user-model pattern -- a
DynamicsModel subclass such as make_golden.py's TVLinear -- written as
per-stage CUDA code, compiled into its own kernel library and run by the
same solver entry points, checked against the reference's own runs."""

import numpy as np
import pytest
from conftest import golden, rel_gap
from test_gpu_newton import _hist
from restart_util import check_iterations, device_restart
from user_models import user_cosine_cost, user_norm_constraints, user_pendulum, user_tvlinear

pytestmark = pytest.mark.gpu

TOL = 1e-9


def test_user_tvlinear_barrier_matches_reference():
    """make_golden's TVLinear (a user DynamicsModel in pintoc) on the
    barrier method: counts, histories and trajectories of the reference."""
    import paper_2409_20027_b200 as P
    from test_gpu_newton import _check_hist, _hist
    g = golden("barrier_tvlinear")
    dyn = user_tvlinear(g["A"], g["B"], g["c"])
    nu = dyn.d_u
    cost = P.QuadraticCost(g["Q"], 0.1 * np.eye(nu), g["Q"])
    box = P.BoxConstraint(dyn.d_x, nu, control_lower=-2.0, control_upper=2.0)
    init = P.rollout(dyn, g["x0"], g["u0"])
    for ex in ("sequential", "parallel"):
        traj, rep = P.barrier_solve(P.ControlProblem(dyn, cost, box), init,
                                    P.BarrierOptions(newton=P.NewtonOptions(executor=ex)))
        assert [r.newton.iterations for r in rep.rounds] == list(g["sol_round_iters"])
        for k, r in enumerate(rep.rounds):
            _check_hist(_hist(r.newton), g[f"sol_hist{k}"])
        assert rel_gap(traj.controls, g["sol_us"]) < TOL
        assert rel_gap(traj.states, g["sol_xs"]) < TOL


def test_user_pendulum_converging_swingup_matches_reference():
    import paper_2409_20027_b200 as P
    from test_gpu_newton import _check_hist, _hist
    g = golden("barrier_pendulum_conv")
    builtin = P.make_swingup_problem("pendulum", 40, 0.05)
    prm = builtin.dynamics.params
    dyn = user_pendulum(40, prm.gravity, prm.length, prm.mass, prm.damping, prm.dt)
    prob = P.ControlProblem(dyn, builtin.cost, builtin.constraints)
    init = P.rollout(dyn, g["x0"], g["u0"])
    traj, rep = P.barrier_solve(prob, init, P.BarrierOptions(newton=P.NewtonOptions(max_iters=300)))
    assert [r.newton.iterations for r in rep.rounds] == list(g["sol_round_iters"])
    for k, r in enumerate(rep.rounds):
        _check_hist(_hist(r.newton), g[f"sol_hist{k}"])
    assert rel_gap(traj.controls, g["sol_us"]) < TOL


def test_user_pendulum_config0_every_iteration():
    """All 600 config-0 iterations restarted from the reference's states
    with the user-code pendulum (the same restart test as the built-in)."""
    import paper_2409_20027_b200 as P
    g = golden("restart_cfg0")
    cost = P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
    box = P.BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0)
    prob = P.ControlProblem(user_pendulum(100), cost, box)
    tin = g["it_in"]
    res = device_restart(prob, g["traj_x"][tin], g["traj_u"][tin], g["it_alpha"], g["it_nu"],
                         mu=g["it_aug"])
    out = check_iterations(res, g, label="user-pendulum cfg0")
    assert out["rows"] == 600


def test_user_model_batched_and_fp32():
    """BatchSolver and the fp32 kernel set run the user model too."""
    import torch

    import paper_2409_20027_b200 as P
    T, B = 64, 16
    dyn = user_pendulum(T)
    prob = P.ControlProblem(dyn, P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]),
                                                 np.diag([100.0, 10.0])),
                            P.BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0))
    rng = np.random.default_rng(3)
    x0 = np.stack([rng.uniform(-0.3, 0.3, B), rng.normal(0, 0.1, B)], 1)
    u0 = torch.as_tensor(np.clip(rng.normal(0, 0.5, (B, T, 1)), -4, 4)).cuda()
    opts = P.BarrierOptions(newton=P.NewtonOptions(max_iters=60))
    bs = P.BatchSolver(prob, B, "barrier", barrier=opts)
    res = bs.solve(bs.rollout(x0, u0), u0)
    for b in range(3):
        init = P.rollout(dyn, x0[b], u0[b].cpu().numpy())
        traj, rep = P.barrier_solve(prob, init, opts)
        assert rel_gap(res.controls[b].cpu().numpy(), traj.controls) < 1e-12
    bs32 = P.BatchSolver(prob, B, "barrier", barrier=opts, dtype=torch.float32)
    X32 = bs32.rollout(x0, u0.float())
    assert torch.isfinite(X32).all()


def test_user_cost_matches_reference():
    """make_golden's CosineCost -- a user CostModel with a non-quadratic,
    indefinite-Hessian stage cost and terminal cost -- written against the
    device hook (DeviceCost) matches pintoc's barrier run of it: per-round
    counts, iteration histories, trajectory at 1e-9."""
    import paper_2409_20027_b200 as P
    from test_gpu_newton import _hist
    g = golden("barrier_pendulum_cosine")
    w = g["weights"]
    dyn = user_pendulum(40)
    cost = user_cosine_cost(*w)
    box = P.BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0)
    prob = P.ControlProblem(dyn, cost, box)
    init = P.rollout(dyn, g["x0"], g["u0"])
    for ex in ("sequential", "parallel"):
        traj, rep = P.barrier_solve(prob, init, P.BarrierOptions(
            newton=P.NewtonOptions(max_iters=300, executor=ex)))
        assert [r.newton.iterations for r in rep.rounds] == list(g["sol_round_iters"]), ex
        assert [r.newton.termination for r in rep.rounds] == list(g["sol_round_term"])
        for k, r in enumerate(rep.rounds):
            _check_hist_band(_hist(r.newton), g[f"sol_hist{k}"])
        assert rel_gap(traj.controls, g["sol_us"]) < TOL
        assert rel_gap(traj.states, g["sol_xs"]) < TOL
        assert rel_gap([r.cost for r in rep.rounds], g["sol_round_cost"]) < TOL


def _check_hist_band(hist, ref):
    """Iteration records equal: accept flags exactly, costs and step norms
    at 1e-9, the gain ratio -- (cur - new) / pred, a difference quotient of
    two costs -- within 1e-9 (|cur| + |new|) / |pred| (restart_util), and
    alpha, which the LM rule derives from the ratios, at 1e-6 (as
    test_gpu_newton's records)."""
    assert hist.shape == ref.shape
    assert np.array_equal(hist[:, 4], ref[:, 4])
    for col, tol in ((0, TOL), (1, 1e-6), (3, TOL)):
        fin = np.isfinite(ref[:, col])
        assert np.array_equal(np.isfinite(hist[:, col]), fin), col
        gap = np.abs(hist[fin, col] - ref[fin, col]) / np.maximum(1.0, np.abs(ref[fin, col]))
        assert gap.max(initial=0.0) < tol, col
    prev = np.concatenate([[np.nan], ref[:-1, 0]])
    fin = np.isfinite(ref[:, 2]) & (ref[:, 4] > 0.5) & np.isfinite(prev)
    if fin.any():
        pred = np.abs(prev[fin] - ref[fin, 0]) / np.abs(ref[fin, 2])
        band = TOL * (np.abs(prev[fin]) + np.abs(ref[fin, 0])) / pred + TOL * np.abs(ref[fin, 2])
        assert np.all(np.abs(hist[fin, 2] - ref[fin, 2]) <= band)


def _norm_problem(P, g):
    wmax, umax = g["limits"]
    dyn = user_pendulum(40)
    cost = P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
    return dyn, P.ControlProblem(dyn, cost, user_norm_constraints(wmax, umax))


def test_user_constraints_barrier_and_admm_match_reference():
    """make_golden's NormConstraints -- a user ConstraintModel with curved
    rows (omega^2 <= wmax^2, u^2 <= umax^2: nonzero gxx, huu) -- as a
    DeviceConstraint: the barrier solve (per-round counts, histories,
    trajectory 1e-9) and the ADMM solve (per-step counts, residuals, z,
    trajectory) of pintoc."""
    import paper_2409_20027_b200 as P
    g = golden("pendulum_norm_constraints")
    dyn, prob = _norm_problem(P, g)
    init = P.rollout(dyn, g["x0"], g["u0"])
    traj, rep = P.barrier_solve(prob, init, P.BarrierOptions(newton=P.NewtonOptions(max_iters=300)))
    assert [r.newton.iterations for r in rep.rounds] == list(g["bar_round_iters"])
    assert [r.newton.termination for r in rep.rounds] == list(g["bar_round_term"])
    for k, r in enumerate(rep.rounds):
        _check_hist_band(_hist(r.newton), g[f"bar_hist{k}"])
    assert rel_gap(traj.controls, g["bar_us"]) < TOL
    assert rel_gap(traj.states, g["bar_xs"]) < TOL
    traj, rep = P.admm_solve(prob, init, P.AdmmOptions(rho=1.0, max_outer=40))
    assert rep.converged == bool(g["admm_converged"])
    assert [r.iterations for r in rep.newton_reports] == list(g["admm_newton_iters"])
    assert rel_gap(np.array(rep.residual_history), g["admm_residuals"]) < 1e-8
    assert rel_gap(rep.state.z, g["admm_z"]) < 1e-8
    assert rel_gap(traj.controls, g["admm_us"]) < TOL


def test_user_constraints_infeasible_start_reports_the_row():
    """An initial control outside the curved box: the barrier solve raises
    InfeasibleError(stage, component, value) for the first violated row, as
    the reference's assert_strictly_feasible does (outer.py:163-177)."""
    import paper_2409_20027_b200 as P
    g = golden("pendulum_norm_constraints")
    dyn, prob = _norm_problem(P, g)
    u0 = np.array(g["u0"])
    u0[7, 0] = 5.5                       # h = 5.5^2 - 25 = 5.25 at stage 7
    with pytest.raises(P.InfeasibleError) as err:
        P.barrier_solve(prob, P.rollout(dyn, g["x0"], u0), P.BarrierOptions())
    assert (err.value.stage, err.value.component) == (7, 1)
    assert abs(err.value.value - 5.25) < 1e-12
