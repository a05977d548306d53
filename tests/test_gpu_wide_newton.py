"""Warp-cooperative Newton kernels for wide affine models (nx >= 8,
csrc/wide_newton.cuh) against the CPU oracle:

* co-state pass and Hamiltonian expansion (passes.py:122-185) with all three
  augmentations, single-sweep and tree plans;
* the rollout API (problem.py:449; an affine scan on tree plans), including
  the divergence index;
* Newton / barrier / ADMM solves with the sequential executor (warp
  sequential candidate rollout) and the parallel executor (exact affine-scan
  candidate rollout; at T >= 1024 the co-state sweep also writes the LQR's
  stage-major staging rows directly): identical iteration counts, controls
  within 1e-8.
Tolerances: fp64, 1e-10 relative for single passes (the oracle folds the
co-state's cost and augmentation parts separately, passes.py:113-148),
1e-8 for whole solves.
"""

import numpy as np
import pytest
from conftest import rel_gap

from oracle import pintoc_oracle as O

pytestmark = pytest.mark.gpu


def _system(nx, nu, T, seed):
    rng = np.random.default_rng([nx, nu, T, seed])
    A = np.eye(nx)[None] + 0.05 * rng.standard_normal((T, nx, nx))
    rad = np.max(np.abs(np.linalg.eigvals(A)), axis=1)
    A *= np.minimum(1.0, 1.0 / rad)[:, None, None]
    B = 0.3 * rng.standard_normal((T, nx, nu))
    c = 0.05 * rng.standard_normal((T, nx))
    x0 = rng.standard_normal(nx)
    u0 = np.clip(0.3 * rng.standard_normal((T, nu)), -1.5, 1.5)
    return A, B, c, x0, u0, rng


def _models(P, nx, nu, A, B, c):
    dyn = P.TimeVaryingLinearDynamics(A, B, c)
    Q = np.eye(nx) + 0.1 * np.ones((nx, nx))
    goal = np.linspace(-0.5, 0.5, nx)
    cost = P.QuadraticCost(Q, 0.1 * np.eye(nu), 5 * Q, x_goal=goal)
    sl = np.full(nx, -np.inf)
    su = np.full(nx, np.inf)
    sl[0], su[0] = -50.0, 50.0
    box = P.BoxConstraint(nx, nu, control_lower=-2.0, control_upper=2.0, state_lower=sl,
                          state_upper=su)
    odyn = O.Linear(A, B, c)
    ocost = O.Quadratic(Q, 0.1 * np.eye(nu), 5 * Q, goal)
    obox = O.Box(nx, nu, control_lower=-2.0, control_upper=2.0, state_lower=sl, state_upper=su)
    return dyn, cost, box, odyn, ocost, obox


@pytest.mark.parametrize("nx,nu,T,executor", [(12, 4, 40, "sequential"), (12, 4, 1500, "parallel"),
                                              (8, 4, 300, "parallel"), (12, 6, 700, "auto")])
@pytest.mark.parametrize("aug_name", ["zero", "barrier", "admm"])
def test_wide_costate_and_expansion_match_oracle(nx, nu, T, executor, aug_name):
    import paper_2409_20027_b200 as P
    A, B, c, x0, u0, rng = _system(nx, nu, T, 1)
    dyn, cost, box, odyn, ocost, obox = _models(P, nx, nu, A, B, c)
    xs = O.rollout(odyn, x0, u0)
    traj = P.Trajectory(xs, u0)
    W = obox.n_total
    z = np.minimum(obox.w(xs, u0) + 0.1 * rng.standard_normal((T, W)), 0.0)
    v = 0.2 * rng.standard_normal((T, W))
    aug, oaug = {"zero": (P.ZeroAugmentation(), ("zero",)),
                 "barrier": (P.BarrierAugmentation(box, 0.1), ("barrier", obox, 0.1)),
                 "admm": (P.AdmmAugmentation(box, 0.7, z, v), ("admm", obox, 0.7, z, v))}[aug_name]
    lam = P.costate_pass(traj, cost, aug, dyn, executor=executor)
    olam = O.costate_pass(odyn, ocost, oaug, xs, u0)
    assert rel_gap(lam, olam) < 1e-10
    exp = P.hamiltonian_expansion(traj, lam, cost, aug, dyn, alpha=0.5, executor=executor)
    oexp = O.expansion(odyn, ocost, oaug, xs, u0, olam, alpha=0.5)
    for f in ("P", "R", "M", "d", "Fx", "Fu"):
        assert rel_gap(getattr(exp, f), getattr(oexp, f)) < 1e-10, f
    assert rel_gap(exp.P_terminal, oexp.PT) < 1e-12


@pytest.mark.parametrize("nx,nu,T", [(12, 4, 3000), (8, 4, 64), (12, 6, 1)])
def test_wide_rollout_matches_oracle(nx, nu, T):
    import paper_2409_20027_b200 as P
    A, B, c, x0, u0, _ = _system(nx, nu, T, 2)
    dyn = P.TimeVaryingLinearDynamics(A, B, c)
    got = P.rollout(dyn, x0, u0)
    ref = O.rollout(O.Linear(A, B, c), x0, u0)
    assert rel_gap(got.states, ref) < 1e-12
    assert np.array_equal(got.states[0], x0)


@pytest.mark.parametrize("T,k", [(9, 3), (2000, 1500)])
def test_wide_rollout_divergence_index(T, k):
    """First non-finite state index (problem.py:449-473); at T = 2000 the
    rollout runs as an affine scan and the sequential recurrence re-derives
    the index of the flagged problem."""
    import paper_2409_20027_b200 as P
    nx, nu = 12, 4
    A = np.repeat(np.eye(nx)[None], T, 0)
    A[k] *= 1e300
    A[k + 1] *= 1e300
    dyn = P.TimeVaryingLinearDynamics(A, np.zeros((T, nx, nu)), np.zeros((T, nx)))
    with pytest.raises(P.DivergenceError) as exc:
        P.rollout(dyn, np.ones(nx), np.zeros((T, nu)))
    assert exc.value.step == k + 2


@pytest.mark.parametrize("executor", ["sequential", "parallel"])
@pytest.mark.parametrize("nx,nu,T", [(12, 4, 200), (8, 4, 120), (12, 4, 1100)])
def test_wide_newton_and_barrier_match_oracle(executor, nx, nu, T):
    import paper_2409_20027_b200 as P
    A, B, c, x0, u0, _ = _system(nx, nu, T, 3)
    dyn, cost, box, odyn, ocost, obox = _models(P, nx, nu, A, B, c)
    init = P.rollout(dyn, x0, u0)
    xs = O.rollout(odyn, x0, u0)
    # unconstrained Newton
    traj, rep = P.newton_solve(dyn, cost, None, init, P.NewtonOptions(executor=executor))
    ref = O.newton_solve(odyn, ocost, ("zero",), xs, u0)
    assert rep.iterations == ref.iterations and rep.converged
    assert rel_gap(traj.controls, ref.us) < 1e-8
    assert rel_gap(traj.states, ref.xs) < 1e-8
    # barrier outer loop
    opts = P.BarrierOptions(newton=P.NewtonOptions(executor=executor))
    traj, rep = P.barrier_solve(P.ControlProblem(dyn, cost, box), init, opts)
    ref = O.barrier_solve(odyn, ocost, obox, xs, u0)
    assert [r.newton.iterations for r in rep.rounds] == [r.iterations for r in ref.newton]
    assert rel_gap(traj.controls, ref.us) < 1e-8
    assert np.abs(traj.controls).max() < 2.0


@pytest.mark.parametrize("executor", ["sequential", "parallel"])
def test_wide_admm_matches_oracle(executor):
    import paper_2409_20027_b200 as P
    nx, nu, T = 12, 4, 150
    A, B, c, x0, u0, _ = _system(nx, nu, T, 4)
    dyn, cost, box, odyn, ocost, obox = _models(P, nx, nu, A, B, c)
    init = P.rollout(dyn, x0, u0)
    xs = O.rollout(odyn, x0, u0)
    opts = P.AdmmOptions(rho=1.0, max_outer=30, newton=P.NewtonOptions(executor=executor))
    traj, rep = P.admm_solve(P.ControlProblem(dyn, cost, box), init, opts)
    ref = O.admm_solve(odyn, ocost, obox, xs, u0, rho=1.0, max_outer=30)
    assert rep.converged == ref.converged
    assert [r.iterations for r in rep.newton_reports] == [r.iterations for r in ref.newton]
    assert rel_gap(traj.controls, ref.us) < 1e-8


@pytest.mark.parametrize("executor,T", [("sequential", 200), ("parallel", 1100)])
def test_wide_batch_matches_single_solves(executor, T):
    """Several wide problems per launch sequence (warp units over problems,
    batch-strided model / trajectory gathers) reproduce the batch-1 solves."""
    import torch
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200 import BatchSolver
    nx, nu, n = 12, 4, 3
    A, B, c, _, u0, rng = _system(nx, nu, T, 5)
    dyn, cost, box, odyn, ocost, obox = _models(P, nx, nu, A, B, c)
    problem = P.ControlProblem(dyn, cost, box)
    opts = P.BarrierOptions(newton=P.NewtonOptions(executor=executor))
    x0 = rng.standard_normal((n, nx))
    U = torch.as_tensor(np.repeat(u0[None], n, 0))
    bs = BatchSolver(problem, n, "barrier", barrier=opts)
    X = bs.rollout(x0, U)
    res = bs.solve(X, U)
    for k in range(n):
        init = P.rollout(dyn, x0[k], u0)
        assert rel_gap(X[k].cpu().numpy(), init.states) < 1e-12
        traj, rep = P.barrier_solve(problem, init, opts)
        got = res.round_iters[:len(rep.rounds), k].cpu().numpy()
        assert list(got) == [r.newton.iterations for r in rep.rounds]
        assert rel_gap(res.controls[k].cpu().numpy(), traj.controls) < 1e-10


@pytest.mark.parametrize("executor", ["sequential", "parallel"])
def test_wide_newton_fp32(executor):
    """fp32 instantiation of the wide Newton kernels: converges to the fp64
    solution within single-precision accuracy (tolerance 1e-4 relative)."""
    import torch
    import paper_2409_20027_b200 as P
    nx, nu, T = 12, 4, 1100
    A, B, c, x0, u0, _ = _system(nx, nu, T, 6)
    dyn, cost, box, odyn, ocost, obox = _models(P, nx, nu, A, B, c)
    init = P.rollout(dyn, x0, u0)
    opts = P.NewtonOptions(executor=executor, inner_tol=1e-5)
    t64, r64 = P.newton_solve(dyn, cost, None, init, opts)
    t32, r32 = P.newton_solve(dyn, cost, None, init, opts, dtype=torch.float32)
    assert r32.converged
    assert rel_gap(t32.controls, t64.controls) < 1e-4
    assert abs(r32.final_cost - r64.final_cost) <= 1e-4 * abs(r64.final_cost)
