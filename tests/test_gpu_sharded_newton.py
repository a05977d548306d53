"""Time-sharded Newton / barrier / ADMM solves (config 4's decomposition,
sharded.TimeShardedNewton over ptc_solver_block_phase) against the
single-device solve of the whole horizon.  Ranks are emulated on one device
phase by phase (all-gathers become stacks, all-reduces elementwise folds);
each rank holds a contiguous block of stages of a time-varying affine
nx = 12 / nx = 8 system.  Same Newton iteration counts per round, controls
within 1e-9 relative (the scans and cost sums associate differently)."""

import numpy as np
import pytest
from conftest import rel_gap

from test_gpu_wide_newton import _models, _system

pytestmark = pytest.mark.gpu


def _blocks(P, dyn, cost, box, settings, world, batch=1):
    from paper_2409_20027_b200.sharded import BlockNewton, split_dynamics
    out = []
    for r in range(world):
        t0, bd = split_dynamics(dyn, world, r)
        out.append((t0, bd.horizon, BlockNewton(bd, cost, box, batch, settings, r, world, t0)))
    return out


def _settings(method, n_rounds=1, **kw):
    from paper_2409_20027_b200 import _native as N
    from paper_2409_20027_b200._device import SolveSettings
    from paper_2409_20027_b200.newton import plan_chunks
    c0, c1 = plan_chunks("parallel", 0)
    m = {"barrier": N.METHOD_BARRIER, "admm": N.METHOD_ADMM, "newton": N.METHOD_NEWTON}[method]
    return SolveSettings(method=m, round_cap=n_rounds, chunk0=c0, chunk=c1, rollout=2, **kw)


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("nx,nu,T", [(12, 4, 1200), (8, 4, 700)])
def test_time_sharded_barrier_matches_whole_horizon(world, nx, nu, T):
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200.sharded import TimeShardedNewton
    A, B, c, x0, u0, _ = _system(nx, nu, T, 7)
    dyn, cost, box, *_ = _models(P, nx, nu, A, B, c)
    problem = P.ControlProblem(dyn, cost, box)
    opts = P.BarrierOptions(newton=P.NewtonOptions(executor="parallel"))
    init = P.rollout(dyn, x0, u0)
    traj, rep = P.barrier_solve(problem, init, opts)
    st = _settings("barrier", opts.rounds(), mu0=opts.mu0, zeta=opts.zeta, mu_tol=opts.mu_tol)
    blocks = _blocks(P, dyn, cost, box, st, world)
    drv = TimeShardedNewton([b for _, _, b in blocks], emulate=True)
    drv.set_initial_state(x0[None])
    Xb = drv.rollout([u0[t0:t0 + m][None] for t0, m, _ in blocks])
    X = np.concatenate([Xb[0][0].cpu().numpy()] + [x[0, 1:].cpu().numpy() for x in Xb[1:]])
    assert rel_gap(X, init.states) < 1e-12
    drv.solve(Xb, [u0[t0:t0 + m][None] for t0, m, _ in blocks])
    s0 = blocks[0][2].solver
    n_rounds = int(s0.read("round")[0])
    iters = s0.rounds("round_iters")[:n_rounds, 0].cpu().numpy()
    assert list(iters) == [r.newton.iterations for r in rep.rounds]
    U = np.concatenate([b.solver.controls()[0].cpu().numpy() for _, _, b in blocks])
    assert rel_gap(U, traj.controls) < 1e-9
    Xs = [b.solver.states()[0].cpu().numpy() for _, _, b in blocks]
    X = np.concatenate([Xs[0]] + [x[1:] for x in Xs[1:]])
    assert rel_gap(X, traj.states) < 1e-9
    # every rank holds the same per-problem control state
    for _, _, b in blocks[1:]:
        assert np.array_equal(b.solver.read("cur_cost").cpu().numpy(),
                              s0.read("cur_cost").cpu().numpy())


@pytest.mark.parametrize("world", [2, 3])
def test_time_sharded_newton_and_admm_match_whole_horizon(world):
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200 import _native as N
    from paper_2409_20027_b200.sharded import TimeShardedNewton
    nx, nu, T = 12, 4, 900
    A, B, c, x0, u0, _ = _system(nx, nu, T, 8)
    dyn, cost, box, *_ = _models(P, nx, nu, A, B, c)
    init = P.rollout(dyn, x0, u0)
    # unconstrained Newton
    traj, rep = P.newton_solve(dyn, cost, None, init, P.NewtonOptions(executor="parallel"))
    blocks = _blocks(P, dyn, cost, None, _settings("newton", aug=N.AUG_ZERO), world)
    drv = TimeShardedNewton([b for _, _, b in blocks], emulate=True)
    drv.set_initial_state(x0[None])
    drv.solve([init.states[t0:t0 + m + 1][None] for t0, m, _ in blocks],
              [u0[t0:t0 + m][None] for t0, m, _ in blocks])
    s0 = blocks[0][2].solver
    assert int(s0.read("iters")[0]) == rep.iterations
    U = np.concatenate([b.solver.controls()[0].cpu().numpy() for _, _, b in blocks])
    assert rel_gap(U, traj.controls) < 1e-9
    # ADMM (z, v per block; residual maxima all-reduced)
    opts = P.AdmmOptions(rho=1.0, max_outer=20, newton=P.NewtonOptions(executor="parallel"))
    traj, rep = P.admm_solve(P.ControlProblem(dyn, cost, box), init, opts)
    blocks = _blocks(P, dyn, cost, box, _settings("admm", opts.max_outer, rho=1.0,
                                                  max_outer=opts.max_outer), world)
    drv = TimeShardedNewton([b for _, _, b in blocks], emulate=True)
    drv.set_initial_state(x0[None])
    drv.solve([init.states[t0:t0 + m + 1][None] for t0, m, _ in blocks],
              [u0[t0:t0 + m][None] for t0, m, _ in blocks])
    s0 = blocks[0][2].solver
    n_rounds = int(s0.read("round")[0])
    assert n_rounds == rep.outer_iterations
    iters = s0.rounds("round_iters")[:n_rounds, 0].cpu().numpy()
    assert list(iters) == [r.iterations for r in rep.newton_reports]
    rp = s0.rounds("round_rp")[:n_rounds, 0].cpu().numpy()
    assert np.allclose(rp, [a for a, _ in rep.residual_history], rtol=1e-8, atol=1e-12)
    U = np.concatenate([b.solver.controls()[0].cpu().numpy() for _, _, b in blocks])
    assert rel_gap(U, traj.controls) < 1e-9


def test_block_mode_rejects_unsupported_models():
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200._device import DeviceSolver
    from paper_2409_20027_b200._native import NativeError
    dyn = P.PendulumDynamics(64, P.PendulumParams(dt=0.05))
    cost = P.QuadraticCost(np.eye(2), np.eye(1), np.eye(2))
    with pytest.raises(NativeError):
        DeviceSolver(dyn, cost, None, 1, _settings("newton", block_mode=1, block_last=1))


def test_time_sharded_batch_and_unequal_blocks():
    """Two problems per block and blocks of unequal length (T = 1201 over 3
    ranks): each problem's rounds and controls equal its whole-horizon solve."""
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200.sharded import TimeShardedNewton
    nx, nu, T, world, n = 12, 4, 1201, 3, 2
    A, B, c, _, u0, rng = _system(nx, nu, T, 9)
    dyn, cost, box, *_ = _models(P, nx, nu, A, B, c)
    problem = P.ControlProblem(dyn, cost, box)
    opts = P.BarrierOptions(newton=P.NewtonOptions(executor="parallel"))
    x0 = rng.standard_normal((n, nx))
    st = _settings("barrier", opts.rounds(), mu0=opts.mu0, zeta=opts.zeta, mu_tol=opts.mu_tol)
    blocks = _blocks(P, dyn, cost, box, st, world, batch=n)
    assert len({m for _, m, _ in blocks}) == 2
    drv = TimeShardedNewton([b for _, _, b in blocks], emulate=True)
    drv.set_initial_state(x0)
    U = [np.repeat(u0[t0:t0 + m][None], n, 0) for t0, m, _ in blocks]
    drv.solve(drv.rollout(U), U)
    s0 = blocks[0][2].solver
    for k in range(n):
        traj, rep = P.barrier_solve(problem, P.rollout(dyn, x0[k], u0), opts)
        nr = int(s0.read("round")[k])
        iters = s0.rounds("round_iters")[:nr, k].cpu().numpy()
        assert list(iters) == [r.newton.iterations for r in rep.rounds]
        Uk = np.concatenate([b.solver.controls()[k].cpu().numpy() for _, _, b in blocks])
        assert rel_gap(Uk, traj.controls) < 1e-9


def test_time_sharded_barrier_through_nccl_world1():
    """The torch.distributed path of the driver (NCCL all-gather and SUM /
    MAX / MIN all-reduces on the solver's stream) at world 1 equals the
    emulated path bit for bit."""
    import os
    import socket
    import torch.distributed as dist
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200.sharded import TimeShardedNewton
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        nx, nu, T = 12, 4, 1100
        A, B, c, x0, u0, _ = _system(nx, nu, T, 10)
        dyn, cost, box, *_ = _models(P, nx, nu, A, B, c)
        opts = P.BarrierOptions(newton=P.NewtonOptions(executor="parallel"))
        st = _settings("barrier", opts.rounds(), mu0=opts.mu0, zeta=opts.zeta, mu_tol=opts.mu_tol)
        res = []
        for emulate in (True, False):
            (_, _, blk), = _blocks(P, dyn, cost, box, st, 1)
            drv = TimeShardedNewton([blk], emulate=emulate)
            drv.set_initial_state(x0[None])
            U = [u0[None]]
            drv.solve(drv.rollout(U), U)
            res.append((blk.solver.controls()[0].cpu().numpy(),
                        blk.solver.rounds("round_iters")[:, 0].cpu().numpy()))
        assert np.array_equal(res[0][0], res[1][0])
        assert np.array_equal(res[0][1], res[1][1])
    finally:
        dist.destroy_process_group()


def test_time_sharded_fp32_solve_close_to_fp64():
    """fp32 block-mode solvers (2 emulated ranks): converged controls within
    single-precision accuracy of the fp64 whole-horizon solve (1e-3)."""
    import torch
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200 import _native as N
    from paper_2409_20027_b200.sharded import BlockNewton, TimeShardedNewton, split_dynamics
    nx, nu, T, world = 12, 4, 1000, 2
    A, B, c, x0, u0, _ = _system(nx, nu, T, 11)
    dyn, cost, *_ = _models(P, nx, nu, A, B, c)
    init = P.rollout(dyn, x0, u0)
    traj, _ = P.newton_solve(dyn, cost, None, init, P.NewtonOptions(executor="parallel"))
    st = _settings("newton", aug=N.AUG_ZERO, inner_tol=1e-5)
    blocks = []
    for r in range(world):
        t0, bd = split_dynamics(dyn, world, r)
        blocks.append((t0, bd.horizon, BlockNewton(bd, cost, None, 1, st, r, world, t0,
                                                   dtype=torch.float32)))
    drv = TimeShardedNewton([b for _, _, b in blocks], emulate=True)
    drv.set_initial_state(x0[None])
    drv.solve([init.states[t0:t0 + m + 1][None] for t0, m, _ in blocks],
              [u0[t0:t0 + m][None] for t0, m, _ in blocks])
    assert int(blocks[0][2].solver.read("status")[0]) == 1   # done
    U = np.concatenate([b.solver.controls()[0].double().cpu().numpy() for _, _, b in blocks])
    assert rel_gap(U, traj.controls) < 1e-3
