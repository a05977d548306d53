"""Edge cases and known answers of the reference's own test-suite, on the
CUDA path (through the C ABI), checked against independent oracles:

* executor equivalence over many horizons / dimensions / scan plans
  (reference acceptance criterion 1, test_pass_executor_equivalence);
* the scan solution equals a dense KKT solve of the subproblem for N <= 5
  (criterion 3, test_scan_solution_matches_kkt);
* time-invariant LQ: gains equal the classical Riccati recursion, s = 0,
  gamma = 0 (test_value_pass_matches_riccati, ..._no_gradient_...);
* single-stage horizons (test_*_single_stage), the SPEC's scalar example,
  zero feed-forward fixed point (test_propagation_zero_feedforward_...);
* rollout divergence index, telescoping rollout, log-depth vs sequential
  candidate rollout inside the Newton loop.
Tolerances: fp64 1e-9 relative unless a test says otherwise.
"""

import numpy as np
import pytest
from conftest import rel_gap

from oracle import pintoc_oracle as O

pytestmark = pytest.mark.gpu

PLANS = [(0, 0), (1, 2), (2, 3), (4, 8), ("T", 0)]


def _exp(e):
    import paper_2409_20027_b200 as P
    return P.StageExpansion.build(e.P, e.R, e.M, e.d, e.Fx, e.Fu, e.PT, e.alpha)


def _solve(e, plan):
    import torch
    from paper_2409_20027_b200 import passes
    n, nx, nu = e.P.shape[0], e.P.shape[1], e.R.shape[1]
    c0, c1 = (n, 0) if plan[0] == "T" else plan
    sol = passes.LqrSolver(1, n, nx, nu, chunk0=c0, chunk=c1, with_value=True)
    dev = sol.device
    soa = lambda a, c: passes._soa(torch, a, torch.float64, dev, c)
    args = [soa(e.P, nx * nx), soa(e.R, nu * nu), soa(e.M, nx * nu), soa(e.d, nu),
            soa(e.Fx, nx * nx), soa(e.Fu, nx * nu), soa(e.PT[None], nx * nx)]
    sol.solve(*args, torch.full((1,), float(e.alpha), dtype=torch.float64, device=dev))
    torch.cuda.synchronize()
    host = lambda t, shape: t[..., 0].t().reshape(shape).cpu().numpy()
    return (host(sol.S, (n + 1, nx, nx)), host(sol.s, (n + 1, nx)), host(sol.Gamma, (n, nu, nx)),
            host(sol.gamma, (n, nu)), host(sol.dx, (n + 1, nx)), host(sol.du, (n, nu)),
            int(sol.flags[0]))


@pytest.mark.parametrize("n", [1, 2, 3, 7, 16, 33, 64, 100])
def test_plan_equivalence_many_horizons(n):
    for nx, nu in ((1, 1), (2, 1), (3, 2), (3, 3), (4, 2)):
        e = O.random_lqr_expansion(np.random.default_rng([n, nx, nu]), n, nx, nu, alpha=0.1)
        ref = O.lqr_solve(e)
        for plan in PLANS:
            out = _solve(e, plan)
            assert out[6] == 0
            for k in range(6):
                assert rel_gap(out[k], ref[k]) < 1e-9, (n, nx, nu, plan, k)


def _kkt(e):
    """Dense KKT solve of min sum 1/2 dx'P dx + dx'M du + 1/2 du'Rr du + d'du
    + 1/2 dx_N' PT dx_N  s.t.  dx_{t+1} = Fx dx_t + Fu du_t, dx_0 = 0."""
    n, nx, nu = e.P.shape[0], e.P.shape[1], e.R.shape[1]
    nz = (n + 1) * nx + n * nu
    H = np.zeros((nz, nz))
    g = np.zeros(nz)
    xi = lambda t: slice(t * nx, (t + 1) * nx)
    ui = lambda t: slice((n + 1) * nx + t * nu, (n + 1) * nx + (t + 1) * nu)
    Rr = e.R + e.alpha * np.eye(nu)
    for t in range(n):
        H[xi(t), xi(t)] = e.P[t]
        H[ui(t), ui(t)] = Rr[t]
        H[xi(t), ui(t)] = e.M[t]
        H[ui(t), xi(t)] = e.M[t].T
        g[ui(t)] = e.d[t]
    H[xi(n), xi(n)] = e.PT
    A = np.zeros(((n + 1) * nx, nz))
    A[xi(0), xi(0)] = np.eye(nx)
    for t in range(n):
        r = slice((t + 1) * nx, (t + 2) * nx)
        A[r, xi(t + 1)] = -np.eye(nx)
        A[r, xi(t)] = e.Fx[t]
        A[r, ui(t)] = e.Fu[t]
    K = np.block([[H, A.T], [A, np.zeros((A.shape[0], A.shape[0]))]])
    sol = np.linalg.solve(K, np.concatenate([-g, np.zeros(A.shape[0])]))
    z = sol[:nz]
    return z[:(n + 1) * nx].reshape(n + 1, nx), z[(n + 1) * nx:].reshape(n, nu)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_scan_solution_matches_dense_kkt(n):
    for trial in range(4):
        nx, nu = 1 + trial % 3, 1 + trial % 2
        e = O.random_lqr_expansion(np.random.default_rng([7, n, trial]), n, nx, nu, alpha=0.5)
        dx_ref, du_ref = _kkt(e)
        for plan in PLANS:
            out = _solve(e, plan)
            assert rel_gap(out[4], dx_ref) < 1e-7, (n, trial, plan)
            assert rel_gap(out[5], du_ref) < 1e-7, (n, trial, plan)


def test_time_invariant_lq_is_classical_riccati():
    rng = np.random.default_rng(21)
    n, nx, nu = 50, 3, 2
    A = np.eye(nx) + 0.1 * rng.standard_normal((nx, nx))
    B = rng.standard_normal((nx, nu))
    Q, R, QT = np.eye(nx), 0.5 * np.eye(nu), 3 * np.eye(nx)
    e = O.Expansion(P=np.tile(Q, (n, 1, 1)), R=np.tile(R, (n, 1, 1)), M=np.zeros((n, nx, nu)),
                    d=np.zeros((n, nu)), Fx=np.tile(A, (n, 1, 1)), Fu=np.tile(B, (n, 1, 1)),
                    PT=QT, alpha=0.0)
    # textbook Riccati recursion
    S = QT.copy()
    gains = [None] * n
    for t in range(n - 1, -1, -1):
        K = -np.linalg.solve(R + B.T @ S @ B, B.T @ S @ A)
        gains[t] = K
        S = Q + A.T @ S @ A + A.T @ S @ B @ K
    for plan in PLANS:
        out = _solve(e, plan)
        assert rel_gap(out[2], np.array(gains)) < 1e-9, plan
        assert np.abs(out[1]).max() == 0.0 and np.abs(out[3]).max() == 0.0
        assert rel_gap(out[0][0], S) < 1e-9


def test_spec_scalar_value_element_example():
    """SPEC value_element_init example: P=2, Rr=1, M=0, d=1, Fx=1, Fu=1,
    terminal P_T = 0: one Bellman backup from V_2 = 0 gives S_1 = 2,
    gamma = -1, Gamma = 0."""
    e = O.Expansion(P=np.array([[[2.0]]]), R=np.array([[[1.0]]]), M=np.zeros((1, 1, 1)),
                    d=np.array([[1.0]]), Fx=np.array([[[1.0]]]), Fu=np.array([[[1.0]]]),
                    PT=np.zeros((1, 1)), alpha=0.0)
    for plan in PLANS:
        S, s, G, g, dx, du, fl = _solve(e, plan)
        assert fl == 0
        assert S[0, 0, 0] == pytest.approx(2.0) and s[0, 0] == pytest.approx(0.0)
        assert G[0, 0, 0] == pytest.approx(0.0) and g[0, 0] == pytest.approx(-1.0)
        assert du[0, 0] == pytest.approx(-1.0) and dx[1, 0] == pytest.approx(-1.0)


def test_zero_feedforward_is_fixed_point():
    e = O.random_lqr_expansion(np.random.default_rng(4), 40, 3, 2)
    e.d[:] = 0.0
    for plan in PLANS:
        out = _solve(e, plan)
        assert np.abs(out[4]).max() == 0.0 and np.abs(out[5]).max() == 0.0


def test_rollout_telescoping_and_divergence_index():
    import paper_2409_20027_b200 as P
    dyn = P.LinearDynamics(np.eye(1), np.eye(1), 3)
    traj = P.rollout(dyn, np.zeros(1), np.ones((3, 1)))
    assert np.array_equal(traj.states[:, 0], [0.0, 1.0, 2.0, 3.0])
    # reference test_rollout_divergence_reports_index: x + 1 for t < 2, then
    # x * 1e200 -> inf at step 4
    A = np.ones((6, 1, 1))
    A[2:] = 1e200
    c = np.zeros((6, 1))
    c[:2] = 1.0
    boom = P.TimeVaryingLinearDynamics(A, np.zeros((6, 1, 1)), c)
    with pytest.raises(P.DivergenceError) as exc:
        P.rollout(boom, np.ones(1), np.zeros((6, 1)))
    assert exc.value.step == 4


@pytest.mark.parametrize("T", [40, 1500])
def test_log_depth_rollout_matches_sequential_in_newton(T):
    """The Newton loop with the parallel executor (log-depth candidate
    rollout on a tree plan) reproduces the sequential executor on an LQ
    problem with time-varying affine dynamics, where the log-depth rollout
    is exact after one sweep."""
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(T)
    nx, nu = 3, 2
    A = np.eye(nx)[None] + 0.05 * rng.standard_normal((T, nx, nx))
    B = 0.3 * rng.standard_normal((T, nx, nu))
    dyn = P.TimeVaryingLinearDynamics(A, B, 0.1 * rng.standard_normal((T, nx)))
    cost = P.QuadraticCost(np.eye(nx), 0.1 * np.eye(nu), 5 * np.eye(nx))
    init = P.rollout(dyn, rng.standard_normal(nx), 0.1 * rng.standard_normal((T, nu)))
    res = {}
    for ex in ("sequential", "parallel"):
        res[ex] = P.newton_solve(dyn, cost, None, init, P.NewtonOptions(executor=ex))
    (ts, rs), (tp, rp) = res["sequential"], res["parallel"]
    assert rs.iterations == rp.iterations and rs.termination == rp.termination
    assert rel_gap(tp.controls, ts.controls) < 1e-9
    assert rel_gap(tp.states, ts.states) < 1e-9
    assert abs(rp.final_cost - rs.final_cost) <= 1e-9 * max(1.0, abs(rs.final_cost))


def test_single_stage_newton_matches_oracle():
    import paper_2409_20027_b200 as P
    dyn = P.PendulumDynamics(1, P.PendulumParams(dt=0.05))
    cost = P.QuadraticCost(np.diag([10.0, 1.0]), np.diag([0.1]), np.diag([100.0, 10.0]))
    init = P.rollout(dyn, np.array([0.3, -0.2]), np.array([[0.5]]))
    traj, rep = P.newton_solve(dyn, cost, None, init, P.NewtonOptions())
    odyn = O.Pendulum(dt=0.05)
    ocost = O.Quadratic(np.diag([10.0, 1.0]), np.diag([0.1]), np.diag([100.0, 10.0]))
    ref = O.newton_solve(odyn, ocost, ("zero",), init.states, init.controls)
    assert rep.iterations == ref.iterations
    assert rel_gap(traj.controls, ref.us) < 1e-9


def test_batch_solver_concurrent_matches_single_and_oracle():
    """Two batches advanced concurrently on two streams give the same result
    as solving them one after the other; a problem of the batch matches the
    CPU oracle's barrier solve (iteration counts and controls)."""
    import torch
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200 import BatchSolver
    T, n = 24, 5
    rng = np.random.default_rng(31)
    pend = P.ControlProblem(P.PendulumDynamics(T, P.PendulumParams(damping=0.1, dt=0.05)),
                            P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]),
                                            np.diag([100.0, 10.0])),
                            P.BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0))
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    cart = P.ControlProblem(P.CartPoleDynamics(T, P.CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                                                   pole_length=0.5, dt=0.02)),
                            P.QuadraticCost(Q, np.diag([0.01]), 10 * Q,
                                            x_goal=np.array([0.0, np.pi, 0.0, 0.0])),
                            P.BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0))
    opts = P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-3, newton=P.NewtonOptions(max_iters=40))
    jobs, singles = [], []
    for prob, nx, bound in ((pend, 2, 5.0), (cart, 4, 10.0)):
        x0 = rng.uniform(-0.3, 0.3, (n, nx))   # near the goal: a converging, well-posed solve
        u0 = torch.as_tensor(np.clip(0.1 * bound * rng.standard_normal((n, T, 1)),
                                     -0.9 * bound, 0.9 * bound))
        bs = BatchSolver(prob, n, "barrier", barrier=opts)
        xs = bs.rollout(x0, u0)
        singles.append(bs.solve(xs, u0))
        bs2 = BatchSolver(prob, n, "barrier", barrier=opts)
        jobs.append((bs2, xs, u0))
    conc = BatchSolver.solve_concurrently(jobs)
    for a, b in zip(singles, conc):
        assert torch.equal(a.status, b.status)
        assert torch.equal(a.round_iters, b.round_iters)
        assert torch.equal(a.controls, b.controls)
    # problem 0 of the pendulum batch against the oracle barrier solve
    x_init = jobs[0][1][0].cpu().numpy()
    u_init = jobs[0][2][0].numpy()
    ref = O.barrier_solve(O.Pendulum(damping=0.1, dt=0.05),
                          O.Quadratic(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0])),
                          O.Box(2, 1, control_lower=-5.0, control_upper=5.0), x_init, u_init,
                          mu0=0.1, zeta=0.2, mu_tol=1e-3, max_iters=40)
    got = conc[0].round_iters[:, 0].cpu().numpy()[:len(ref.newton)]
    assert list(got) == [r.iterations for r in ref.newton]
    assert rel_gap(conc[0].controls[0].cpu().numpy(), ref.us) < 1e-9


@pytest.mark.parametrize("nx,nu,T", [(8, 4, 1500), (12, 4, 2048), (12, 6, 1100)])
def test_wide_staged_long_horizon_matches_oracle(nx, nu, T):
    """Batch-1 wide problems with T >= 1024 run the stage-major staged path
    (transposed expansion, stage-major gains); also through two emulated
    time blocks of >= 1024 stages."""
    import torch
    from paper_2409_20027_b200.sharded import CudaBlockOps, block_bounds, emulate_ranks
    e = O.random_lqr_expansion(np.random.default_rng([nx, nu, T]), T, nx, nu, alpha=0.2)
    ref = O.lqr_solve(e)
    for plan in ((0, 0), (8, 8), (T, 0)):
        out = _solve(e, plan)
        assert out[6] == 0
        for k in range(6):
            assert rel_gap(out[k], ref[k]) < 1e-9, (plan, k)
    soa = lambda a, c: torch.as_tensor(np.asarray(a, float)).reshape(a.shape[0], c).t() \
        .contiguous().unsqueeze(-1).cuda()
    full = dict(P=soa(e.P, nx * nx), R=soa(e.R, nu * nu), M=soa(e.M, nx * nu), d=soa(e.d, nu),
                Fx=soa(e.Fx, nx * nx), Fu=soa(e.Fu, nx * nu))
    PT = soa(e.PT[None], nx * nx)
    alpha = torch.full((1,), 0.2, dtype=torch.float64, device="cuda")
    world = 2 if T >= 2048 else 1
    ops = []
    for r in range(world):
        t0, m = block_bounds(T, world, r)
        loc = {k: v[:, t0:t0 + m].contiguous() for k, v in full.items()}
        ops.append(CudaBlockOps(r, world, t0, loc["P"], loc["R"], loc["M"], loc["d"], loc["Fx"],
                                loc["Fu"], PT, alpha, nx, nu))
    emulate_ranks(ops)
    torch.cuda.synchronize()
    host = lambda t: t[..., 0].t().cpu().numpy()
    G = np.concatenate([host(o.Gamma) for o in ops]).reshape(T, nu, nx)
    du = np.concatenate([host(o.du) for o in ops])
    assert rel_gap(G, ref[2]) < 1e-9 and rel_gap(du, ref[5]) < 1e-9


def test_nan_step_is_rejected_not_converged():
    """A NaN goal makes every gradient, hence the control step, NaN.  The
    reference (newton.py:177-206) gets step_norm = NaN (not <= tol), rolls
    out u + NaN, rejects on DivergenceError with ratio -inf, and after nine
    rejections (alpha 1, 2, 8, ..., 2^36; pintoc run in the build container)
    ends 'stalled'.  NaN-propagating step-norm reduction: a NaN step must
    never read as a converged (zero) step."""
    import paper_2409_20027_b200 as P
    dyn = P.LinearDynamics(np.eye(2) * 0.9, np.array([[0.0], [1.0]]), horizon=6)
    cost = P.QuadraticCost(np.eye(2), np.eye(1), np.eye(2), x_goal=np.array([np.nan, 0.0]))
    init = P.rollout(dyn, np.array([0.5, -0.5]), np.zeros((6, 1)))
    for ex in ("sequential", "parallel"):
        _, rep = P.newton_solve(dyn, cost, None, init, P.NewtonOptions(executor=ex))
        assert rep.termination == "stalled", (ex, rep.termination)
        assert rep.iterations == 9
        assert [r.alpha for r in rep.history] == [2.0 ** (k * (k + 1) // 2) for k in range(9)]
        for r in rep.history:
            assert r.gain_ratio == -np.inf and np.isnan(r.step_norm) and not r.accepted


@pytest.mark.parametrize("model", ["pendulum", "cartpole", "tvlinear12"])
def test_device_loop_matches_host_polled_loop(model, monkeypatch):
    """ptc_solver_loop (the whole solve as one conditional-graph loop on the
    device) takes exactly the steps of the host-polled iterate / running
    loop: same status, per-round counts, launches and controls, bitwise."""
    import torch
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200 import BatchSolver
    rng = np.random.default_rng(47)
    if model == "pendulum":
        T, n, nx = 64, 37, 2
        prob = P.ControlProblem(P.PendulumDynamics(T, P.PendulumParams(damping=0.1, dt=0.05)),
                                P.QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]),
                                                np.diag([100.0, 10.0])),
                                P.BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0))
        x0 = np.stack([rng.uniform(-np.pi, np.pi, n), rng.normal(0, 0.5, n)], 1)
        u0 = torch.as_tensor(np.clip(rng.standard_normal((n, T, 1)), -4.5, 4.5))
    elif model == "cartpole":
        T, n, nx = 64, 21, 4
        Q = np.diag([1.0, 10.0, 0.1, 0.1])
        prob = P.ControlProblem(
            P.CartPoleDynamics(T, P.CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                                   pole_length=0.5, dt=0.02)),
            P.QuadraticCost(Q, np.diag([0.01]), 10 * Q, x_goal=np.array([0.0, np.pi, 0.0, 0.0])),
            P.BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0))
        x0 = rng.uniform(-0.5, 0.5, (n, nx))
        u0 = torch.as_tensor(np.clip(rng.standard_normal((n, T, 1)), -9.0, 9.0))
    else:
        T, n, nx, nu = 96, 3, 12, 4
        A = np.eye(nx) + 0.01 * rng.standard_normal((nx, nx))
        Bm = 0.1 * rng.standard_normal((nx, nu))
        prob = P.ControlProblem(P.LinearDynamics(A, Bm, T),
                                P.QuadraticCost(np.eye(nx), 0.1 * np.eye(nu), np.eye(nx)),
                                P.BoxConstraint(nx, nu, control_lower=-2.0, control_upper=2.0))
        x0 = rng.standard_normal((n, nx))
        u0 = torch.as_tensor(np.clip(0.3 * rng.standard_normal((n, T, nu)), -1.5, 1.5))
    opts = P.BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-4, newton=P.NewtonOptions(max_iters=30))
    res = {}
    for mode in ("device", "host"):
        if mode == "host":
            monkeypatch.setenv("PTC_HOST_LOOP", "1")
        bs = BatchSolver(prob, n, "barrier", barrier=opts)
        xs = bs.rollout(x0, u0)
        single = bs.solve(xs, u0)
        bs2 = BatchSolver(prob, n, "barrier", barrier=opts)
        conc = BatchSolver.solve_concurrently([(bs2, xs, u0)])[0]
        if mode == "device":
            assert bs.solver._device_loop and bs2.solver._device_loop, "device loop not built"
        res[mode] = (single, conc)
    for a, b in zip(res["device"], res["host"]):
        assert torch.equal(a.status, b.status)
        assert torch.equal(a.round_iters, b.round_iters)
        assert torch.equal(a.controls, b.controls)
        assert torch.equal(a.states, b.states)
    # one batch on the device loop, one host-polled, side by side
    monkeypatch.delenv("PTC_HOST_LOOP")
    bs3, bs4 = (BatchSolver(prob, n, "barrier", barrier=opts) for _ in range(2))
    bs4.solver._device_loop = False
    mixed = BatchSolver.solve_concurrently([(bs3, xs, u0), (bs4, xs, u0)])
    for r in mixed:
        assert torch.equal(r.status, res["host"][1].status)
        assert torch.equal(r.controls, res["host"][1].controls)
