"""BASELINE sizes through size-independent properties (the oracle cannot
solve these sizes in test time):

* config 3 -- 65,536 LQR subproblems (32,768 pendulum + 32,768 cart-pole,
  T = 256, fp64) built exactly as bench.py builds them: every stage of every
  problem satisfies the subproblem's KKT conditions
      Rr du_t + M^T dx_t + d_t + Fu^T (S_{t+1} dx_{t+1} + s_{t+1}) = 0,
      dx_{t+1} = Fx dx_t + Fu du_t,  dx_0 = 0,  du_t = Gamma_t dx_t + gamma_t
  (reference passes.py:291-361), and a sample of problems equals the
  oracle's solve;
* config 4 -- one T = 2^20, nx = 12, nu = 4 LQR solve, whole and as two
  time blocks: the same KKT residuals at every stage, and the two
  decompositions agree.
Residuals relative to the magnitude of the terms, 1e-9.
"""

import numpy as np
import pytest
from conftest import rel_gap

from oracle import pintoc_oracle as O

pytestmark = pytest.mark.gpu


def _kkt_residuals(torch, P, R, M, d, Fx, Fu, alpha, S, s, G, g, dx, du, nx, nu):
    """max relative residual of stationarity, dynamics and the feedback law
    over every stage of every problem (SoA (comps, rows, B) tensors)."""
    T, B = du.shape[1], du.shape[2]
    mat = lambda t, r, c: t.permute(2, 1, 0).reshape(B, -1, r, c)   # (B, rows, r, c)
    vec = lambda t: t.permute(2, 1, 0)                               # (B, rows, n)
    Rr = mat(R, nu, nu) + alpha.view(B, 1, 1, 1) * torch.eye(nu, dtype=R.dtype, device=R.device)
    Mm, Fxm, Fum = mat(M, nx, nu), mat(Fx, nx, nx), mat(Fu, nx, nu)
    Sm, sv = mat(S, nx, nx), vec(s)
    dxv, duv, dv = vec(dx), vec(du), vec(d)
    x0, x1 = dxv[:, :T], dxv[:, 1:]
    mv = lambda A, v: (A @ v.unsqueeze(-1)).squeeze(-1)
    mtv = lambda A, v: (A.transpose(-1, -2) @ v.unsqueeze(-1)).squeeze(-1)
    lam = mv(Sm[:, 1:], x1) + sv[:, 1:]
    terms = [mv(Rr, duv), mtv(Mm, x0), dv, mtv(Fum, lam)]
    scale = max(1.0, max(float(t.abs().max()) for t in terms))
    stat = float((terms[0] + terms[1] + terms[2] + terms[3]).abs().max()) / scale
    pred = mv(Fxm, x0) + mv(Fum, duv)
    dyn = float((x1 - pred).abs().max()) / max(1.0, float(pred.abs().max()))
    law = mv(mat(G, nu, nx), x0) + vec(g)
    fb = float((duv - law).abs().max()) / max(1.0, float(law.abs().max()))
    return stat, dyn, fb, float(dxv[:, 0].abs().max())


def test_config3_full_size_kkt_and_oracle_sample():
    import torch
    import bench
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200.passes import LqrSolver
    T = bench.T
    for system in ("pendulum", "cartpole"):
        n = 32768
        inputs, nx, nu = bench.build_inputs(P, torch, system, n, 0)
        alpha = bench.lm_alpha_device(torch, LqrSolver(n, T, nx, nu), inputs, n)
        sol = LqrSolver(n, T, nx, nu, with_value=True)
        sol.solve(*inputs, alpha)
        torch.cuda.synchronize()
        ok = sol.flags == 0
        assert float(ok.double().mean()) > 0.99, system
        sel = torch.nonzero(ok).flatten()
        pick = lambda t: t[..., sel]
        Pm, Rm, Mm, dm, Fxm, Fum, _ = (pick(t) for t in inputs)
        stat, dyn, fb, x0 = _kkt_residuals(torch, Pm, Rm, Mm, dm, Fxm, Fum, alpha[sel],
                                           pick(sol.S), pick(sol.s), pick(sol.Gamma),
                                           pick(sol.gamma), pick(sol.dx), pick(sol.du), nx, nu)
        assert stat < 1e-9 and dyn < 1e-12 and fb < 1e-12 and x0 == 0.0, (system, stat, dyn, fb)
        # a sample of problems against the oracle
        host = lambda t, b, shape: t[:, :, b].t().reshape(shape).cpu().numpy()
        for b in [int(v) for v in sel[:: max(1, len(sel) // 6)][:6]]:
            e = O.Expansion(P=host(inputs[0], b, (T, nx, nx)), R=host(inputs[1], b, (T, nu, nu)),
                            M=host(inputs[2], b, (T, nx, nu)), d=host(inputs[3], b, (T, nu)),
                            Fx=host(inputs[4], b, (T, nx, nx)), Fu=host(inputs[5], b, (T, nx, nu)),
                            PT=inputs[6][:, 0, b].reshape(nx, nx).cpu().numpy(),
                            alpha=float(alpha[b]))
            ref = O.lqr_solve(e)
            assert rel_gap(host(sol.du, b, (T, nu)), ref[5]) < 1e-9, (system, b)
            assert rel_gap(host(sol.dx, b, (T + 1, nx)), ref[4]) < 1e-9, (system, b)
        # the flagged problems are ones the reference rejects too
        # (passes.py:231-241: a non-positive-definite R + alpha I or Q)
        bad = torch.nonzero(~ok).flatten()
        for b in [int(v) for v in bad[:: max(1, len(bad) // 6)][:6]]:
            e = O.Expansion(P=host(inputs[0], b, (T, nx, nx)), R=host(inputs[1], b, (T, nu, nu)),
                            M=host(inputs[2], b, (T, nx, nu)), d=host(inputs[3], b, (T, nu)),
                            Fx=host(inputs[4], b, (T, nx, nx)), Fu=host(inputs[5], b, (T, nx, nu)),
                            PT=inputs[6][:, 0, b].reshape(nx, nx).cpu().numpy(),
                            alpha=float(alpha[b]))
            with pytest.raises((O.Definiteness, O.Conditioning)):
                O.lqr_solve(e)
        del inputs, sol
        torch.cuda.empty_cache()


def test_config4_full_size_kkt_whole_and_time_blocks():
    import torch
    from paper_2409_20027_b200.passes import LqrSolver
    from paper_2409_20027_b200.sharded import CudaBlockOps, block_bounds, emulate_ranks
    T, nx, nu = 1 << 20, 12, 4
    dev = torch.device("cuda")
    f64 = torch.float64
    g = torch.Generator(device=dev).manual_seed(4)
    F = torch.randn(T, nx, nx, generator=g, device=dev, dtype=f64) * (0.2 ** 0.5)
    A = torch.eye(nx, dtype=f64, device=dev) + 0.01 * F
    del F
    Bm = torch.randn(T, nx, nu, generator=g, device=dev, dtype=f64) * (0.1 ** 0.5)
    qd = torch.empty(nx, dtype=f64, device=dev).uniform_(0.1, 10.0, generator=g)
    c = torch.randn(T, nx, generator=g, device=dev, dtype=f64) * 0.1
    soa = lambda t, comps: t.reshape(-1, comps).t().contiguous().unsqueeze(-1)
    ins = [soa(torch.diag(qd).expand(T, nx, nx), nx * nx),
           soa((0.1 * torch.eye(nu, dtype=f64, device=dev)).expand(T, nu, nu), nu * nu),
           torch.zeros(nx * nu, T, 1, dtype=f64, device=dev),
           soa(torch.einsum("tij,ti->tj", Bm, c), nu), soa(A, nx * nx), soa(Bm, nx * nu),
           (10.0 * torch.diag(qd)).reshape(nx * nx, 1, 1).contiguous()]
    del A, Bm, c
    alpha = torch.zeros(1, dtype=f64, device=dev)
    sol = LqrSolver(1, T, nx, nu, with_value=True)
    sol.solve(*ins, alpha)
    torch.cuda.synchronize()
    assert int(sol.flags[0]) == 0
    stat, dyn, fb, x0 = _kkt_residuals(torch, *ins[:6], alpha, sol.S, sol.s, sol.Gamma,
                                       sol.gamma, sol.dx, sol.du, nx, nu)
    assert stat < 1e-9 and dyn < 1e-12 and fb < 1e-12 and x0 == 0.0, (stat, dyn, fb)
    # the same solve as two time blocks
    ops = []
    for r in range(2):
        t0, m = block_bounds(T, 2, r)
        loc = [t[:, t0:t0 + m].contiguous() for t in ins[:6]]
        ops.append(CudaBlockOps(r, 2, t0, *loc, ins[6], alpha, nx, nu))
    emulate_ranks(ops)
    torch.cuda.synchronize()
    du = torch.cat([o.du for o in ops], 1)
    dx = torch.cat([ops[0].dx[:, :-1], ops[1].dx], 1)
    scale = max(1.0, float(sol.du.abs().max()))
    assert float((du - sol.du).abs().max()) / scale < 1e-9
    assert float((dx - sol.dx).abs().max()) / max(1.0, float(sol.dx.abs().max())) < 1e-9


def test_config4_full_size_barrier_solve_properties():
    """Config 4 as a full barrier solve (T = 2^20, nx = 12, nu = 4, |u| <= 2;
    A scaled by 0.9999 as in bench.py): every round converges, the returned
    controls are strictly inside the box and the trajectory satisfies the
    dynamics at every stage."""
    import torch
    import paper_2409_20027_b200 as P
    T, nx, nu = 1 << 20, 12, 4
    dev = torch.device("cuda")
    f64 = torch.float64
    g = torch.Generator(device=dev).manual_seed(5)
    band = torch.zeros(nx, nx, dtype=f64, device=dev)
    for i in range(4):
        for j in (i, i + 1):
            if j < 4:
                band[3 * i:3 * i + 3, 3 * j:3 * j + 3] = 1.0
    F = torch.randn(T, nx, nx, generator=g, device=dev, dtype=f64) * (0.2 ** 0.5) * band
    A = (0.9999 * (torch.eye(nx, dtype=f64, device=dev) + 0.01 * F)).cpu().numpy()
    del F
    B = (torch.randn(T, nx, nu, generator=g, device=dev, dtype=f64) * (0.1 ** 0.5)).cpu().numpy()
    qd = np.random.default_rng(5).uniform(0.1, 10.0, nx)
    dyn = P.TimeVaryingLinearDynamics(A, B)
    cost = P.QuadraticCost(np.diag(qd), 0.1 * np.eye(nu), 10 * np.diag(qd))
    box = P.BoxConstraint(nx, nu, control_lower=-2.0, control_upper=2.0)
    x0 = np.random.default_rng(6).standard_normal(nx)
    init = P.rollout(dyn, x0, np.zeros((T, nu)))
    traj, rep = P.barrier_solve(P.ControlProblem(dyn, cost, box), init,
                                P.BarrierOptions(newton=P.NewtonOptions(max_iters=50)))
    assert rep.converged and rep.outer_iterations == 5
    assert np.abs(traj.controls).max() < 2.0
    xs = torch.as_tensor(traj.states, device=dev)
    us = torch.as_tensor(traj.controls, device=dev)
    At, Bt = torch.as_tensor(A, device=dev), torch.as_tensor(B, device=dev)
    pred = (At @ xs[:-1].unsqueeze(-1) + Bt @ us.unsqueeze(-1)).squeeze(-1)
    assert float((pred - xs[1:]).abs().max()) / max(1.0, float(xs.abs().max())) < 1e-9
    assert all(np.isfinite(r.cost) for r in rep.rounds)


@pytest.mark.parametrize("world", [1, 2])
def test_block_solve_from_stage_rows_equals_component_layout(world):
    """ptc_lqr_block_solve_rows (the expansion as stage rows, no transpose)
    gives bit-identical gains and deviations to the component-major entry."""
    import torch
    from paper_2409_20027_b200.sharded import CudaBlockOps, block_bounds, emulate_ranks
    T, nx, nu = 4096, 12, 4
    e = O.random_lqr_expansion(np.random.default_rng(12), T, nx, nu, alpha=0.2)
    dev = torch.device("cuda")
    flat = lambda a: torch.as_tensor(np.ascontiguousarray(a)).reshape(T, -1).to(dev)
    fields = [flat(e.P), flat(e.R), flat(e.M), flat(e.d), flat(e.Fx), flat(e.Fu)]
    PT = torch.as_tensor(e.PT).reshape(nx * nx, 1, 1).to(dev)
    alpha = torch.full((1,), 0.2, dtype=torch.float64, device=dev)
    outs = []
    for use_rows in (False, True):
        ops = []
        for r in range(world):
            t0, m = block_bounds(T, world, r)
            if use_rows:
                rows = torch.cat([f[t0:t0 + m] for f in fields], 1).contiguous()
                ops.append(CudaBlockOps.from_rows(r, world, t0, rows, PT, alpha, nx, nu))
            else:
                loc = [f[t0:t0 + m].t().contiguous().unsqueeze(-1) for f in fields]
                ops.append(CudaBlockOps(r, world, t0, *loc, PT, alpha, nx, nu))
        emulate_ranks(ops)
        torch.cuda.synchronize()
        outs.append([torch.cat([getattr(o, n) for o in ops], 1)
                     for n in ("Gamma", "gamma", "du")])
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    ref = O.lqr_solve(e)
    du = outs[1][2][..., 0].t().cpu().numpy()
    assert rel_gap(du, ref[5]) < 1e-9


@pytest.mark.parametrize("nx,nu,T", [(12, 4, 1100), (8, 4, 2048)])
def test_pass_level_lqr_from_stage_rows(nx, nu, T):
    """value_pass / propagation_pass on a StageExpansion with nx >= 8 and
    T >= 1024 hand the reference's per-stage arrays to the device as stage
    rows (ptc_lqr_solve_rows): bit-identical to the component-major entry,
    within 1e-9 of the oracle."""
    import torch
    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200 import passes
    e = O.random_lqr_expansion(np.random.default_rng([nx, T]), T, nx, nu, alpha=0.3)
    exp = P.StageExpansion.build(e.P, e.R, e.M, e.d, e.Fx, e.Fu, e.PT, 0.3)
    S, s, law, dxs, dus = passes.lqr_solve(exp)
    ref = O.lqr_solve(e)
    assert rel_gap(dus, ref[5]) < 1e-9 and rel_gap(dxs, ref[4]) < 1e-9
    assert rel_gap(law.Gamma, ref[2]) < 1e-9 and rel_gap(S, ref[0]) < 1e-9
    sol = passes.LqrSolver(1, T, nx, nu)
    soa = lambda a, c: passes._soa(torch, a, torch.float64, sol.device, c)
    sol.solve(soa(e.P, nx * nx), soa(e.R, nu * nu), soa(e.M, nx * nu), soa(e.d, nu),
              soa(e.Fx, nx * nx), soa(e.Fu, nx * nu), soa(e.PT[None], nx * nx),
              torch.full((1,), 0.3, dtype=torch.float64, device=sol.device))
    host = lambda t, shape: t[..., 0].t().reshape(shape).cpu().numpy()
    assert np.array_equal(host(sol.du, (T, nu)), dus)
