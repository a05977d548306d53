"""GPU parity of the LQR-scan solve (value pass + propagation pass).

CUDA path (through the C ABI) vs the reference's own outputs (golden
fixtures) and vs the pinned CPU oracle on seeded inputs, across scan plans:
sequential sweep, default tree, and a deliberately deep binary tree.
Tolerances: fp64 1e-9 relative (BASELINE north_star), fp32 1e-4.
"""

import numpy as np
import pytest
from conftest import golden, rel_gap

from oracle import pintoc_oracle as O

pytestmark = pytest.mark.gpu

PLANS = [("sequential", None), ("auto", (0, 0)), ("deep", (2, 2)), ("wide", (3, 5))]


def _exp_from_golden(g, p):
    import paper_2409_20027_b200 as P
    return P.StageExpansion.build(g[p + "P"], g[p + "R"], g[p + "M"], g[p + "d"], g[p + "Fx"],
                                  g[p + "Fu"], g[p + "PT"], float(g[p + "alpha"]))


def _solve(exp, plan, dtype=None):
    import torch
    from paper_2409_20027_b200 import passes
    n, nx, nu = exp.horizon, exp.d_x, exp.d_u
    if plan[0] == "sequential":
        c0, c1 = n, 0
    else:
        c0, c1 = plan[1]
    dtype = dtype or torch.float64
    solver = passes.LqrSolver(1, n, nx, nu, dtype=dtype, chunk0=c0, chunk=c1, with_value=True)
    dev = solver.device
    soa = lambda a, c: passes._soa(torch, a, dtype, dev, c)
    args = [soa(exp.P, nx * nx), soa(exp.R, nu * nu), soa(exp.M, nx * nu), soa(exp.d, nu),
            soa(exp.Fx, nx * nx), soa(exp.Fu, nx * nu), soa(exp.P_terminal[None], nx * nx)]
    alpha = torch.full((1,), float(exp.alpha), dtype=torch.float64, device=dev)
    solver.solve(*args, alpha)
    torch.cuda.synchronize()
    host = lambda t, shape: t[..., 0].t().reshape(shape).double().cpu().numpy()
    return (host(solver.S, (n + 1, nx, nx)), host(solver.s, (n + 1, nx)),
            host(solver.Gamma, (n, nu, nx)), host(solver.gamma, (n, nu)),
            host(solver.dx, (n + 1, nx)), host(solver.du, (n, nu)), int(solver.flags[0]))


@pytest.mark.parametrize("plan", PLANS, ids=[p[0] for p in PLANS])
def test_lqr_small_matches_reference(plan):
    g = golden("lqr_small")
    for i in range(int(g["count"])):
        p = f"{i}_"
        S, s, Gam, gam, dxs, dus, fl = _solve(_exp_from_golden(g, p), plan)
        assert fl == 0
        for name, val in dict(S=S, s=s, Gamma=Gam, gamma=gam, dxs=dxs, dus=dus).items():
            assert rel_gap(val, g[p + name]) < 1e-9, (i, name, plan)


@pytest.mark.parametrize("plan", PLANS, ids=[p[0] for p in PLANS])
def test_lqr_config1_matches_reference(plan):
    g = golden("lqr_config1")
    for nx in (2, 4, 8, 12):
        p = f"{nx}_"
        S, s, Gam, gam, dxs, dus, fl = _solve(_exp_from_golden(g, p), plan)
        assert fl == 0
        for name, val in dict(S=S, s=s, Gamma=Gam, gamma=gam, dxs=dxs, dus=dus).items():
            assert rel_gap(val, g[p + name]) < 1e-9, (nx, name, plan)


@pytest.mark.parametrize("nx,T", [(2, 4096), (4, 2048), (8, 512), (12, 256)])
def test_lqr_long_horizon_vs_oracle(nx, T):
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(7000 + nx)
    e = O.random_lqr_expansion(rng, T, nx, nx // 2)
    ref = O.lqr_solve(e)
    exp = P.StageExpansion.build(e.P, e.R, e.M, e.d, e.Fx, e.Fu, e.PT, 0.0)
    for plan in PLANS:
        S, s, Gam, gam, dxs, dus, fl = _solve(exp, plan)
        assert fl == 0
        for k, val in enumerate((S, s, Gam, gam, dxs, dus)):
            assert rel_gap(val, ref[k]) < 1e-9, (nx, T, plan[0], k)


def test_lqr_fp32_within_tolerance():
    import torch
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(11)
    e = O.random_lqr_expansion(rng, 256, 4, 2)
    ref = O.lqr_solve(e)
    exp = P.StageExpansion.build(e.P, e.R, e.M, e.d, e.Fx, e.Fu, e.PT, 0.0)
    for plan in PLANS:
        out = _solve(exp, plan, dtype=torch.float32)
        for k in range(6):
            assert rel_gap(out[k], ref[k]) < 1e-4, (plan[0], k)


def test_lqr_batch_matches_per_problem_oracle():
    """B independent problems in one launch (SoA batch-minor layout)."""
    import torch
    from paper_2409_20027_b200 import passes
    B, T, nx, nu = 37, 64, 3, 2
    rng = np.random.default_rng(5)
    exps = [O.random_lqr_expansion(rng, T, nx, nu, alpha=0.3 * b / B) for b in range(B)]
    for c0, c1 in [(T, 0), (0, 0), (2, 3)]:
        sol = passes.LqrSolver(B, T, nx, nu, chunk0=c0, chunk=c1, with_value=True)
        dev = sol.device
        stack = lambda f, c: torch.as_tensor(np.stack([f(e).reshape(T, c) for e in exps], -1)
                                             ).permute(1, 0, 2).contiguous().to(dev)
        args = [stack(lambda e: e.P, nx * nx), stack(lambda e: e.R, nu * nu),
                stack(lambda e: e.M, nx * nu), stack(lambda e: e.d, nu),
                stack(lambda e: e.Fx, nx * nx), stack(lambda e: e.Fu, nx * nu),
                torch.as_tensor(np.stack([e.PT.reshape(1, nx * nx) for e in exps], -1)
                                ).permute(1, 0, 2).contiguous().to(dev)]
        alpha = torch.tensor([e.alpha for e in exps], dtype=torch.float64, device=dev)
        sol.solve(*args, alpha)
        du = sol.du.permute(2, 1, 0).cpu().numpy()
        G = sol.Gamma.permute(2, 1, 0).cpu().numpy().reshape(B, T, nu, nx)
        for b in (0, 17, B - 1):
            ref = O.lqr_solve(exps[b])
            assert rel_gap(du[b], ref[5]) < 1e-9
            assert rel_gap(G[b], ref[2]) < 1e-9


def test_propagation_of_foreign_law_matches_oracle():
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(3)
    e = O.random_lqr_expansion(rng, 40, 3, 2)
    exp = P.StageExpansion.build(e.P, e.R, e.M, e.d, e.Fx, e.Fu, e.PT, 0.0)
    law = P.FeedbackLaw(rng.normal(size=(40, 2, 3)), rng.normal(size=(40, 2)))
    dxs, dus = P.propagation_pass(law, exp)
    rx, ru = O.propagation_pass(law.Gamma, law.gamma, e)
    assert rel_gap(dxs, rx) < 1e-10 and rel_gap(dus, ru) < 1e-10
    law0 = P.FeedbackLaw(law.Gamma, np.zeros((40, 2)))
    dxs, dus = P.propagation_pass(law0, exp)
    assert np.allclose(dxs, 0.0) and np.allclose(dus, 0.0)


def test_indefinite_regularised_r_raises_definiteness():
    import paper_2409_20027_b200 as P
    exp = P.StageExpansion.build(np.eye(1)[None], np.array([[[-1.0]]]), np.zeros((1, 1, 1)),
                                 np.zeros((1, 1)), np.eye(1)[None], np.eye(1)[None],
                                 np.zeros((1, 1)))
    with pytest.raises(P.DefinitenessError):
        P.value_pass(exp)


def test_value_pass_pure_regularisation_is_zero():
    import paper_2409_20027_b200 as P
    n = 5
    exp = P.StageExpansion.build(np.zeros((n, 2, 2)), np.zeros((n, 1, 1)), np.zeros((n, 2, 1)),
                                 np.zeros((n, 1)), np.tile(np.eye(2), (n, 1, 1)),
                                 np.ones((n, 2, 1)), np.zeros((2, 2)), alpha=4.0)
    S, s, law = P.value_pass(exp)
    assert np.allclose(S, 0.0) and np.allclose(law.Gamma, 0.0) and np.allclose(law.gamma, 0.0)


@pytest.mark.parametrize("nx,nu,T,B", [(2, 1, 256, 64), (4, 1, 256, 300), (4, 2, 1024, 3),
                                       (12, 4, 1500, 1)])
def test_lqr_host_buffers_equal_device_solve(nx, nu, T, B):
    """ptc_lqr_solve_host (host tensors in and out, copies on the solver's
    stream) gives bit-identical gains and deviations to the device entry on
    the same inputs; for nx < 8 the strictly-lower triangles of the host P
    and R are NaN, proving only the upper triangles the kernels read cross
    PCIe."""
    import torch
    from paper_2409_20027_b200 import passes
    rng = np.random.default_rng([nx, nu, T, B])
    exps = [O.random_lqr_expansion(rng, T, nx, nu, alpha=0.2) for _ in range(B)]
    stack = lambda f, c: torch.as_tensor(np.stack([f(e).reshape(-1, c) for e in exps], -1)
                                         ).permute(1, 0, 2).contiguous()
    h = [stack(lambda e: e.P, nx * nx), stack(lambda e: e.R, nu * nu),
         stack(lambda e: e.M, nx * nu), stack(lambda e: e.d, nu), stack(lambda e: e.Fx, nx * nx),
         stack(lambda e: e.Fu, nx * nu), stack(lambda e: e.PT[None], nx * nx)]
    alpha = torch.full((B,), 0.2, dtype=torch.float64)
    dev = passes.LqrSolver(B, T, nx, nu)
    dev.solve(*[t.cuda() for t in h], alpha.cuda())
    if nx < 8:
        for t, n in ((h[0], nx), (h[1], nu)):
            for i in range(n):
                for j in range(i):
                    t[i * n + j] = float("nan")
    hs = passes.HostLqrSolver(B, T, nx, nu)
    out = hs.outputs()
    flags = torch.zeros(B, dtype=torch.int32).pin_memory()
    h = [t.pin_memory() for t in h]
    s = torch.cuda.Stream()
    hs.solve(*h, alpha.pin_memory(), out, flags=flags, stream=s)
    s.synchronize()
    assert int(flags.max()) == 0
    for got, want in zip(out, (dev.Gamma, dev.gamma, dev.dx, dev.du)):
        assert torch.equal(got, want.cpu())


@pytest.mark.parametrize("nx,nu,T,B", [(2, 1, 256, 64), (4, 1, 256, 300), (4, 2, 100, 33),
                                       (12, 4, 1500, 1), (3, 2, 7, 5)])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_lqr_host_stacked_equals_soa_solve(nx, nu, T, B, dtype):
    """ptc_lqr_solve_host_stacked takes the reference's per-problem arrays
    (np.stack of each StageExpansion field over the batch) and returns the
    gains and deviations in the same stacking -- bit-identical to the SoA
    host entry on the same problems, with ragged batch / component counts
    (not multiples of the 32 x 32 restack tile)."""
    import torch
    from paper_2409_20027_b200 import passes
    td = torch.float64 if dtype == "f64" else torch.float32
    rng = np.random.default_rng([nx, nu, T, B, 7])
    exps = [O.random_lqr_expansion(rng, T, nx, nu, alpha=0.2) for _ in range(B)]
    fields = (lambda e: e.P, lambda e: e.R, lambda e: e.M, lambda e: e.d, lambda e: e.Fx,
              lambda e: e.Fu, lambda e: e.PT[None])
    stacked = [torch.as_tensor(np.stack([f(e) for e in exps]), dtype=td) for f in fields]
    stacked[6] = stacked[6].reshape(B, nx, nx)
    soa = [t.reshape(B, t.shape[1] if i < 6 else 1, -1).permute(2, 1, 0).contiguous()
           for i, t in enumerate(stacked)]
    alpha = torch.full((B,), 0.2, dtype=torch.float64).pin_memory()
    s = torch.cuda.Stream()
    ref = passes.HostLqrSolver(B, T, nx, nu, dtype=td)
    want = ref.outputs()
    # (the pinned inputs stay referenced until the stream is synchronised:
    # torch's host allocator does not see the C ABI's async copies, so a
    # dropped buffer could be handed out again before its copy has run)
    ins_soa = [t.pin_memory() for t in soa]
    ref.solve(*ins_soa, alpha, want, stream=s)
    hs = passes.HostLqrSolver(B, T, nx, nu, dtype=td, stacked=True)
    got = hs.outputs()
    flags = torch.zeros(B, dtype=torch.int32).pin_memory()
    ins_st = [t.contiguous().pin_memory() for t in stacked]
    hs.solve(*ins_st, alpha, got, flags=flags, stream=s)
    s.synchronize()
    del ins_soa, ins_st
    assert int(flags.max()) == 0
    assert got[0].shape == (B, T, nu, nx) and got[2].shape == (B, T + 1, nx)
    for g, w in zip(got, want):
        w = w.reshape(-1, g.shape[1], B).permute(2, 1, 0).reshape(g.shape)
        assert torch.equal(g, w)
    if dtype == "f64":  # one problem against the oracle's value + propagation pass
        k = B // 2
        _, _, Gam, gam, dxs, dus = O.lqr_solve(exps[k])
        for g, w in zip(got, (Gam, gam, dxs, dus)):
            g = g[k].numpy()
            assert np.max(np.abs(g - w)) <= 1e-9 * max(1.0, np.max(np.abs(w)))


@pytest.mark.parametrize("nx,nu", [(2, 1), (4, 2), (12, 4)])
def test_definiteness_error_names_the_reference_stage(nx, nu):
    """DefinitenessError.stage is the stage the reference's gates name
    (passes.py:231-241): the first stage whose R + alpha I fails, else the
    first stage whose Q_t = Rr + Fu^T S_{t+1} Fu fails; checked against the
    oracle's value_pass on the same expansions."""
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(nx)
    T = 40
    e = O.random_lqr_expansion(rng, T, nx, nu)
    # (a) R + alpha I indefinite at stages 17 and 29 -> 17
    R = e.R.copy()
    R[17] = -np.eye(nu)
    R[29] = -np.eye(nu)
    exp = P.StageExpansion.build(e.P, R, e.M, e.d, e.Fx, e.Fu, e.PT, 0.0)
    with pytest.raises(O.Definiteness) as want:
        O.value_pass(O.Expansion(e.P, R, e.M, e.d, e.Fx, e.Fu, e.PT, 0.0))
    with pytest.raises(P.DefinitenessError) as got:
        P.value_pass(exp)
    assert got.value.stage == want.value.stage == 17 and got.value.what == "R + alpha*I"
    # (b) R fine, Q_t indefinite through strongly negative P at two stages
    Pm = e.P.copy()
    Pm[8] = -60.0 * np.eye(nx)
    Pm[25] = -60.0 * np.eye(nx)
    oe = O.Expansion(Pm, e.R, e.M, e.d, e.Fx, e.Fu, e.PT, 0.0)
    with pytest.raises(O.Definiteness) as want:
        O.value_pass(oe)
    with pytest.raises(P.DefinitenessError) as got:
        P.value_pass(P.StageExpansion.build(Pm, e.R, e.M, e.d, e.Fx, e.Fu, e.PT, 0.0))
    assert got.value.what == "Q" and got.value.stage == want.value.stage >= 0


def test_infeasible_error_carries_the_constraint_value():
    """InfeasibleError(stage, component, value) from a barrier Newton solve
    entered at an infeasible point (outer.py:47-52: the value is w >= 0)."""
    import paper_2409_20027_b200 as P
    T = 8
    dyn = P.LinearDynamics(np.eye(2) * 0.9, np.array([[0.0], [1.0]]), horizon=T)
    cost = P.QuadraticCost(np.eye(2), np.eye(1), np.eye(2))
    box = P.BoxConstraint(2, 1, control_lower=-1.0, control_upper=1.0)
    us = np.zeros((T, 1))
    us[5, 0] = 1.25                       # w = u - 1 = 0.25 at stage 5, row 1 (upper bound)
    init = P.rollout(dyn, np.array([0.5, -0.5]), us)
    with pytest.raises(P.InfeasibleError) as err:
        P.newton_solve(dyn, cost, P.BarrierAugmentation(box, 0.1), init)
    ob = O.Box(2, 1, control_lower=-1.0, control_upper=1.0)
    w = ob.w(init.states[:-1], us)
    st, comp = np.argwhere(w >= 0)[0]
    assert (err.value.stage, err.value.component) == (st, comp)
    assert err.value.value == w[st, comp]


@pytest.mark.parametrize("nx,nu,B", [(2, 1, 2050), (4, 1, 4096), (4, 2, 2048), (3, 2, 2049)])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_bulk_ring_sweeps_match_register_path(nx, nu, B, dtype, monkeypatch):
    """With PTC_BULK=1 the single-sweep plan at batches >= 2048 runs the
    TMA-fed ring kernels (bulk_sweeps.cuh; an odd batch keeps the register
    path): same results as the blocked-tree plan and the oracle, S / s
    included, partial last tile (B % 128 != 0) included."""
    import torch

    import paper_2409_20027_b200 as P
    from paper_2409_20027_b200.passes import LqrSolver
    rng = np.random.default_rng(B + nx)
    T = 48
    dt = torch.float64 if dtype == "f64" else torch.float32
    es = [O.random_lqr_expansion(rng, T, nx, nu) for _ in range(4)]
    # batch: the four oracle problems repeated, SoA batch-minor
    def field(name, comps):
        a = np.stack([getattr(es[b % 4], name).reshape(T, comps) for b in range(B)], -1)
        return torch.as_tensor(a.transpose(1, 0, 2).copy(), dtype=dt).cuda()
    ins = [field("P", nx * nx), field("R", nu * nu), field("M", nx * nu), field("d", nu),
           field("Fx", nx * nx), field("Fu", nx * nu)]
    PT = torch.as_tensor(np.stack([es[b % 4].PT.reshape(-1) for b in range(B)], -1)[:, None, :],
                         dtype=dt).cuda()
    alpha = torch.full((B,), 0.5, dtype=torch.float64, device="cuda")
    out = {}
    monkeypatch.setenv("PTC_BULK", "1")
    for plan, (c0, c1) in {"sweep": (T, 0), "tree": (4, 8)}.items():
        s = LqrSolver(B, T, nx, nu, dtype=dt, chunk0=c0, chunk=c1, with_value=True)
        s.solve(*ins, PT, alpha)
        torch.cuda.synchronize()
        assert int(s.flags.abs().sum()) == 0
        out[plan] = [t.double().cpu().numpy() for t in (s.Gamma, s.gamma, s.dx, s.du, s.S, s.s)]
    tol = 1e-9 if dtype == "f64" else 1e-4
    for a, b in zip(out["sweep"], out["tree"]):
        assert rel_gap(a, b) < tol
    for k in range(4):
        ref = O.lqr_solve(es[k].with_alpha(0.5))   # S, s, Gamma, gamma, dx, du
        got = out["sweep"]
        for want, have in zip(ref, (got[4][..., k], got[5][..., k], got[0][..., k],
                                     got[1][..., k], got[2][..., k], got[3][..., k])):
            w = np.asarray(want).reshape(T + 1 if have.shape[1] == T + 1 else T, -1)
            assert rel_gap(have.T.reshape(w.shape), w) < tol


@pytest.mark.parametrize("nx,nu", [(1, 1), (2, 1), (3, 2), (4, 1), (4, 2)])
def test_one_cta_solve_matches_oracle(nx, nu):
    """Small batches with the automatic plan take the one-CTA-per-problem
    solve (k_lqr_cta: both trees in shared memory, 32 <= T <= 1024, batch
    <= 16) or, for 1024 < T <= 16384, the same on a thread-block cluster
    (tree levels across CTAs through DSMEM); every output against the
    oracle, fp64 1e-9 and fp32 1e-4, for horizons that are and are not
    powers of two, and a flagged problem (indefinite R) reported for that
    problem only."""
    import torch
    from paper_2409_20027_b200 import passes
    cases = [(1, 32), (5, 100), (16, 257), (3, 1024), (2, 2500), (1, 4096)]
    if nx <= 2:
        cases.append((1, 16384))
    for B, T in cases:
        rng = np.random.default_rng([nx, nu, B, T])
        exps = [O.random_lqr_expansion(rng, T, nx, nu, alpha=0.2) for _ in range(B)]
        if B > 1:
            exps[1].R[T // 3] = -10.0 * np.eye(nu)   # indefinite R + alpha I at one stage
        refs = [O.lqr_solve(e) if (B == 1 or b != 1) else None for b, e in enumerate(exps)]
        for dtype, tol in ((torch.float64, 1e-9), (torch.float32, 1e-4)):
            sol = passes.LqrSolver(B, T, nx, nu, dtype=dtype, with_value=True)
            dev = sol.device
            stack = lambda f, c, rows=T: torch.as_tensor(np.stack(
                [f(e).reshape(rows, c) for e in exps], -1)).permute(1, 0, 2).contiguous().to(dev, dtype)
            args = [stack(lambda e: e.P, nx * nx), stack(lambda e: e.R, nu * nu),
                    stack(lambda e: e.M, nx * nu), stack(lambda e: e.d, nu),
                    stack(lambda e: e.Fx, nx * nx), stack(lambda e: e.Fu, nx * nu),
                    stack(lambda e: e.PT, nx * nx, 1)]
            alpha = torch.tensor([e.alpha for e in exps], dtype=torch.float64, device=dev)
            sol.solve(*args, alpha)
            torch.cuda.synchronize()
            flags = sol.flags.cpu().numpy()
            host = lambda t, rows, shape: t.permute(2, 1, 0).double().cpu().numpy().reshape(
                (B, rows) + shape)
            outs = (host(sol.S, T + 1, (nx, nx)), host(sol.s, T + 1, (nx,)),
                    host(sol.Gamma, T, (nu, nx)), host(sol.gamma, T, (nu,)),
                    host(sol.dx, T + 1, (nx,)), host(sol.du, T, (nu,)))
            for b in range(B):
                if refs[b] is None:
                    assert flags[b] != 0, (B, T, b)
                    continue
                assert flags[b] == 0, (B, T, b, flags[b])
                for k in range(6):
                    assert rel_gap(outs[k][b], refs[b][k]) < tol, (B, T, b, k, dtype)
