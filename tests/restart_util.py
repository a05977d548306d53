"""Restart parity: run the device solver from states the REFERENCE recorded
(tests/golden/make_restart.py) and compare the step it takes with the step
the reference took from the same state.

One device batch holds every restart of a fixture: problem i is loaded with
the trajectory, the Levenberg-Marquardt state (alpha, nu) and the barrier
weight mu (or ADMM z, v) the reference carried into its step i
(``ptc_solver_write``), so a 600-iteration run is checked in one launch
sequence with no error accumulation between steps.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from paper_2409_20027_b200.newton import regularization_update

TERM_DEVICE = {0: 3, 1: 1, 2: 2, 4: 4}     # fixture code -> PTC_TERM_*
TOL = 1e-9


@dataclass
class Restart:
    status: np.ndarray      # (B,) device status
    iters: np.ndarray       # (B,)
    term: np.ndarray        # (B,) PTC_TERM_*
    hist: np.ndarray        # (cap, 5, B)
    states: np.ndarray      # (B, T+1, nx)
    controls: np.ndarray    # (B, T, nu)
    alpha: np.ndarray
    nu: np.ndarray
    cost: np.ndarray
    cand: np.ndarray        # the step's candidate cost (inf: infeasible / diverged)


def device_restart(prob, X, U, alpha, nu, *, mu=None, z=None, v=None, rho=1.0,
                   max_iters=1, executor="auto", dtype=None) -> Restart:
    from paper_2409_20027_b200 import _native as N
    from paper_2409_20027_b200._device import DeviceSolver, SolveSettings
    from paper_2409_20027_b200.newton import plan_chunks, rollout_mode
    B = len(alpha)
    aug = N.AUG_BARRIER if mu is not None else (N.AUG_ADMM if z is not None else N.AUG_ZERO)
    c0, c1 = plan_chunks(executor, prob.horizon)
    st = SolveSettings(method=N.METHOD_NEWTON, aug=aug,
                       aug_mu=float(mu[0]) if mu is not None else 0.0, max_iters=max_iters,
                       hist_cap=max_iters, round_cap=1, rho=rho, chunk0=c0, chunk=c1,
                       rollout=rollout_mode(executor))
    s = DeviceSolver(prob.dynamics, prob.cost, prob.constraints, B, st, dtype=dtype)
    s.load(X, U, z, v)
    s.write("alpha", alpha)
    s.write("nu", nu)
    if mu is not None:
        s.write("mu", mu)
    s.run()
    rd = lambda n: s.read(n).cpu().numpy()
    return Restart(status=rd("status"), iters=rd("iters"), term=s.rounds("round_term")[0].cpu().numpy(),
                   hist=s.history().cpu().numpy(), states=s.states().cpu().numpy(),
                   controls=s.controls().cpu().numpy(), alpha=rd("alpha"), nu=rd("nu"),
                   cost=rd("cur_cost"), cand=rd("cand_cost"))


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(1.0, float(np.abs(b).max()))) if a.size else 0.0


def ratio_noise(hist_ref, cur_cost):
    """Tolerance band of the gain ratio (cur - new) / pred, a difference
    quotient of two costs: with each cost held to the parity tolerance 1e-9
    relative (the candidate cost is a sum over a rollout of up to 500 stages
    that amplifies the step's rounding), the ratio is known to
    1e-9 (|cur| + |new|) / |pred| (plus 1e-9 relative)."""
    r = hist_ref[:, 2]
    new = hist_ref[:, 0]
    with np.errstate(all="ignore"):
        pred = np.where(np.isfinite(r) & (r != 0), (cur_cost - new) / r, np.inf)
        band = TOL * (np.abs(cur_cost) + np.abs(new)) / np.abs(pred) + TOL * np.abs(r)
    return np.where(np.isfinite(band), band, 0.0)


def check_iterations(res: Restart, g, prefix="", label="", cur=None):
    """Compare B single-iteration restarts with the reference's records.
    Returns a dict of counters (for the test log)."""
    term = g[prefix + "it_term"]
    hist = g[prefix + "it_hist"]
    tout = g[prefix + "it_out"]
    X, U = g[prefix + "traj_x"], g[prefix + "traj_u"]
    B = len(term)
    stalled = term == -1
    assert np.array_equal(res.status == -1, stalled), (
        label, "SolverStalledError rows differ", np.flatnonzero((res.status == -1) != stalled)[:10])
    ok = ~stalled
    dh = res.hist[0].T                      # (B, 5) the device's record of its one step
    band = ratio_noise(hist, cur) if cur is not None else band_full(g, prefix)
    # a rejected step's record holds the entering cost, not the candidate's:
    # there the band's scale |pred| = |cur - cand| / |ratio| comes from the
    # device's own candidate cost
    rej = ok & (hist[:, 4] < 0.5) & np.isfinite(hist[:, 2]) & (hist[:, 2] != 0)
    if rej.any():
        with np.errstate(all="ignore"):
            pred = np.abs(hist[rej, 0] - res.cand[rej]) / np.abs(hist[rej, 2])
            b2 = TOL * (np.abs(hist[rej, 0]) + np.abs(res.cand[rej])) / pred
        band[rej] = np.where(np.isfinite(b2), b2, band[rej]) + TOL * np.abs(hist[rej, 2])
    acc_ref = hist[:, 4] > 0.5
    acc_dev = dh[:, 4] > 0.5
    # a flip is allowed only where the reference's ratio is within its own
    # rounding band of zero (the decision is noise in the reference too)
    amb = ok & np.isfinite(hist[:, 2]) & (np.abs(hist[:, 2]) <= band)
    bad_acc = ok & (acc_dev != acc_ref) & ~amb
    assert not bad_acc.any(), (label, "accept/reject differs", np.flatnonzero(bad_acc)[:10],
                               hist[bad_acc][:3], dh[bad_acc][:3])
    same = ok & (acc_dev == acc_ref)
    want = np.array([TERM_DEVICE.get(int(t), -1) for t in term])
    assert np.array_equal(res.term[same], want[same]), (
        label, "termination differs", np.flatnonzero(res.term[same] != want[same])[:10])
    # step norm (NaN on a definiteness reject) and the recorded cost
    assert np.array_equal(np.isnan(dh[same, 3]), np.isnan(hist[same, 3])), label
    fin = same & np.isfinite(hist[:, 3])
    if fin.any():
        sn = np.abs(dh[fin, 3] - hist[fin, 3]) / np.maximum(1.0, np.abs(hist[fin, 3]))
        assert sn.max() < TOL, (label, "step norm", sn.max(), np.flatnonzero(fin)[sn.argmax()])
    cg = np.abs(dh[same, 0] - hist[same, 0]) / np.maximum(1.0, np.abs(hist[same, 0]))
    assert cg.max(initial=0.0) < TOL, (label, "cost", cg.max())
    # gain ratio: -inf / NaN markers identical, finite values within the band
    assert np.array_equal(np.isposinf(-dh[same, 2]), np.isposinf(-hist[same, 2])), label
    rf = same & np.isfinite(hist[:, 2])
    worst = 0.0
    if rf.any():
        lim = np.maximum(band[rf], TOL * np.maximum(1.0, np.abs(hist[rf, 2])))
        q = np.abs(dh[rf, 2] - hist[rf, 2]) / lim
        worst = float(q.max())
        assert worst <= 1.0, (label, "gain ratio", worst, np.flatnonzero(rf)[q.argmax()])
    # Levenberg-Marquardt state after the step: nu exactly; alpha by the
    # reference's rule applied to the device's ratio, and within the band
    assert np.array_equal(res.nu[same], g[prefix + "it_nu_next"][same]), (label, "nu")
    a_in, n_in = g[prefix + "it_alpha"], g[prefix + "it_nu"]
    rule = np.array([regularization_update(a, n, r)[0] if acc else res_a
                     for a, n, r, acc, res_a in zip(a_in[same], n_in[same], dh[same, 2],
                                                    acc_dev[same], res.alpha[same])])
    assert np.allclose(res.alpha[same], rule, rtol=1e-14, atol=0), (label, "alpha rule")
    an = g[prefix + "it_alpha_next"][same]
    ag = float((np.abs(res.alpha[same] - an) / np.abs(an)).max(initial=0.0))
    # trajectory after the step (unchanged on a reject)
    idx = np.flatnonzero(same)
    gx = max((rel(res.states[i], X[tout[i]]) for i in idx), default=0.0)
    gu = max((rel(res.controls[i], U[tout[i]]) for i in idx), default=0.0)
    assert gx < TOL and gu < TOL, (label, "trajectory", gx, gu)
    return {"rows": B, "stalled": int(stalled.sum()), "accepted": int(acc_ref.sum()),
            "ambiguous_flips": int((ok & (acc_dev != acc_ref)).sum()),
            "max_ratio_gap_in_bands": worst, "max_alpha_gap": ag, "traj_gap": max(gx, gu)}


def band_full(g, prefix=""):
    """ratio_noise with the cost entering every step reconstructed from the
    records: a row's entering cost is the previous row's recorded cost when
    both act on the same trajectory chain (rejected: cost unchanged;
    accepted: the new cost), else the row's own cost for a rejection."""
    hist = g[prefix + "it_hist"]
    if prefix + "it_cur" in g.files:          # the entering cost, recorded
        return ratio_noise(hist, g[prefix + "it_cur"])
    tin, tout, aug = g[prefix + "it_in"], g[prefix + "it_out"], g[prefix + "it_aug"]
    cur = np.where(hist[:, 4] > 0.5, np.nan, hist[:, 0])
    for i in range(1, len(hist)):
        if (np.isnan(cur[i]) and tout[i - 1] == tin[i] and aug[i - 1] == aug[i]
                and np.isfinite(hist[i - 1, 0])):
            cur[i] = hist[i - 1, 0]
    cur = np.where(np.isnan(cur), hist[:, 0], cur)
    return ratio_noise(hist, cur)


def admm_states(g, box_oracle):
    """z, v entering every outer step, re-derived from the recorded
    trajectories with the reference's elementwise update (outer.py:418-420);
    pinned bitwise to the reference's checkpoints by
    tests/test_restart_fixtures.py."""
    X, U = g["step_traj_x"], g["step_traj_u"]
    w0 = box_oracle.w(X[0][:-1], U[0])
    z = np.minimum(w0, 0.0)
    v = np.zeros_like(z)
    zs, vs = [z], [v]
    for k in range(len(g["step_iters"]) - 1):
        w = box_oracle.w(X[k + 1][:-1], U[k + 1])
        z_new = np.minimum(w + v / 1.0, 0.0)
        v = v + 1.0 * (w - z_new)
        z = z_new
        zs.append(z)
        vs.append(v)
    return np.stack(zs), np.stack(vs)


def cfg2_box_oracle():
    from oracle import pintoc_oracle as O
    return O.Box(4, 1, control_lower=-10.0, control_upper=10.0,
                 state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                 state_upper=[1.5, np.inf, np.inf, np.inf])


def mu_schedule(mu0, zeta, mu_tol):
    """The barrier weights of outer.py:237-244 (mu *= zeta while mu > tol)."""
    out, mu = [], mu0
    while mu > mu_tol:
        out.append(mu)
        mu *= zeta
    return out
