"""Pin the CPU oracle against fixtures produced by the real reference.

The fixtures (tests/golden/*.npz) come from tests/golden/make_golden.py,
which imports the reference package itself.  Passing here is what makes the
oracle a trustworthy checker for the CUDA path.
"""

import math

import numpy as np
import pytest
from conftest import golden, rel_gap

from oracle import pintoc_oracle as O


def _exp(g, p):
    return O.Expansion(P=g[p + "P"], R=g[p + "R"], M=g[p + "M"], d=g[p + "d"],
                       Fx=g[p + "Fx"], Fu=g[p + "Fu"], PT=g[p + "PT"],
                       alpha=float(g[p + "alpha"]))


def test_lqr_small_matches_reference():
    g = golden("lqr_small")
    for i in range(int(g["count"])):
        p = f"{i}_"
        S, s, Gam, gam, dxs, dus = O.lqr_solve(_exp(g, p))
        for name, val in dict(S=S, s=s, Gamma=Gam, gamma=gam, dxs=dxs, dus=dus).items():
            assert rel_gap(val, g[p + name]) < 1e-12, (i, name)


def test_lqr_config1_matches_reference():
    g = golden("lqr_config1")
    for nx in (2, 4, 8, 12):
        p = f"{nx}_"
        S, s, Gam, gam, dxs, dus = O.lqr_solve(_exp(g, p))
        for name, val in dict(S=S, s=s, Gamma=Gam, gamma=gam, dxs=dxs, dus=dus).items():
            assert rel_gap(val, g[p + name]) < 1e-11, (nx, name)


def _models(g):
    pend = O.Pendulum(damping=0.1, dt=0.05)
    pcost = O.Quadratic(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
    pbox = O.Box(2, 1, control_lower=-5.0, control_upper=5.0)
    cp = O.CartPole(cart_mass=1.0, pole_mass=0.1, pole_length=0.5, dt=0.02)
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    ccost = O.Quadratic(Q, np.diag([0.01]), 10 * Q, goal=np.array([0.0, math.pi, 0.0, 0.0]))
    cbox = O.Box(4, 1, control_lower=-10.0, control_upper=10.0,
                 state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                 state_upper=[1.5, np.inf, np.inf, np.inf])
    return {"pendulum": (pend, pcost, pbox), "cartpole": (cp, ccost, cbox)}


def test_passes_on_models_match_reference():
    g = golden("passes_models")
    for name, (dyn, cost, box) in _models(g).items():
        xs = O.rollout(dyn, g[f"{name}_x0"], g[f"{name}_us"])
        us = g[f"{name}_us"]
        assert rel_gap(xs, g[f"{name}_xs"]) < 1e-13, name
        augs = {"zero": ("zero",), "barrier": ("barrier", box, 0.1),
                "admm": ("admm", box, 0.7, g[f"{name}_z"], g[f"{name}_v"])}
        for an, aug in augs.items():
            key = f"{name}_{an}_"
            lam = O.costate_pass(dyn, cost, aug, xs, us)
            assert rel_gap(lam, g[key + "lam"]) < 1e-12, key
            e = O.expansion(dyn, cost, aug, xs, us, lam, 0.5)
            for f in ("P", "R", "M", "d", "Fx", "Fu", "PT"):
                assert rel_gap(getattr(e, f), g[key + f]) < 1e-12, (key, f)
            assert abs(O.total_cost(cost, aug, xs, us) - float(g[key + "cost"])) <= 1e-12 * max(
                1.0, abs(float(g[key + "cost"])))


def _check_hist(hist, ref, tol=1e-9):
    assert hist.shape == ref.shape
    # accepted flags and termination path identical, numbers to tolerance
    assert np.array_equal(hist[:, 4], ref[:, 4])
    for col in range(4):
        a, b = hist[:, col], ref[:, col]
        fin = np.isfinite(b)
        assert np.array_equal(np.isfinite(a), fin)
        assert np.array_equal(np.sign(a[~fin]), np.sign(b[~fin]), equal_nan=True)
        if fin.any():
            scale = np.maximum(1.0, np.abs(b[fin]))
            assert np.max(np.abs(a[fin] - b[fin]) / scale) < tol, col


def test_newton_lq_matches_reference():
    g = golden("newton_lq")
    for i in range(int(g["count"])):
        p = f"{i}_"
        dyn = O.Linear(g[p + "A"], g[p + "B"])
        cost = O.Quadratic(g[p + "Q"], g[p + "R"], g[p + "Qf"], g[p + "goal"])
        n, du = g[p + "us"].shape
        us0 = np.zeros((n, du))
        xs0 = O.rollout(dyn, g[p + "x0"], us0)
        r = O.newton_solve(dyn, cost, None, xs0, us0, alpha0=float(g[p + "alpha0"]))
        assert r.termination == str(g[p + "term"])
        _check_hist(np.array(r.history).reshape(-1, 5), g[p + "hist"])
        assert rel_gap(r.us, g[p + "us"]) < 1e-9
        assert rel_gap(r.xs, g[p + "xs"]) < 1e-9


def _check_barrier(res, g, tol=1e-9):
    assert np.allclose(res.mus, g["sol_mus"], rtol=1e-15)
    assert [r.iterations for r in res.newton] == list(g["sol_round_iters"])
    assert [r.termination for r in res.newton] == list(g["sol_round_term"])
    for k, r in enumerate(res.newton):
        _check_hist(np.array(r.history).reshape(-1, 5), g[f"sol_hist{k}"], tol)
    assert rel_gap(res.us, g["sol_us"]) < tol
    assert rel_gap(res.xs, g["sol_xs"]) < tol


def test_barrier_pendulum_config0_matches_reference():
    g = golden("barrier_pendulum_cfg0")
    dyn = O.Pendulum(damping=0.1, dt=0.05)
    cost = O.Quadratic(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]))
    box = O.Box(2, 1, control_lower=-5.0, control_upper=5.0)
    xs0 = O.rollout(dyn, g["x0"], g["u0"])
    res = O.barrier_solve(dyn, cost, box, xs0, g["u0"], mu0=0.1, zeta=0.1, mu_tol=5e-7,
                          max_iters=100)
    _check_barrier(res, g)


def test_barrier_tvlinear_matches_reference():
    g = golden("barrier_tvlinear")
    dyn = O.Linear(g["A"], g["B"], g["c"])
    nx, nu = dyn.nx, dyn.nu
    cost = O.Quadratic(g["Q"], 0.1 * np.eye(nu), g["Q"])
    box = O.Box(nx, nu, control_lower=-2.0, control_upper=2.0)
    xs0 = O.rollout(dyn, g["x0"], g["u0"])
    res = O.barrier_solve(dyn, cost, box, xs0, g["u0"])
    _check_barrier(res, g)


def _check_admm(res, g, p, tol=1e-9):
    assert res.converged == bool(g[p + "converged"])
    assert [r.iterations for r in res.newton] == list(g[p + "newton_iters"])
    assert rel_gap(np.array(res.residuals), g[p + "residuals"]) < 1e-7
    assert rel_gap(res.us, g[p + "us"]) < tol
    assert rel_gap(res.xs, g[p + "xs"]) < tol


def test_admm_small_matches_reference():
    g = golden("admm_small")
    dyn = O.Pendulum(dt=0.05)
    cost = O.Quadratic(np.diag([10.0, 1.0]), np.diag([0.1]), 10 * np.diag([10.0, 1.0]))
    box = O.Box(2, 1, control_lower=-5.0, control_upper=5.0)
    xs0 = O.rollout(dyn, g["pend_x0"], g["pend_u0"])
    res = O.admm_solve(dyn, cost, box, xs0, g["pend_u0"], rho=1.0, max_outer=150)
    _check_admm(res, g, "pend_")

    cp = O.CartPole(cart_mass=1.0, pole_mass=0.1, pole_length=0.5, dt=0.02)
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    ccost = O.Quadratic(Q, np.diag([0.01]), 10 * Q, goal=np.array([0.0, math.pi, 0.0, 0.0]))
    cbox = O.Box(4, 1, control_lower=-10.0, control_upper=10.0,
                 state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                 state_upper=[1.5, np.inf, np.inf, np.inf])
    xs0 = O.rollout(cp, g["cp_x0"], g["cp_u0"])
    res = O.admm_solve(cp, ccost, cbox, xs0, g["cp_u0"], rho=1.0, max_outer=40)
    _check_admm(res, g, "cp_")


def test_oracle_lm_rules():
    assert O.regularization_update(3.0, 2.0, 1.0) == (1.0, 2.0, True)
    a, n, ok = O.regularization_update(3.0, 2.0, -0.2)
    assert (a, n, ok) == (6.0, 4.0, False)
    assert O.gain_ratio(1.0, 0.0) == -math.inf
    assert math.isnan(O.gain_ratio(1.0, math.nan))
