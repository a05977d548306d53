"""Host-side API checks (no GPU): options validation, LM rules, box row
stacking, scan-schedule span, expansion helpers."""

import math

import numpy as np
import pytest

import paper_2409_20027_b200 as P


def test_regularization_update_and_gain_ratio():
    a, n, ok = P.regularization_update(3.0, 2.0, 1.0)
    assert ok and math.isclose(a, 1.0) and n == 2.0
    a, n, ok = P.regularization_update(3.0, 2.0, 0.5)
    assert ok and math.isclose(a, 3.0)
    a, n, ok = P.regularization_update(3.0, 2.0, -0.2)
    assert not ok and math.isclose(a, 6.0) and n == 4.0
    assert P.gain_ratio(2.0, 2.0) == 1.0
    assert P.gain_ratio(1.0, 0.0) == -math.inf
    dus = np.array([[1.0], [2.0]])
    d = np.array([[0.5], [-1.0]])
    assert math.isclose(P.predicted_reduction(dus, d, 3.0), 0.5 * (15.0 + 1.5))


def test_options_validation():
    with pytest.raises(ValueError):
        P.NewtonOptions(alpha0=-1.0)
    with pytest.raises(ValueError):
        P.NewtonOptions(nu0=1.0)
    with pytest.raises(ValueError):
        P.NewtonOptions(executor="gpu")
    with pytest.raises(ValueError):
        P.BarrierOptions(zeta=1.5)
    with pytest.raises(ValueError):
        P.AdmmOptions(rho=0.0)
    assert P.BarrierOptions().rounds() == 5
    assert P.BarrierOptions(mu0=0.1, zeta=0.1, mu_tol=5e-7).rounds() == 6
    assert P.BarrierOptions(mu0=1e-5, mu_tol=1e-4).rounds() == 0


def test_box_rows_follow_reference_stacking():
    box = P.BoxConstraint(2, 2, control_lower=(-2.0, -3.0), control_upper=(2.0, np.inf),
                          state_upper=(1.5, np.inf), state_lower=(-1.5, -1.0))
    assert box.n_state == 3 and box.n_control == 3
    xs = np.array([[0.5, 0.2], [0.0, 0.0]])
    us = np.array([[1.0, -1.0]])
    w = box.w_batch(xs, us)
    # [x0 - 1.5, -1.5 - x0, -1 - x1, u0 - 2, -2 - u0, -3 - u1]
    assert np.allclose(w[0], [-1.0, -2.0, -1.2, -1.0, -3.0, -2.0])


def test_project_box_is_idempotent_clamp(rng):
    p = rng.normal(size=8)
    once = P.project_box(p)
    assert np.array_equal(P.project_box(once), once)
    assert np.allclose(P.project_box(np.array([-1.0, 2.0, 0.0])), [-1.0, 0.0, 0.0])


def test_scan_plan_reference_semantics():
    """Acceptance criterion 2: the parallel plan's critical
    path is at most 2*ceil(log2 n) for every n; levels write distinct
    destinations from earlier sources; replaying the plan with a
    non-commutative combine (string concatenation) gives every prefix."""
    for n in list(range(1, 300)) + [1000, 1024, 1 << 12]:
        depth = P.scan_depth_probe(n)
        assert depth <= (0 if n == 1 else 2 * math.ceil(math.log2(n))), (n, depth)
        buf = [str(i) + "," for i in range(n)]
        for level in P.scan_plan(n):
            dsts = [d for _, d in level]
            assert len(set(dsts)) == len(dsts)
            assert all(s < d for s, d in level)
            for s, d in level:
                buf[d] = buf[s] + buf[d]
        assert buf == ["".join(f"{j}," for j in range(i + 1)) for i in range(n)]
    assert P.scan_plan(1) == []
    with pytest.raises(P.EmptySequenceError):
        P.scan_plan(0)


def test_scan_user_combine_both_directions():
    words = [chr(97 + i) for i in range(40)]
    cat = lambda a, b: a + b
    for ex in ("sequential", "parallel"):
        fw = P.scan(words, cat, P.ScanDirection.FORWARD, executor=ex)
        rv = P.scan(words, cat, P.ScanDirection.REVERSE, executor=ex)
        assert fw == ["".join(words[:i + 1]) for i in range(40)]
        assert rv == ["".join(words[i:]) for i in range(40)]


def test_device_scan_tree_has_log_span():
    """The solver's own schedule (csrc/common.cuh make_plan): depth
    2 (K0 + K L) with L = log_K(n / K0) levels."""
    for n in list(range(1, 300)) + [1 << 12, 1 << 16, 1 << 20]:
        depth = P.device_scan_depth(n)
        bound = 0 if n == 1 else 4 + 16 * math.ceil(math.log(n, 8)) + 8
        if n > 64:
            assert depth <= bound, (n, depth)
    lv = P.device_scan_plan(1 << 16)
    assert lv[0] == 1 << 16 and lv[-1] <= 8


def test_stage_expansion_with_alpha():
    e = P.StageExpansion.build(np.zeros((3, 1, 1)), np.ones((3, 1, 1)), np.zeros((3, 1, 1)),
                               np.zeros((3, 1)), np.ones((3, 1, 1)), np.ones((3, 1, 1)),
                               np.zeros((1, 1)), alpha=10.0)
    assert np.allclose(e.R_reg, 11.0)
    assert np.allclose(e.with_alpha(0.0).R_reg, 1.0)


def test_pendulum_and_cartpole_steps():
    params = P.PendulumParams(dt=0.01)
    nxt = P.pendulum_step(np.array([np.pi / 2, 0.0]), np.zeros(1), params)
    assert np.isclose(nxt[1], -0.0981)
    cp = P.CartPoleParams(dt=0.03)
    assert np.allclose(P.cartpole_step(np.zeros(4), np.zeros(1), cp), 0.0)


def test_swingup_problem_shapes():
    prob = P.make_swingup_problem("cartpole", 1000, 0.01)
    assert prob.dynamics.d_x == 4 and prob.horizon == 1000
    assert prob.constraints.n_control == 2
