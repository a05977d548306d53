"""Element-level operations of the three scans on the device
(value_element_init, value_combine, costate_combine, rollout_combine,
costate_boundary; reference passes.py:30-119, 192-288, 330-335) against the
pinned oracle and the reference's definitions, including the reference's
acceptance criterion 10 (associativity suite, test_acceptance.py:235) and
the suffix fold that defines value_pass (S_t = Y, s_t = -eta of the
combined suffix).  fp64, 1e-10 relative unless stated.
"""

import numpy as np
import pytest
from conftest import rel_gap

from oracle import pintoc_oracle as O

pytestmark = pytest.mark.gpu


def _exp(seed, T=6, nx=3, nu=2, alpha=0.3):
    import paper_2409_20027_b200 as P
    e = O.random_lqr_expansion(np.random.default_rng(seed), T, nx, nu, alpha=alpha)
    return e, P.StageExpansion.build(e.P, e.R, e.M, e.d, e.Fx, e.Fu, e.PT, alpha)


def _elem(arrs, t):
    import paper_2409_20027_b200 as P
    return P.ValueElement(*[a[t] for a in arrs])


@pytest.mark.parametrize("nx,nu", [(2, 1), (3, 2), (4, 2), (8, 4), (12, 4)])
def test_value_element_init_matches_oracle(nx, nu):
    import paper_2409_20027_b200 as P
    e, exp = _exp(nx * 10 + nu, 5, nx, nu)
    ref = O.value_elements(e)
    for t in range(exp.horizon + 1):
        got = P.value_element_init(exp, t)
        for g, r in zip(got, (a[t] for a in ref)):
            assert rel_gap(g, r) < 1e-10, t


def test_value_element_init_raises_definiteness():
    import paper_2409_20027_b200 as P
    e, exp = _exp(3)
    bad = P.StageExpansion.build(e.P, -np.abs(e.R), e.M, e.d, e.Fx, e.Fu, e.PT, 0.0)
    with pytest.raises(P.DefinitenessError) as exc:
        P.value_element_init(bad, 2)
    assert exc.value.stage == 2
    with pytest.raises(IndexError):
        P.value_element_init(exp, exp.horizon + 1)


def test_value_combine_matches_oracle_single_and_batched():
    import paper_2409_20027_b200 as P
    e, _ = _exp(4, T=9)
    A = O.value_elements(e)
    pairs = [(t, t + 1) for t in range(8)]
    for i, j in pairs:
        got = P.value_combine(_elem(A, i), _elem(A, j))
        ref = O.value_combine([a[i] for a in A], [a[j] for a in A])
        for g, r in zip(got, ref):
            assert rel_gap(g, r) < 1e-10
    # a leading item axis: all pairs in one launch
    L = P.ValueElement(*[a[:8] for a in A])
    R = P.ValueElement(*[a[1:9] for a in A])
    got = P.value_combine(L, R)
    for k, (i, j) in enumerate(pairs):
        ref = O.value_combine([a[i] for a in A], [a[j] for a in A])
        for g, r in zip(got, ref):
            assert rel_gap(g[k], r) < 1e-10


def test_value_combine_singular_raises_conditioning():
    import paper_2409_20027_b200 as P
    nx = 2
    z, eye = np.zeros((nx, nx)), np.eye(nx)
    left = P.ValueElement(eye, z, eye, np.zeros(nx), np.zeros(nx))
    right = P.ValueElement(eye, -eye, z, np.zeros(nx), np.zeros(nx))   # I + C_l Y_r = 0
    with pytest.raises(P.ConditioningError):
        P.value_combine(left, right)


def test_suffix_fold_of_elements_is_the_value_function():
    """S_t = Y and s_t = -eta of elements t..N folded right to left
    (passes.py:291-323), against the oracle's value pass."""
    import paper_2409_20027_b200 as P
    e, exp = _exp(5, T=7)
    S, s = O.value_pass(e)[:2]
    acc = P.value_element_init(exp, exp.horizon)
    for t in range(exp.horizon - 1, -1, -1):
        acc = P.value_combine(P.value_element_init(exp, t), acc)
        assert rel_gap(acc.Y, S[t]) < 1e-10 and rel_gap(-acc.eta, s[t]) < 1e-10


def test_associativity_suite():
    """Reference acceptance criterion 10: every combine is associative
    (random elements, 1e-9 relative)."""
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(6)
    e, _ = _exp(6, T=3)
    v = O.value_elements(e)
    a, b, c = (_elem(v, t) for t in range(3))
    lhs = P.value_combine(P.value_combine(a, b), c)
    rhs = P.value_combine(a, P.value_combine(b, c))
    for x, y in zip(lhs, rhs):
        assert rel_gap(x, y) < 1e-9
    nx = 4
    r = [P.RolloutElement(rng.standard_normal((nx, nx)), rng.standard_normal(nx)) for _ in range(3)]
    lhs = P.rollout_combine(P.rollout_combine(r[0], r[1]), r[2])
    rhs = P.rollout_combine(r[0], P.rollout_combine(r[1], r[2]))
    for x, y in zip(lhs, rhs):
        assert rel_gap(x, y) < 1e-9
    c3 = [P.CostateElement(rng.standard_normal(nx), rng.standard_normal(nx),
                           rng.standard_normal((nx, nx))) for _ in range(3)]
    lhs = P.costate_combine(P.costate_combine(c3[0], c3[1]), c3[2])
    rhs = P.costate_combine(c3[0], P.costate_combine(c3[1], c3[2]))
    for x, y in zip(lhs, rhs):
        assert rel_gap(x, y) < 1e-9


def test_affine_combines_follow_the_reference_definitions():
    """rollout_combine: first then second (F2 F1, F2 e1 + e2); costate_combine:
    left earlier (dl_l + df_l^T dl_r, dc_l + df_l^T dc_r, df_r df_l)."""
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(7)
    nx = 3
    F1, F2 = rng.standard_normal((2, nx, nx))
    e1, e2 = rng.standard_normal((2, nx))
    got = P.rollout_combine(P.RolloutElement(F1, e1), P.RolloutElement(F2, e2))
    assert rel_gap(got.F, F2 @ F1) < 1e-12 and rel_gap(got.e, F2 @ e1 + e2) < 1e-12
    l = P.CostateElement(*rng.standard_normal((2, nx)), rng.standard_normal((nx, nx)))
    r = P.CostateElement(*rng.standard_normal((2, nx)), rng.standard_normal((nx, nx)))
    got = P.costate_combine(l, r)
    assert rel_gap(got.dl, l.dl + l.df.T @ r.dl) < 1e-12
    assert rel_gap(got.dc, l.dc + l.df.T @ r.dc) < 1e-12
    assert rel_gap(got.df, r.df @ l.df) < 1e-12


def test_costate_boundary_is_terminal_gradient():
    import paper_2409_20027_b200 as P
    rng = np.random.default_rng(8)
    Qf = rng.standard_normal((3, 3))
    Qf = Qf @ Qf.T
    goal = rng.standard_normal(3)
    cost = P.QuadraticCost(np.eye(3), np.eye(1), Qf, x_goal=goal)
    x = rng.standard_normal(3)
    assert rel_gap(P.costate_boundary(cost, x), Qf @ (x - goal)) < 1e-12


def test_device_scan_over_element_tuples():
    """scan() (scan.py:133-166) with the path's combines: a REVERSE scan of
    the value elements is the value function (S_t = Y, s_t = -eta), a
    FORWARD scan of rollout maps equals the sequential composition, also
    through a user combine."""
    import paper_2409_20027_b200 as P
    e, exp = _exp(9, T=11)
    elems = [P.value_element_init(exp, t) for t in range(exp.horizon + 1)]
    out = P.scan(elems, P.value_combine, P.ScanDirection.REVERSE, executor="parallel")
    S, s = O.value_pass(e)[:2]
    for t in range(exp.horizon):
        assert rel_gap(out[t].Y, S[t]) < 1e-10 and rel_gap(-out[t].eta, s[t]) < 1e-10
    rng = np.random.default_rng(10)
    maps = [P.RolloutElement(np.eye(3) + 0.1 * rng.standard_normal((3, 3)),
                             rng.standard_normal(3)) for _ in range(13)]
    out = P.scan(maps, P.rollout_combine)
    F, c = maps[0].F, maps[0].e
    for t in range(1, 13):
        F, c = maps[t].F @ F, maps[t].F @ c + maps[t].e
        assert rel_gap(out[t].F, F) < 1e-10 and rel_gap(out[t].e, c) < 1e-10
    # a user combine runs the same schedule pair by pair
    user = P.scan(maps, lambda a, b: P.RolloutElement(b.F @ a.F, b.F @ a.e + b.e),
                  executor="parallel", parallel_threshold=2)
    for t in range(13):
        assert rel_gap(user[t].F, out[t].F) < 1e-10 and rel_gap(user[t].e, out[t].e) < 1e-10
    with pytest.raises(P.EmptySequenceError):
        P.scan([], P.rollout_combine)
