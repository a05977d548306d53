"""Restart-parity fixtures: the REAL reference run one Newton iteration (or
one outer step) at a time, with every state it passes through recorded.

Chaotic runs (config 0's 100-iteration rounds, config 2's 200 ADMM steps,
config 3's random swing-ups) cannot be compared end to end: the reference
itself moves by up to 6e-3 when its inputs move by one ulp.  What can be
compared is each step from the reference's OWN entering state: the device
restarted from the state the reference recorded must produce the
reference's next state.  This script records those states.

The replay drives pintoc's public functions only: ``newton_solve`` is called
with ``max_iters=1`` and the loop state (trajectory, alpha, nu) handed from
call to call -- exactly the state ``newton.py:157-208`` carries between
iterations (a rejected step reuses the expansion via ``with_alpha``, which
recomputes ``R + alpha I`` from the same P, R: the same bits as a fresh
expansion).  The outer loops are ``outer.py:221-245`` / ``outer.py:392-435``
restated with pintoc's own ``BarrierAugmentation``, ``AdmmAugmentation``,
``project_box`` and ``_stack_w``.  Every replay is checked against the
reference's own uninterrupted run (bitwise) before it is saved.

    python tests/golden/make_restart.py [--only NAME] [--workers 7]

Outputs ``restart_cfg0.npz``, ``restart_cfg2.npz``, ``restart_cfg4.npz``,
``cfg3_sample.npz`` next to this file.  Record layout (per iteration i):
  it_in[i], it_out[i]   trajectory ids before / after the iteration
  it_alpha, it_nu       the loop state entering it
  it_aug                barrier: mu; ADMM: outer-step index (z, v derived)
  it_hist[i]            the reference's IterationRecord (cost, alpha,
                        gain_ratio, step_norm, accepted)
  it_term[i]            0 continue, 1 converged_cost, 2 converged_step,
                        4 stalled, -1 SolverStalledError raised
  it_alpha_next, it_nu_next   loop state after it
Trajectories: traj_x (K, T+1, nx), traj_u (K, T, nu).
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))

import pintoc  # noqa: E402  (the reference, read-only)
from pintoc import (  # noqa: E402
    AdmmOptions, BarrierOptions, BoxConstraint, CartPoleDynamics, CartPoleParams,
    ControlProblem, NewtonOptions, PendulumDynamics, PendulumParams, QuadraticCost,
    admm_solve, barrier_solve, newton_solve, rollout, total_cost,
)
from pintoc.exceptions import InfeasibleError
from pintoc.exceptions import SolverStalledError  # noqa: E402
from pintoc.newton import TERM_COST, TERM_STALLED, TERM_STEP, regularization_update  # noqa: E402
from pintoc.outer import (  # noqa: E402
    AdmmAugmentation, BarrierAugmentation, _stack_w, assert_strictly_feasible, project_box,
)

TERM_CODE = {"max_iters": 0, TERM_COST: 1, TERM_STEP: 2, TERM_STALLED: 4}


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)", flush=True)


class Recorder:
    """Trajectory table + per-iteration records."""

    def __init__(self, keep_trajs=True):
        self.trajs = []
        self.ids = {}
        self.rows = []
        self.keep = keep_trajs

    def tid(self, traj):
        if not self.keep:
            return -1
        k = id(traj)
        if k not in self.ids:
            self.ids[k] = len(self.trajs)
            self.trajs.append(traj)   # keeps the object alive, so ids stay unique
        return self.ids[k]

    def arrays(self, prefix=""):
        out = {}
        if self.trajs:
            out[prefix + "traj_x"] = np.stack([t.states for t in self.trajs])
            out[prefix + "traj_u"] = np.stack([t.controls for t in self.trajs])
        cols = ("in", "out", "alpha", "nu", "aug", "term", "alpha_next", "nu_next", "cur")
        for j, c in enumerate(cols):
            v = np.array([r[j if j < 8 else 10] for r in self.rows], dtype=float)
            out[prefix + "it_" + c] = v.astype(np.int64) if c in ("in", "out", "term") else v
        out[prefix + "it_hist"] = np.array([r[9] for r in self.rows], float).reshape(-1, 5)
        return out


def newton_chain(dyn, cost, aug, traj, opts, rec=None, aug_tag=0.0):
    """pintoc.newton_solve replayed one iteration at a time.  Returns
    (traj, iterations, termination, final_cost, history, stalled_error)."""
    alpha, nu = opts.alpha0, opts.nu0
    hist = []
    term = "max_iters"
    cur_cost = None
    while len(hist) < opts.max_iters:
        tin = rec.tid(traj) if rec is not None else -1
        one = NewtonOptions(alpha0=alpha, nu0=nu, inner_tol=opts.inner_tol, max_iters=1,
                            executor=opts.executor)
        # the cost newton_solve computes on entry (newton.py:152), recorded so
        # the gain ratio's rounding band can be stated for every step
        try:
            entering = total_cost(cost, aug, traj) if rec is not None else math.nan
        except InfeasibleError:
            entering = math.nan
        try:
            traj2, rep = newton_solve(dyn, cost, aug, traj, one)
        except SolverStalledError:
            if rec is not None:
                rec.rows.append((tin, tin, alpha, nu, aug_tag, -1, math.nan, math.nan,
                                 None, (math.nan,) * 5, entering))
            return traj, len(hist), "error", cur_cost, hist, True
        r = rep.history[0]
        hist.append(r)
        cur_cost = rep.final_cost
        t1 = rep.termination
        if r.gain_ratio == -math.inf and math.isnan(r.step_norm):
            a2, n2 = (alpha * nu if alpha > 0 else 1e-6), 2.0 * nu     # newton.py:172-175
        elif t1 == TERM_STEP:
            a2, n2 = alpha, nu
        else:
            a2, n2, acc = regularization_update(alpha, nu, r.gain_ratio)
            assert acc == r.accepted
        if rec is not None:
            rec.rows.append((tin, rec.tid(traj2), alpha, nu, aug_tag, TERM_CODE[t1], a2, n2, None,
                             (r.cost, r.alpha, r.gain_ratio, r.step_norm, float(r.accepted)),
                             entering))
        traj, alpha, nu = traj2, a2, n2
        if t1 != "max_iters":
            term = t1
            break
    return traj, len(hist), term, cur_cost, hist, False


def nudged(dyn, traj, sign):
    """The trajectory with x_0 and every control moved by one ulp, re-rolled
    through the reference's dynamics."""
    d = np.inf if sign > 0 else -np.inf
    return rollout(dyn, np.nextafter(traj.states[0], d), np.nextafter(traj.controls, d))


def step_floor(dyn, cost, aug, traj, opts, count, out):
    """The reference's own reproducibility of one Newton solve: rerun it from
    the entering trajectory moved by one ulp either way.  Returns (floor,
    stable): how far the solution moves (relative, max of states and
    controls) and whether the iteration count stays `count`."""
    floor, stable = 0.0, True
    for sign in (1, -1):
        try:
            t2, n2, _, _, _, err = newton_chain(dyn, cost, aug, nudged(dyn, traj, sign), opts)
        except Exception:               # e.g. a nudge leaves the barrier domain
            return math.inf, False
        if err:
            return math.inf, False
        stable = stable and n2 == count
        for a, b in ((t2.states, out.states), (t2.controls, out.controls)):
            floor = max(floor, float(np.abs(a - b).max() / max(1.0, np.abs(b).max())))
    return floor, stable


def barrier_chain(problem, initial, opts, rec=None, rounds_out=None):
    """outer.py:221-245 over newton_chain.  rounds_out collects per round
    (mu, entering traj, iterations, termination, cost).  Returns
    (traj, status) with status 'done' or 'stalled' (SolverStalledError)."""
    assert_strictly_feasible(problem.constraints, initial)
    traj = initial
    mu = opts.mu0
    while mu > opts.mu_tol:
        aug = BarrierAugmentation(problem.constraints, mu)
        t_in = traj
        traj, n, term, c, _, err = newton_chain(problem.dynamics, problem.cost, aug, traj,
                                                opts.newton, rec, mu)
        if rounds_out is not None:
            rounds_out.append((mu, t_in, n, term, c, traj))
        if err:
            return traj, "stalled"
        mu *= opts.zeta
    return traj, "done"


# ---------------------------------------------------------------------------

def pend_cfg0(T=100):
    dyn = PendulumDynamics(T, PendulumParams(damping=0.1, dt=0.05))
    cost = QuadraticCost(np.diag([10.0, 0.1]), np.diag([0.01]), np.diag([100.0, 10.0]),
                         x_goal=np.zeros(2))
    box = BoxConstraint(2, 1, control_lower=-5.0, control_upper=5.0)
    return ControlProblem(dyn, cost, box)


def cartpole_cfg2(T=500, state_box=True):
    dyn = CartPoleDynamics(T, CartPoleParams(cart_mass=1.0, pole_mass=0.1,
                                             pole_length=0.5, dt=0.02))
    Q = np.diag([1.0, 10.0, 0.1, 0.1])
    cost = QuadraticCost(Q, np.diag([0.01]), 10 * Q, x_goal=np.array([0.0, math.pi, 0.0, 0.0]))
    if state_box:
        box = BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0,
                            state_lower=[-1.5, -np.inf, -np.inf, -np.inf],
                            state_upper=[1.5, np.inf, np.inf, np.inf])
    else:
        box = BoxConstraint(4, 1, control_lower=-10.0, control_upper=10.0)
    return ControlProblem(dyn, cost, box)


def case_cfg0():
    """BASELINE config 0 (the make_golden barrier_pendulum_cfg0 run): all 600
    Newton iterations of the 6 barrier rounds as restart records."""
    T = 100
    prob = pend_cfg0(T)
    rng = np.random.default_rng(0)
    u0 = np.clip(rng.standard_normal((T, 1)), -4.5, 4.5)
    x0 = np.array([math.pi, 0.0])
    init = rollout(prob.dynamics, x0, u0)
    opts = BarrierOptions(mu0=0.1, zeta=0.1, mu_tol=5e-7, newton=NewtonOptions(max_iters=100))
    rec = Recorder()
    rounds = []
    traj, status = barrier_chain(prob, init, opts, rec, rounds)
    ref, rep = barrier_solve(prob, init, opts)
    assert status == "done"
    assert np.array_equal(traj.controls, ref.controls) and np.array_equal(traj.states, ref.states)
    assert [r[2] for r in rounds] == [r.newton.iterations for r in rep.rounds]
    save("restart_cfg0", x0=x0, u0=u0, round_mu=np.array([r[0] for r in rounds]),
         round_iters=np.array([r[2] for r in rounds]), final_u=traj.controls,
         final_x=traj.states, **rec.arrays())


def case_cfg2(workers=7, sample_steps=(0, 1, 2, 100, 199)):
    """BASELINE config 2 (T=500 cart-pole ADMM, rho=1, 200 outer steps): the
    trajectory entering every outer step (z, v are re-derived from them by
    the exact elementwise update, checked against the checkpoints stored
    here), each step's Newton count / termination / final cost, and full
    per-iteration records for the outer steps in `sample_steps`."""
    T = 500
    prob = cartpole_cfg2(T)
    con = prob.constraints
    rng = np.random.default_rng(0)
    u0 = 0.1 * rng.standard_normal((T, 1))
    x0 = np.zeros(4)
    init = rollout(prob.dynamics, x0, u0)
    opts = AdmmOptions(rho=1.0, max_outer=200)
    steps = Recorder()          # one trajectory per outer step
    its = Recorder()            # per-iteration restarts of the sampled steps
    traj = init
    z = project_box(_stack_w(con, traj), con)
    v = np.zeros_like(z)
    step_iters, step_term, step_cost, resid = [], [], [], []
    ckpt = {}
    converged = False
    t0 = time.perf_counter()
    zv = []
    for k in range(opts.max_outer):
        steps.tid(traj)
        zv.append((z, v))
        if k in (0, 1, 50, 100, 199):
            ckpt[f"z_{k}"], ckpt[f"v_{k}"] = z.copy(), v.copy()
        aug = AdmmAugmentation(con, opts.rho, z, v)
        rec = its if k in sample_steps else None
        traj, n, term, c, _, err = newton_chain(prob.dynamics, prob.cost, aug, traj,
                                                opts.newton, rec, float(k))
        assert not err
        step_iters.append(n)
        step_term.append(TERM_CODE[term])
        step_cost.append(c)
        w_val = _stack_w(con, traj)
        z_prev = z
        z = project_box(w_val + v / opts.rho, con)
        v = v + opts.rho * (w_val - z)
        r_p = float(np.max(np.abs(w_val - z)))
        r_d = float(np.max(np.abs(z - z_prev)))
        resid.append((r_p, r_d))
        if k % 10 == 0:
            print(f"  cfg2 step {k}: {n} iterations ({time.perf_counter() - t0:.0f}s)", flush=True)
        if r_p <= opts.residual_tol and r_d <= opts.residual_tol:
            converged = True
            break
    steps.tid(traj)
    # the replay IS the reference run: compare with its recorded end state
    g = np.load(os.path.join(OUT, "admm_cartpole_cfg2.npz"))
    assert list(g["sol_newton_iters"]) == step_iters, "replay differs from the reference run"
    assert np.array_equal(g["sol_us"], traj.controls)
    assert np.array_equal(g["sol_z"], z) and np.array_equal(g["sol_v"], v)
    # the reference's reproducibility of every outer step's Newton solve
    import multiprocessing as mp
    global _CFG2_JOBS
    _CFG2_JOBS = (prob, opts, steps.trajs, zv, step_iters)
    t1 = time.perf_counter()
    with mp.get_context("fork").Pool(workers) as pool:
        fl = pool.map(_cfg2_floor, range(len(step_iters)), chunksize=1)
    print(f"  cfg2 floors: {time.perf_counter() - t1:.0f}s", flush=True)
    save("restart_cfg2", x0=x0, u0=u0, step_iters=np.array(step_iters),
         step_floor=np.array([f[0] for f in fl]), step_stable=np.array([f[1] for f in fl]),
         step_term=np.array(step_term), step_cost=np.array(step_cost),
         residuals=np.array(resid), converged=np.array(converged),
         sample_steps=np.array(sample_steps), z_final=z, v_final=v,
         **ckpt, **steps.arrays("step_"), **its.arrays())


_CFG2_JOBS = None


def _cfg2_floor(k):
    prob, opts, trajs, zv, iters = _CFG2_JOBS
    aug = AdmmAugmentation(prob.constraints, opts.rho, zv[k][0], zv[k][1])
    return step_floor(prob.dynamics, prob.cost, aug, trajs[k], opts.newton, iters[k],
                      trajs[k + 1])


def cfg4_instance(T=256, nx=12, nu=4, seed=20029):
    """Config 4's model at a reduced horizon (numpy generator): A_k = I + dt
    F_k, dt = 0.01, F_k ~ N(0, 0.2) on the 3x3-block upper bidiagonal
    pattern, B_k ~ N(0, 0.1), Q = diag(U(0.1, 10)), R = 0.1 I, Qf = 10 Q,
    |u| <= 2."""
    rng = np.random.default_rng(seed)
    band = np.zeros((nx, nx))
    for i in range(4):
        for j in (i, i + 1):
            if j < 4:
                band[3 * i:3 * i + 3, 3 * j:3 * j + 3] = 1.0
    F = rng.normal(size=(T, nx, nx)) * math.sqrt(0.2) * band
    A = np.eye(nx)[None] + 0.01 * F
    B = rng.normal(size=(T, nx, nu)) * math.sqrt(0.1)
    qd = rng.uniform(0.1, 10.0, size=nx)
    x0 = rng.normal(size=nx)
    return A, B, qd, x0


def case_cfg4():
    """Config 4 reduced to T = 256 (nx 12, nu 4, barrier mu 0.1 -> 1e-4):
    whole solve and per-iteration records."""
    sys.path.insert(0, OUT)
    from make_golden import TVLinear
    T, nx, nu = 256, 12, 4
    A, B, qd, x0 = cfg4_instance(T, nx, nu)
    dyn = TVLinear(A, B, np.zeros((T, nx)))
    cost = QuadraticCost(np.diag(qd), 0.1 * np.eye(nu), 10 * np.diag(qd), x_goal=np.zeros(nx))
    box = BoxConstraint(nx, nu, control_lower=-2.0, control_upper=2.0)
    prob = ControlProblem(dyn, cost, box)
    init = rollout(dyn, x0, np.zeros((T, nu)))
    opts = BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-4, newton=NewtonOptions(max_iters=50))
    rec = Recorder()
    rounds = []
    traj, status = barrier_chain(prob, init, opts, rec, rounds)
    ref, rep = barrier_solve(prob, init, opts)
    assert status == "done"
    assert np.array_equal(traj.controls, ref.controls)
    save("restart_cfg4", A=A, B=B, qd=qd, x0=x0,
         round_mu=np.array([r.mu for r in rep.rounds]),
         round_iters=np.array([r.newton.iterations for r in rep.rounds]),
         round_term=np.array([TERM_CODE[r.newton.termination] for r in rep.rounds]),
         round_cost=np.array([r.cost for r in rep.rounds]),
         final_x=traj.states, final_u=traj.controls, **rec.arrays())


# --------------------------------------------------------------- config 3

CFG3_T = 256
CFG3_N = {"pendulum": 48, "cartpole": 16}
CFG3_FULL = 32768          # the bench's per-half batch at N = 1: the sample is its head


def cfg3_problem(system):
    if system == "pendulum":
        p = pend_cfg0(CFG3_T)
        return p
    return cartpole_cfg2(CFG3_T, state_box=False)


def cfg3_starts(system):
    """First problems of bench.py mpc_leg's rank-0 batch (same generator)."""
    rng = np.random.default_rng([2409, 20027, 0, 0 if system == "pendulum" else 1])
    n = CFG3_FULL
    if system == "pendulum":
        x0 = np.stack([rng.uniform(-np.pi, np.pi, n), 0.5 * rng.standard_normal(n)], 1)
    else:
        x0 = np.stack([rng.uniform(-1, 1, n), rng.uniform(-np.pi, np.pi, n),
                       0.5 * rng.standard_normal(n), 0.5 * rng.standard_normal(n)], 1)
    bound = 5.0 if system == "pendulum" else 10.0
    u0 = np.clip(0.1 * bound * rng.standard_normal((n, CFG3_T, 1)), -0.9 * bound, 0.9 * bound)
    k = CFG3_N[system]
    return x0[:k], u0[:k]


CFG3_OPTS = BarrierOptions(mu0=0.1, zeta=0.2, mu_tol=1e-6, newton=NewtonOptions(max_iters=50))
CFG3_SHIFT = 10


def _cfg3_one(job):
    system, i, x0, u0 = job
    prob = cfg3_problem(system)
    dyn = prob.dynamics
    out = {}
    for leg in ("cold", "warm"):
        init = rollout(dyn, x0, u0)
        rounds = []
        tail = Recorder()
        traj, status = barrier_chain(prob, init, CFG3_OPTS, None, rounds)
        if status == "stalled":
            # the failing round again, recorded, for per-iteration restarts of the stall
            mu, t_in = rounds[-1][0], rounds[-1][1]
            aug = BarrierAugmentation(prob.constraints, mu)
            t_end = newton_chain(dyn, prob.cost, aug, t_in, CFG3_OPTS.newton, tail, mu)[0]
            assert np.array_equal(t_end.controls, traj.controls)
            # keep the records on the last accepted trajectory (the stall
            # sequence: rejections with growing alpha, then the error)
            last = tail.rows[-1][0]
            tail.rows = [r for r in tail.rows if r[0] == last]
            tail.trajs = [tail.trajs[last]]
            tail.rows = [(0, 0) + tuple(r[2:]) for r in tail.rows]
            try:
                barrier_solve(prob, init, CFG3_OPTS)
                raise AssertionError(f"reference did not stall on {system} {i} {leg}")
            except SolverStalledError:
                pass
        else:
            # the reference's own uninterrupted run must agree bitwise
            ref, rep = barrier_solve(prob, init, CFG3_OPTS)
            assert np.array_equal(ref.controls, traj.controls), (system, i, leg)
            assert [r.newton.iterations for r in rep.rounds] == [r[2] for r in rounds]
        floors = []
        for q, (mu, t_in, n, term, c, t_out) in enumerate(rounds):
            if status == "stalled" and q == len(rounds) - 1:
                floors.append((math.nan, False))
                continue
            aug = BarrierAugmentation(prob.constraints, mu)
            floors.append(step_floor(dyn, prob.cost, aug, t_in, CFG3_OPTS.newton, n, t_out))
        out[leg] = dict(status=status, rounds=rounds, traj=traj, tail=tail, floors=floors)
        # receding-horizon step: start at x_10, controls shifted by 10 with the
        # last repeated (bench.py mpc_leg / BatchSolver.shift_controls)
        x0 = traj.states[CFG3_SHIFT].copy()
        u0 = np.concatenate([traj.controls[CFG3_SHIFT:],
                             np.repeat(traj.controls[-1:], CFG3_SHIFT, 0)], 0)
    return system, i, out


def case_cfg3(workers=7):
    import multiprocessing as mp
    jobs = []
    for system in ("pendulum", "cartpole"):
        x0, u0 = cfg3_starts(system)
        jobs += [(system, i, x0[i], u0[i]) for i in range(len(x0))]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(workers) as pool:
        res = pool.map(_cfg3_one, jobs, chunksize=1)
    print(f"  cfg3 reference runs: {time.perf_counter() - t0:.0f}s", flush=True)
    out = {}
    mu, R = CFG3_OPTS.mu0, 0
    while mu > CFG3_OPTS.mu_tol:
        R, mu = R + 1, mu * CFG3_OPTS.zeta
    for system in ("pendulum", "cartpole"):
        x0, u0 = cfg3_starts(system)
        rs = [r for r in res if r[0] == system]
        out[f"{system}_x0"], out[f"{system}_u0"] = x0, u0
        for leg in ("cold", "warm"):
            p = f"{system}_{leg}_"
            n = len(rs)
            status = np.array([1 if r[2][leg]["status"] == "done" else -1 for r in rs])
            iters = np.zeros((n, R), np.int64)
            terms = np.zeros((n, R), np.int64)
            costs = np.full((n, R), np.nan)
            nrounds = np.zeros(n, np.int64)
            floor = np.full((n, R), np.nan)
            stable = np.zeros((n, R), bool)
            tin_x = np.zeros((n, R) + rs[0][2][leg]["traj"].states.shape)
            tin_u = np.zeros((n, R) + rs[0][2][leg]["traj"].controls.shape)
            fin_x = np.stack([r[2][leg]["traj"].states for r in rs])
            fin_u = np.stack([r[2][leg]["traj"].controls for r in rs])
            for j, r in enumerate(rs):
                rounds = r[2][leg]["rounds"]
                nrounds[j] = len(rounds)
                for q, (mu, t_in, k, term, c, _) in enumerate(rounds):
                    iters[j, q] = k
                    terms[j, q] = TERM_CODE.get(term, -1)
                    costs[j, q] = np.nan if c is None else c
                    tin_x[j, q], tin_u[j, q] = t_in.states, t_in.controls
                    floor[j, q], stable[j, q] = r[2][leg]["floors"][q]
            out.update({p + "status": status, p + "iters": iters, p + "terms": terms,
                        p + "costs": costs, p + "nrounds": nrounds, p + "round_in_x": tin_x,
                        p + "round_in_u": tin_u, p + "final_x": fin_x, p + "final_u": fin_u,
                        p + "floor": floor, p + "stable": stable})
            # stall tails: one table over the problems of this leg
            tails = Recorder()
            owner = []
            for j, r in enumerate(rs):
                tl = r[2][leg]["tail"]
                if not tl.rows:
                    continue
                base = len(tails.trajs)
                tails.trajs.extend(tl.trajs)
                for row in tl.rows:
                    tails.rows.append((row[0] + base, row[1] + base) + tuple(row[2:]))
                    owner.append(j)
            if tails.rows:
                out.update(tails.arrays(p + "tail_"))
                out[p + "tail_owner"] = np.array(owner)
    mus, mu = [], CFG3_OPTS.mu0
    while mu > CFG3_OPTS.mu_tol:
        mus.append(mu)
        mu *= CFG3_OPTS.zeta
    out["mu_schedule"] = np.array(mus)
    save("cfg3_sample", shift=np.array(CFG3_SHIFT), **out)


CASES = {"cfg0": case_cfg0, "cfg4": case_cfg4, "cfg3": case_cfg3, "cfg2": case_cfg2}

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--workers", type=int, default=7)
    args = ap.parse_args()
    sys.path.insert(0, OUT)
    for name, fn in CASES.items():
        if args.only and args.only != name:
            continue
        t0 = time.perf_counter()
        fn(args.workers) if name in ("cfg2", "cfg3") else fn()
        print(f"  {name}: {time.perf_counter() - t0:.1f}s", flush=True)
