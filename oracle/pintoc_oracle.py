"""Plain-numpy restatement of the reference path -- TEST INFRASTRUCTURE ONLY.

This is the CPU oracle the CUDA product is checked against (tests, smoke)
and the CPU arm timed by ``bench.py`` (``cpu_baseline`` / ``--impl
reference``).  It restates, in its own structure, the algorithm of the
reference package ``pintoc`` (arxiv 2409.20027 artifact):

* models .............. reference ``systems.py`` (pendulum 161-231,
                        cart-pole 260-437, linear 32-77, quadratic cost
                        80-139) and ``problem.py:233-340`` (box constraints)
* augmentations ....... ``outer.py:30-157`` (log barrier), ``outer.py:252-333``
                        (ADMM consensus penalty)
* rollout / cost ...... ``problem.py:449-486``
* co-state pass ....... ``passes.py:108-148``  (Alg. 1, suffix scan)
* expansion ........... ``passes.py:155-185``
* value pass .......... ``passes.py:192-323``  (Alg. 2, dual elements,
                        combine rule, gains)
* propagation pass .... ``passes.py:330-361``  (Alg. 3)
* Newton loop ......... ``newton.py:93-215``   (Alg. 4 + LM trust region)
* outer loops ......... ``outer.py:221-245`` (barrier), ``outer.py:392-435``
                        (ADMM)

Scans run in the reference's *sequential executor* order (``scan.py:95-112``)
so that oracle numerics track the reference to rounding.  Parity of this file
with the real reference is pinned by ``tests/test_oracle_golden.py`` against
fixtures generated from the reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

ALPHA_MAX = 1e12


# ---------------------------------------------------------------------------
# errors (mirror reference exceptions.py)
# ---------------------------------------------------------------------------

class OracleError(Exception):
    pass


class Divergence(OracleError):
    def __init__(self, step):
        self.step = step
        super().__init__(f"non-finite state at rollout step {step}")

    def __reduce__(self):  # picklable across the CPU baseline's worker pool
        return (type(self), (self.step,))


class Infeasible(OracleError):
    def __init__(self, stage, component, value):
        self.stage, self.component, self.value = stage, component, value
        super().__init__(f"stage {stage} component {component} value {value}")

    def __reduce__(self):
        return (type(self), (self.stage, self.component, self.value))


class Definiteness(OracleError):
    def __init__(self, stage, what):
        self.stage, self.what = stage, what
        super().__init__(f"{what} not positive definite at stage {stage}")

    def __reduce__(self):
        return (type(self), (self.stage, self.what))


class Conditioning(OracleError):
    pass


class Stalled(OracleError):
    pass


def _sym(a):
    return 0.5 * (a + np.swapaxes(a, -1, -2))


# ---------------------------------------------------------------------------
# second-order jets in three variables (used for the cart-pole accelerations)
# ---------------------------------------------------------------------------

class _Jet:
    """value / gradient / Hessian of a scalar function of (theta, omega, F),
    vectorised over a leading stage axis."""

    __slots__ = ("v", "g", "h")

    def __init__(self, v, g, h):
        self.v, self.g, self.h = v, g, h

    @staticmethod
    def const(c, n):
        return _Jet(np.full(n, float(c)), np.zeros((n, 3)), np.zeros((n, 3, 3)))

    @staticmethod
    def var(vals, k):
        n = len(vals)
        g = np.zeros((n, 3))
        g[:, k] = 1.0
        return _Jet(np.asarray(vals, float), g, np.zeros((n, 3, 3)))

    def __add__(self, o):
        if not isinstance(o, _Jet):
            return _Jet(self.v + o, self.g, self.h)
        return _Jet(self.v + o.v, self.g + o.g, self.h + o.h)

    __radd__ = __add__

    def __neg__(self):
        return _Jet(-self.v, -self.g, -self.h)

    def __sub__(self, o):
        return self + (-o)

    def __mul__(self, o):
        if not isinstance(o, _Jet):
            return _Jet(self.v * o, self.g * o, self.h * o)
        outer = self.g[:, :, None] * o.g[:, None, :]
        return _Jet(self.v * o.v,
                    self.g * o.v[:, None] + o.g * self.v[:, None],
                    self.h * o.v[:, None, None] + o.h * self.v[:, None, None]
                    + outer + np.swapaxes(outer, 1, 2))

    __rmul__ = __mul__

    def recip(self):
        r = 1.0 / self.v
        r2 = r * r
        gg = self.g[:, :, None] * self.g[:, None, :]
        return _Jet(r, -self.g * r2[:, None],
                    -self.h * r2[:, None, None] + 2.0 * gg * (r2 * r)[:, None, None])

    def __truediv__(self, o):
        if not isinstance(o, _Jet):
            return self * (1.0 / o)
        return self * o.recip()

    def sin(self):
        s, c = np.sin(self.v), np.cos(self.v)
        gg = self.g[:, :, None] * self.g[:, None, :]
        return _Jet(s, self.g * c[:, None], self.h * c[:, None, None] - gg * s[:, None, None])

    def cos(self):
        s, c = np.sin(self.v), np.cos(self.v)
        gg = self.g[:, :, None] * self.g[:, None, :]
        return _Jet(c, -self.g * s[:, None], -self.h * s[:, None, None] - gg * c[:, None, None])


# ---------------------------------------------------------------------------
# dynamics models.  derivs(xs, us) returns fx, fu, fxx, fuu, fxu stacked over
# stages with the output-component-first Hessian layout of the reference.
# ---------------------------------------------------------------------------

@dataclass
class Pendulum:
    """Damped torque pendulum, state (theta, omega), upright at the origin
    (reference systems.py:146-231)."""
    gravity: float = 9.81
    length: float = 1.0
    mass: float = 1.0
    damping: float = 1e-3
    dt: float = 0.01
    nx: int = 2
    nu: int = 1

    def step(self, t, x, u):
        th, om = float(x[0]), float(x[1])
        acc = (-(self.gravity / self.length) * math.sin(th)
               + (float(np.reshape(u, -1)[0]) - self.damping * om)
               / (self.mass * self.length ** 2))
        return np.array([th + self.dt * om, om + self.dt * acc])

    def derivs(self, xs, us):
        n = len(us)
        inertia = self.mass * self.length ** 2
        fx = np.zeros((n, 2, 2))
        fx[:, 0, 0] = 1.0
        fx[:, 0, 1] = self.dt
        fx[:, 1, 0] = -self.dt * (self.gravity / self.length) * np.cos(xs[:n, 0])
        fx[:, 1, 1] = 1.0 - self.dt * self.damping / inertia
        fu = np.zeros((n, 2, 1))
        fu[:, 1, 0] = self.dt / inertia
        fxx = np.zeros((n, 2, 2, 2))
        fxx[:, 1, 0, 0] = self.dt * (self.gravity / self.length) * np.sin(xs[:n, 0])
        return fx, fu, fxx, np.zeros((n, 2, 1, 1)), np.zeros((n, 2, 2, 1))


@dataclass
class CartPole:
    """Force-driven cart-pole, state (pos, theta, vel, omega), theta = 0 pole
    down (reference systems.py:244-437)."""
    gravity: float = 9.81
    pole_length: float = 0.5
    cart_mass: float = 10.0
    pole_mass: float = 1.0
    dt: float = 0.01
    nx: int = 4
    nu: int = 1

    def _accels(self, th, om, force):
        n = len(th)
        TH, OM, FF = _Jet.var(th, 0), _Jet.var(om, 1), _Jet.var(force, 2)
        s, c = TH.sin(), TH.cos()
        mp, mc, ln, g = self.pole_mass, self.cart_mass, self.pole_length, self.gravity
        den = s * s * mp + mc
        cart = (FF + s * mp * (OM * ln + c * g)) / den
        pole = (-(FF * c) - OM * OM * c * s * (mp * ln) - s * ((mc + mp) * g)) / (den * ln)
        return cart, pole

    def step(self, t, x, u):
        f = float(np.reshape(u, -1)[0])
        cart, pole = self._accels(np.array([float(x[1])]), np.array([float(x[3])]),
                                  np.array([f]))
        dt = self.dt
        return np.array([x[0] + dt * x[2], x[1] + dt * x[3],
                         x[2] + dt * cart.v[0], x[3] + dt * pole.v[0]])

    def derivs(self, xs, us):
        n = len(us)
        dt = self.dt
        cart, pole = self._accels(xs[:n, 1], xs[:n, 3], us[:, 0])
        fx = np.zeros((n, 4, 4))
        fx[:, 0, 0] = fx[:, 1, 1] = fx[:, 2, 2] = 1.0
        fx[:, 0, 2] = fx[:, 1, 3] = dt
        fu = np.zeros((n, 4, 1))
        fxx = np.zeros((n, 4, 4, 4))
        fxu = np.zeros((n, 4, 4, 1))
        for row, acc in ((2, cart), (3, pole)):
            fx[:, row, 1] = dt * acc.g[:, 0]
            fx[:, row, 3] = dt * acc.g[:, 1]
            fu[:, row, 0] = dt * acc.g[:, 2]
            fxx[:, row, 1, 1] = dt * acc.h[:, 0, 0]
            fxx[:, row, 1, 3] = fxx[:, row, 3, 1] = dt * acc.h[:, 0, 1]
            fxx[:, row, 3, 3] = dt * acc.h[:, 1, 1]
            fxu[:, row, 1, 0] = dt * acc.h[:, 0, 2]
            fxu[:, row, 3, 0] = dt * acc.h[:, 1, 2]
        fx[:, 3, 3] += 1.0
        return fx, fu, fxx, np.zeros((n, 4, 1, 1)), fxu


class Linear:
    """Affine dynamics x' = A_t x + B_t u + c_t; A, B, c either shared over
    stages (reference systems.py:32-77) or stacked per stage (a user
    DynamicsModel with time-varying matrices)."""

    def __init__(self, A, B, c=None):
        self.A = np.asarray(A, float)
        self.B = np.asarray(B, float)
        self.nx = self.A.shape[-1]
        self.nu = self.B.shape[-1]
        self.c = np.zeros(self.A.shape[:-1]) if c is None else np.asarray(c, float)
        self.tv = self.A.ndim == 3

    def mats(self, t):
        A = self.A[t] if self.A.ndim == 3 else self.A
        B = self.B[t] if self.B.ndim == 3 else self.B
        c = self.c[t] if self.c.ndim == 2 else self.c
        return A, B, c

    def step(self, t, x, u):
        A, B, c = self.mats(t)
        return A @ x + B @ u + c

    def derivs(self, xs, us):
        n = len(us)
        fx = self.A[:n] if self.A.ndim == 3 else np.broadcast_to(self.A, (n,) + self.A.shape)
        fu = self.B[:n] if self.B.ndim == 3 else np.broadcast_to(self.B, (n,) + self.B.shape)
        nx, nu = self.nx, self.nu
        return (fx, fu, np.zeros((n, nx, nx, nx)), np.zeros((n, nx, nu, nu)),
                np.zeros((n, nx, nx, nu)))


# ---------------------------------------------------------------------------
# cost and constraints
# ---------------------------------------------------------------------------

class Quadratic:
    """0.5 (x-g)^T Q (x-g) + 0.5 u^T R u, terminal 0.5 (x-g)^T Qf (x-g)
    (reference systems.py:80-139)."""

    def __init__(self, Q, R, Qf, goal=None):
        self.Q = np.atleast_2d(np.asarray(Q, float))
        self.R = np.atleast_2d(np.asarray(R, float))
        self.Qf = np.atleast_2d(np.asarray(Qf, float))
        self.goal = np.zeros(self.Q.shape[0]) if goal is None else np.asarray(goal, float)

    def stage(self, xs, us):
        e = xs - self.goal
        return 0.5 * (np.einsum("ti,ij,tj->t", e, self.Q, e)
                      + np.einsum("ti,ij,tj->t", us, self.R, us))

    def terminal(self, x):
        e = x - self.goal
        return 0.5 * float(e @ self.Qf @ e)

    def terminal_grad(self, x):
        return self.Qf @ (x - self.goal)


class Box:
    """Componentwise bounds stacked as one-sided rows w = [g(x); h(u)] <= 0
    (reference problem.py:233-340).  Each row is (var, index, sign, bound)
    with w = sign * (var[index] - bound)."""

    def __init__(self, nx, nu, control_lower=None, control_upper=None,
                 state_lower=None, state_upper=None):
        def full(v, n, d):
            return np.full(n, d) if v is None else np.broadcast_to(np.asarray(v, float), (n,)).copy()
        self.nx, self.nu = nx, nu
        self.cl = full(control_lower, nu, -np.inf)
        self.cu = full(control_upper, nu, np.inf)
        self.sl = full(state_lower, nx, -np.inf)
        self.su = full(state_upper, nx, np.inf)
        rows = []
        rows += [("x", i, 1.0, self.su[i]) for i in range(nx) if np.isfinite(self.su[i])]
        rows += [("x", i, -1.0, self.sl[i]) for i in range(nx) if np.isfinite(self.sl[i])]
        self.n_state = len(rows)
        rows += [("u", i, 1.0, self.cu[i]) for i in range(nu) if np.isfinite(self.cu[i])]
        rows += [("u", i, -1.0, self.cl[i]) for i in range(nu) if np.isfinite(self.cl[i])]
        self.rows = rows
        self.n_total = len(rows)
        self.jx = np.zeros((self.n_state, nx))
        self.ju = np.zeros((self.n_total - self.n_state, nu))
        for k, (var, i, s, _) in enumerate(rows):
            if var == "x":
                self.jx[k, i] = s
            else:
                self.ju[k - self.n_state, i] = s

    def w(self, xs, us):
        """Stacked constraint values, shape (N, n_total)."""
        n = len(us)
        out = np.empty((n, self.n_total))
        for k, (var, i, s, b) in enumerate(self.rows):
            src = xs[:n, i] if var == "x" else us[:, i]
            out[:, k] = (src - b) if s > 0 else (b - src)
        return out


# augmentations: tuples ("zero",) | ("barrier", box, mu) | ("admm", box, rho, z, v)

def _aug_terms(aug, xs, us):
    """Per-stage c, cx, cu, cxx, cuu of the augmentation (cxu is zero for
    box constraints)."""
    n, nx, nu = len(us), xs.shape[1], us.shape[1]
    kind = aug[0]
    if kind == "zero":
        return (np.zeros(n), np.zeros((n, nx)), np.zeros((n, nu)),
                np.zeros((n, nx, nx)), np.zeros((n, nu, nu)))
    box = aug[1]
    w = box.w(xs, us)
    ns = box.n_state
    if kind == "barrier":
        mu = aug[2]
        if w.size and w.max() >= 0:
            st, comp = np.nonzero(w >= 0)
            raise Infeasible(int(st[0]), int(comp[0]), float(w[st[0], comp[0]]))
        c = np.zeros(n)
        if ns:
            c = c + np.sum(np.log(-w[:, :ns]), axis=1)
        if box.n_total - ns:
            c = c + np.sum(np.log(-w[:, ns:]), axis=1)
        c = -mu * c
        inv = 1.0 / w
        cx = -mu * (inv[:, :ns] @ box.jx) if ns else np.zeros((n, nx))
        cu = -mu * (inv[:, ns:] @ box.ju) if box.n_total - ns else np.zeros((n, nu))
        sx = box.jx[None] * inv[:, :ns, None]
        su = box.ju[None] * inv[:, ns:, None]
        cxx = mu * np.einsum("tmi,tmj->tij", sx, sx)
        cuu = mu * np.einsum("tmi,tmj->tij", su, su)
        return c, cx, cu, cxx, cuu
    rho, z, v = aug[2], aug[3], aug[4]
    res = w - z + v / rho
    c = 0.5 * rho * np.sum(res * res, axis=1)
    cx = rho * (res[:, :ns] @ box.jx) if ns else np.zeros((n, nx))
    cu = rho * (res[:, ns:] @ box.ju)
    cxx = np.broadcast_to(rho * box.jx.T @ box.jx, (n, nx, nx))
    cuu = np.broadcast_to(rho * box.ju.T @ box.ju, (n, nu, nu))
    return c, cx, cu, cxx, cuu


# ---------------------------------------------------------------------------
# rollout and cost
# ---------------------------------------------------------------------------

def rollout(dyn, x0, us):
    """States x_{0..N} from x0 under controls us (reference problem.py:449)."""
    n = len(us)
    xs = np.empty((n + 1, dyn.nx))
    xs[0] = x0
    for t in range(n):
        nxt = np.asarray(dyn.step(t, xs[t], us[t]), float)
        if not np.all(np.isfinite(nxt)):
            raise Divergence(t + 1)
        xs[t + 1] = nxt
    return xs


def total_cost(cost, aug, xs, us):
    """terminal + sum of stage costs + sum of augmentation (problem.py:476)."""
    c_aug = _aug_terms(aug, xs, us)[0]
    return float(cost.terminal(xs[-1])
                 + (float(np.sum(cost.stage(xs[:-1], us))) + float(np.sum(c_aug))))


# ---------------------------------------------------------------------------
# Alg. 1: co-states as a suffix scan over (dl, dc, df) elements
# ---------------------------------------------------------------------------

def costate_pass(dyn, cost, aug, xs, us):
    n = len(us)
    lam_end = cost.terminal_grad(xs[n])
    xq = xs[:n]
    dl = (xq - cost.goal) @ cost.Q.T
    dc = _aug_terms(aug, xs, us)[1]
    fx = dyn.derivs(xs, us)[0]
    out = np.empty((n + 1, dyn.nx))
    out[n] = lam_end
    # last element absorbs the boundary (zero Jacobian), then fold leftwards
    acc_l = dl[n - 1] + fx[n - 1].T @ lam_end
    acc_c = dc[n - 1].copy()
    out[n - 1] = acc_l + acc_c
    for t in range(n - 2, -1, -1):
        acc_l = dl[t] + fx[t].T @ acc_l
        acc_c = dc[t] + fx[t].T @ acc_c
        out[t] = acc_l + acc_c
    return out


# ---------------------------------------------------------------------------
# quadratic expansion of the augmented Hamiltonian
# ---------------------------------------------------------------------------

@dataclass
class Expansion:
    P: np.ndarray
    R: np.ndarray
    M: np.ndarray
    d: np.ndarray
    Fx: np.ndarray
    Fu: np.ndarray
    PT: np.ndarray
    alpha: float = 0.0

    @property
    def Rr(self):
        return self.R + self.alpha * np.eye(self.R.shape[1])

    def with_alpha(self, alpha):
        return replace(self, alpha=float(alpha))


def expansion(dyn, cost, aug, xs, us, lam, alpha=0.0):
    n = len(us)
    nx, nu = dyn.nx, dyn.nu
    fx, fu, fxx, fuu, fxu = dyn.derivs(xs, us)
    _, _, cu, cxx, cuu = _aug_terms(aug, xs, us)
    nxt = lam[1:]
    P = np.broadcast_to(cost.Q, (n, nx, nx)) + cxx + np.einsum("tk,tkij->tij", nxt, fxx)
    R = np.broadcast_to(cost.R, (n, nu, nu)) + cuu + np.einsum("tk,tkij->tij", nxt, fuu)
    M = np.einsum("tk,tkij->tij", nxt, fxu)
    d = us @ cost.R.T + cu + np.einsum("tkj,tk->tj", fu, nxt)
    return Expansion(P=_sym(P), R=_sym(R), M=np.array(M), d=d, Fx=np.array(fx),
                     Fu=np.array(fu), PT=_sym(cost.Qf.copy()), alpha=float(alpha))


# ---------------------------------------------------------------------------
# Alg. 2: value-function pass over dual elements (A, Y, C, eta, b)
# ---------------------------------------------------------------------------

def _chol_ok(mats):
    try:
        np.linalg.cholesky(mats)
        return -1
    except np.linalg.LinAlgError:
        for t in range(len(mats)):
            try:
                np.linalg.cholesky(mats[t])
            except np.linalg.LinAlgError:
                return t
        return 0


def value_elements(exp):
    """Stage elements (from expansion) plus the terminal element, as arrays
    with N+1 rows (reference passes.py:192-261)."""
    n, nx = exp.P.shape[0], exp.P.shape[1]
    Rr = exp.Rr
    bad = _chol_ok(Rr)
    if bad >= 0:
        raise Definiteness(bad, "R + alpha*I")
    RiM = np.linalg.solve(Rr, np.swapaxes(exp.M, 1, 2))
    RiF = np.linalg.solve(Rr, np.swapaxes(exp.Fu, 1, 2))
    Rid = np.linalg.solve(Rr, exp.d[..., None])[..., 0]
    A = np.zeros((n + 1, nx, nx))
    Y = np.zeros((n + 1, nx, nx))
    C = np.zeros((n + 1, nx, nx))
    eta = np.zeros((n + 1, nx))
    b = np.zeros((n + 1, nx))
    A[:n] = exp.Fx - exp.Fu @ RiM
    Y[:n] = _sym(exp.P - exp.M @ RiM)
    C[:n] = _sym(exp.Fu @ RiF)
    eta[:n] = np.einsum("tij,tj->ti", exp.M, Rid)
    b[:n] = -np.einsum("tij,tj->ti", exp.Fu, Rid)
    Y[n] = exp.PT
    return A, Y, C, eta, b


def value_combine(left, right):
    """(A, Y, C, eta, b) of left (earlier) joined with right (later)
    (reference passes.py:264-288)."""
    Al, Yl, Cl, el, bl = left
    Ar, Yr, Cr, er, br = right
    nx = Al.shape[0]
    G = np.eye(nx) + Cl @ Yr
    try:
        X = np.linalg.solve(G, np.concatenate([Al, Cl, (bl + Cl @ er)[:, None]], axis=1))
        Z = np.linalg.solve(G.T, np.concatenate([Yr @ Al, (er - Yr @ bl)[:, None]], axis=1))
    except np.linalg.LinAlgError as err:
        raise Conditioning(str(err)) from err
    return (Ar @ X[:, :nx],
            _sym(Al.T @ Z[:, :nx] + Yl),
            _sym(Ar @ X[:, nx:2 * nx] @ Ar.T + Cr),
            Al.T @ Z[:, nx] + el,
            Ar @ X[:, 2 * nx] + br)


def value_pass(exp):
    """S_{0..N}, s_{0..N} and gains (Gamma, gamma) (passes.py:291-323)."""
    A, Y, C, eta, b = value_elements(exp)
    n, nx = exp.P.shape[0], exp.P.shape[1]
    S = np.empty((n + 1, nx, nx))
    s = np.empty((n + 1, nx))
    acc = (A[n], Y[n], C[n], eta[n], b[n])
    S[n], s[n] = acc[1], -acc[3]
    for t in range(n - 1, -1, -1):
        acc = value_combine((A[t], Y[t], C[t], eta[t], b[t]), acc)
        S[t], s[t] = acc[1], -acc[3]
    FuT = np.swapaxes(exp.Fu, 1, 2)
    FuTS = FuT @ S[1:]
    Q = _sym(exp.Rr + FuTS @ exp.Fu)
    bad = _chol_ok(Q)
    if bad >= 0:
        raise Definiteness(bad, "Q")
    Gamma = -np.linalg.solve(Q, np.swapaxes(exp.M, 1, 2) + FuTS @ exp.Fx)
    gamma = -np.linalg.solve(Q, (exp.d + np.einsum("tkj,tk->tj", exp.Fu, s[1:]))[..., None])[..., 0]
    return S, s, Gamma, gamma


# ---------------------------------------------------------------------------
# Alg. 3: propagation of the closed loop from dx_0 = 0
# ---------------------------------------------------------------------------

def propagation_pass(Gamma, gamma, exp):
    n, nx = exp.P.shape[0], exp.P.shape[1]
    F = exp.Fx + exp.Fu @ Gamma
    e = np.einsum("tij,tj->ti", exp.Fu, gamma)
    dxs = np.zeros((n + 1, nx))
    # prefix scan of affine maps; the head element has F = 0
    acc_e = e[0].copy()
    dxs[1] = acc_e
    for t in range(1, n):
        acc_e = F[t] @ acc_e + e[t]
        dxs[t + 1] = acc_e
    dus = np.einsum("tij,tj->ti", Gamma, dxs[:-1]) + gamma
    return dxs, dus


def lqr_solve(exp):
    """value pass + propagation pass: the LQR-scan solve of one subproblem."""
    S, s, Gamma, gamma = value_pass(exp)
    dxs, dus = propagation_pass(Gamma, gamma, exp)
    return S, s, Gamma, gamma, dxs, dus


# ---------------------------------------------------------------------------
# Alg. 4: regularised Newton loop (newton.py)
# ---------------------------------------------------------------------------

def gain_ratio(actual, predicted):
    if predicted <= 0:
        return -math.inf
    return actual / predicted


def regularization_update(alpha, nu, ratio):
    if ratio > 0:
        return alpha * max(1.0 / 3.0, 1.0 - (2.0 * ratio - 1.0) ** 3), 2.0, True
    return alpha * nu, 2.0 * nu, False


def predicted_reduction(dus, d, alpha):
    return 0.5 * float(alpha * np.sum(dus * dus) - np.sum(dus * d))


@dataclass
class NewtonResult:
    xs: np.ndarray
    us: np.ndarray
    iterations: int
    final_cost: float
    termination: str
    history: list  # (cost, alpha, gain_ratio, step_norm, accepted)

    @property
    def converged(self):
        return self.termination in ("converged_cost", "converged_step")


def check_consistent(dyn, xs, us):
    for t in range(len(us)):
        pred = np.asarray(dyn.step(t, xs[t], us[t]), float)
        gap = np.max(np.abs(pred - xs[t + 1]))
        if gap > 1e-8 * (1.0 + np.max(np.abs(pred))):
            raise ValueError(f"initial trajectory is not dynamically consistent at step {t}")


def newton_solve(dyn, cost, aug, xs, us, alpha0=1.0, nu0=2.0, inner_tol=1e-8,
                 max_iters=100, check=True):
    aug = ("zero",) if aug is None else aug
    if check:
        check_consistent(dyn, xs, us)
    cur = total_cost(cost, aug, xs, us)
    alpha, nu = alpha0, nu0
    exp = None
    hist = []
    term = "max_iters"
    while len(hist) < max_iters:
        if exp is None:
            lam = costate_pass(dyn, cost, aug, xs, us)
            exp = expansion(dyn, cost, aug, xs, us, lam, alpha)
        elif exp.alpha != alpha:
            exp = exp.with_alpha(alpha)
        try:
            _, _, Gamma, gamma = value_pass(exp)
            _, dus = propagation_pass(Gamma, gamma, exp)
        except (Definiteness, Conditioning) as err:
            if alpha > ALPHA_MAX:
                raise Stalled(str(err)) from err
            hist.append((cur, alpha, -math.inf, math.nan, False))
            alpha = alpha * nu if alpha > 0 else 1e-6
            nu = 2.0 * nu
            continue
        step = float(np.max(np.abs(dus)))
        if step <= inner_tol:
            hist.append((cur, alpha, math.nan, step, False))
            term = "converged_step"
            break
        pred = predicted_reduction(dus, exp.d, alpha)
        used = alpha
        new = math.inf
        cand = None
        try:
            cand_us = us + dus
            cand = rollout(dyn, xs[0], cand_us)
            new = total_cost(cost, aug, cand, cand_us)
            ratio = gain_ratio(cur - new, pred)
        except (Infeasible, Divergence):
            ratio = -math.inf
        alpha, nu, ok = regularization_update(alpha, nu, ratio)
        if ok:
            rel = abs(cur - new) / max(1.0, abs(cur))
            hist.append((new, used, ratio, step, True))
            xs, us, cur = cand, cand_us, new
            exp = None
            if rel <= inner_tol:
                term = "converged_cost"
                break
        else:
            hist.append((cur, used, ratio, step, False))
            if alpha > ALPHA_MAX:
                term = "stalled"
                break
    return NewtonResult(xs, us, len(hist), cur, term, hist)


# ---------------------------------------------------------------------------
# outer loops (outer.py)
# ---------------------------------------------------------------------------

def assert_strictly_feasible(box, xs, us):
    w = box.w(xs, us)
    if w.size and w.max() >= 0:
        st, comp = np.nonzero(w >= 0)
        raise Infeasible(int(st[0]), int(comp[0]), float(w[st[0], comp[0]]))


@dataclass
class BarrierResult:
    xs: np.ndarray
    us: np.ndarray
    mus: list
    costs: list
    controls: list
    newton: list

    @property
    def outer_iterations(self):
        return len(self.mus)

    @property
    def inner_iterations(self):
        return sum(r.iterations for r in self.newton)

    @property
    def converged(self):
        return all(r.converged for r in self.newton)


def barrier_solve(dyn, cost, box, xs, us, mu0=0.1, zeta=0.2, mu_tol=1e-4, **newton):
    assert_strictly_feasible(box, xs, us)
    mu = mu0
    res = BarrierResult(xs, us, [], [], [], [])
    while mu > mu_tol:
        r = newton_solve(dyn, cost, ("barrier", box, mu), xs, us, **newton)
        xs, us = r.xs, r.us
        res.mus.append(mu)
        res.costs.append(r.final_cost)
        res.controls.append(us.copy())
        res.newton.append(r)
        mu *= zeta
    res.xs, res.us = xs, us
    return res


def project_box(p):
    return np.minimum(np.asarray(p, float), 0.0)


@dataclass
class AdmmResult:
    xs: np.ndarray
    us: np.ndarray
    z: np.ndarray
    v: np.ndarray
    residuals: list
    newton: list
    converged: bool

    @property
    def outer_iterations(self):
        return len(self.residuals)

    @property
    def inner_iterations(self):
        return sum(r.iterations for r in self.newton)


def admm_solve(dyn, cost, box, xs, us, rho=1.0, residual_tol=1e-2, max_outer=200, **newton):
    z = project_box(box.w(xs, us))
    v = np.zeros_like(z)
    residuals, reports = [], []
    converged = False
    for _ in range(max_outer):
        r = newton_solve(dyn, cost, ("admm", box, rho, z, v), xs, us, **newton)
        reports.append(r)
        xs, us = r.xs, r.us
        w = box.w(xs, us)
        z_prev = z
        z = project_box(w + v / rho)
        v = v + rho * (w - z)
        rp = float(np.max(np.abs(w - z))) if z.size else 0.0
        rd = float(np.max(np.abs(z - z_prev))) if z.size else 0.0
        residuals.append((rp, rd))
        if rp <= residual_tol and rd <= residual_tol:
            converged = True
            break
    return AdmmResult(xs, us, z, v, residuals, reports, converged)


# ---------------------------------------------------------------------------
# seeded synthetic workloads (BASELINE.json configs)
# ---------------------------------------------------------------------------

def random_lqr_expansion(rng, T, nx, nu, alpha=0.0):
    """Config 1: time-varying random LQR subproblem.  A_k = I + 0.05 N(0,1)
    with spectral radius clipped to <= 1.05, B_k ~ N(0, 0.1), Q_k = M M^T +
    0.1 I, R_k = 0.1 I, affine terms c_k ~ N(0, 0.01) (entering the control
    gradient d through B_k^T c_k)."""
    A = np.eye(nx)[None] + 0.05 * rng.standard_normal((T, nx, nx))
    rad = np.max(np.abs(np.linalg.eigvals(A)), axis=1)
    scale = np.where(rad > 1.05, 1.05 / rad, 1.0)
    A = A * scale[:, None, None]
    B = np.sqrt(0.1) * rng.standard_normal((T, nx, nu))
    Mq = rng.standard_normal((T, nx, nx))
    Q = Mq @ np.swapaxes(Mq, 1, 2) + 0.1 * np.eye(nx)
    R = np.broadcast_to(0.1 * np.eye(nu), (T, nu, nu)).copy()
    c = 0.1 * rng.standard_normal((T, nx))
    d = np.einsum("tij,ti->tj", B, c)
    Mm = np.zeros((T, nx, nu))
    Mq2 = rng.standard_normal((nx, nx))
    PT = Mq2 @ Mq2.T + 0.1 * np.eye(nx)
    return Expansion(P=Q, R=R, M=Mm, d=d, Fx=A, Fu=B, PT=PT, alpha=float(alpha))
