// Device-side models: dynamics (pendulum, cart-pole, affine), quadratic cost,
// box constraints and the two outer-loop augmentations.  Each stage
// evaluation is fused: one call produces everything the expansion needs,
// with dynamics Hessians contracted against lambda_{t+1} on the fly (no
// d_x^3 tensors ever reach HBM).
//
// Reference: systems.py (pendulum 161-231, cart-pole 260-437, linear 32-77,
// quadratic cost 80-139), problem.py:233-340 (BoxConstraint),
// outer.py:30-157 (barrier), outer.py:252-333 (ADMM penalty),
// passes.py:155-185 (expansion).
#pragma once

#include <type_traits>

#include "elements.cuh"

namespace ptc {

enum : int { DYN_PENDULUM = 0, DYN_CARTPOLE = 1, DYN_LINEAR = 2 };

constexpr int kMaxNX = 12;
constexpr int kMaxNU = 6;
constexpr int kMaxRows = 2 * (kMaxNX + kMaxNU);

// Problem description shared by every problem of a batch (lives in HBM,
// read through the read-only path; all threads read the same words).
struct ProblemParams {
  int dyn_kind;
  double dyn[8];            // pendulum: g, l, m, b, dt ; cart-pole: g, l, mc, mp, dt
  int lin_T, lin_B;         // affine model: A/B/c vary over stages if lin_T > 1,
                            // over problems if lin_B > 1
  const void* lin_A;        // (nx*nx, lin_T, lin_B) in the solver dtype
  const void* lin_Bm;       // (nx*nu, lin_T, lin_B)
  const void* lin_c;        // (nx,    lin_T, lin_B)
  const void* lin_st;       // stage-major copy [t][A | Bm | c] (lin_T rows) for
                            // time-varying models shared by the batch, nx >= 8
                            // (warp kernels: one contiguous row per stage), or null
  double Q[kMaxNX * kMaxNX], Rc[kMaxNU * kMaxNU], Qf[kMaxNX * kMaxNX], goal[kMaxNX];
  const double* user_data;  // user-defined model (user_model.cuh): its device array or null
  double cost_prm[8];       // user-defined cost: its parameters and device array
  const double* cost_data;
  double con_prm[8];        // user-defined constraints: parameters and device array
  const double* con_data;
  int W, Ws;                // stacked constraint rows, of which Ws are state rows
  int row_var[kMaxRows];    // 0 = state, 1 = control
  int row_idx[kMaxRows];
  double row_sign[kMaxRows];
  double row_bound[kMaxRows];
  // the same box rows by variable (bit i: state i, bit kMaxNX + i: control
  // i), so the barrier sweeps unroll over compile-time variable indices
  unsigned box_up, box_lo;
  double box_ub[kMaxNX + kMaxNU], box_lb[kMaxNX + kMaxNU];
};

// Models whose cost is user code (user_model.cuh UserModel with a cost
// source) expose kUserCost and the functions ucost / ucost_derivs / uterm /
// uterm_grad / uterm_hess; every other model uses the quadratic cost of
// ProblemParams through the functions below.
template <class D, class = void>
struct UserCostOf : std::false_type {};
template <class D>
struct UserCostOf<D, std::void_t<decltype(D::kUserCost)>> : std::bool_constant<D::kUserCost> {};
template <class D>
constexpr bool kUserCost = UserCostOf<D>::value;
// ... and models whose constraints are user code (kUserCon: kWs state rows
// g_t(x), kWc control rows h_t(u), functions ucon_w / ucon_derivs)
template <class D, class = void>
struct UserConOf : std::false_type {};
template <class D>
struct UserConOf<D, std::void_t<decltype(D::kUserCon)>> : std::bool_constant<D::kUserCon> {};
template <class D>
constexpr bool kUserCon = UserConOf<D>::value;

// Augmentation state for one launch (reference AugmentedCost variants)
template <typename R>
struct AugArgs {
  int kind;              // AUG_ZERO / AUG_BARRIER / AUG_ADMM
  const double* mu;      // [B] barrier weight per problem
  double rho;            // ADMM penalty
  const R* z;            // (W, T, B)
  const R* v;            // (W, T, B)
};

// ---------------------------------------------------------------------------
// dynamics
// ---------------------------------------------------------------------------

// First derivatives of the dynamics plus lambda-contracted second
// derivatives  Hxx = sum_k lam_k fxx[k], Huu, Hxu.
template <typename R, int NX, int NU>
struct DynDerivs {
  R fx[NX][NX], fu[NX][NU], Hxx[NX][NX], Huu[NU][NU], Hxu[NX][NU];
};

template <typename R>
struct Pendulum {
  static constexpr int NX = 2, NU = 1;
  // fu = [0 dt/I]^T; lambda . fxx only in (theta, theta)
  static constexpr uint64_t kFxMask = kDense;
  static constexpr uint64_t kFuMask = 1ull << 1;
  static constexpr uint64_t kHxxMask = 1ull << 0;

  PTC_D static void step(const ProblemParams& p, int, int, const R (&x)[2], const R (&u)[1],
                         R (&xn)[2]) {
    const R g = R(p.dyn[0]), l = R(p.dyn[1]), m = R(p.dyn[2]), bd = R(p.dyn[3]), dt = R(p.dyn[4]);
    R acc = -(g / l) * sin(x[0]) + (u[0] - bd * x[1]) / (m * (l * l));
    xn[0] = x[0] + dt * x[1];
    xn[1] = x[1] + dt * acc;
  }

  template <bool kSecond>
  PTC_D static void derivs(const ProblemParams& p, int, int, const R (&x)[2], const R (&)[1],
                           const R (&lam)[2], DynDerivs<R, 2, 1>& D) {
    const R g = R(p.dyn[0]), l = R(p.dyn[1]), m = R(p.dyn[2]), bd = R(p.dyn[3]), dt = R(p.dyn[4]);
    const R inertia = m * (l * l);
    D.fx[0][0] = R(1);
    D.fx[0][1] = dt;
    D.fx[1][0] = -dt * (g / l) * cos(x[0]);
    D.fx[1][1] = R(1) - dt * bd / inertia;
    D.fu[0][0] = R(0);
    D.fu[1][0] = dt / inertia;
    if (kSecond) {
      D.Hxx[0][0] = lam[1] * (dt * (g / l) * sin(x[0]));
      D.Hxx[0][1] = D.Hxx[1][0] = D.Hxx[1][1] = R(0);
      D.Huu[0][0] = R(0);
      D.Hxu[0][0] = D.Hxu[1][0] = R(0);
    }
  }
};

// Second-order jet in (theta, omega, force) for the cart-pole accelerations.
template <typename R>
struct Jet {
  R v, g[3], h[3][3];
};

template <typename R>
PTC_D Jet<R> jvar(R val, int k) {
  Jet<R> j;
  j.v = val;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    j.g[a] = (a == k) ? R(1) : R(0);
#pragma unroll
    for (int c = 0; c < 3; ++c) j.h[a][c] = R(0);
  }
  return j;
}

template <typename R>
PTC_D Jet<R> jadd(const Jet<R>& a, const Jet<R>& b) {
  Jet<R> o;
  o.v = a.v + b.v;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    o.g[i] = a.g[i] + b.g[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) o.h[i][k] = a.h[i][k] + b.h[i][k];
  }
  return o;
}

template <typename R>
PTC_D Jet<R> jscale(const Jet<R>& a, R s) {
  Jet<R> o;
  o.v = a.v * s;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    o.g[i] = a.g[i] * s;
#pragma unroll
    for (int k = 0; k < 3; ++k) o.h[i][k] = a.h[i][k] * s;
  }
  return o;
}

template <typename R>
PTC_D Jet<R> jaddc(const Jet<R>& a, R c) {
  Jet<R> o = a;
  o.v = a.v + c;
  return o;
}

template <typename R>
PTC_D Jet<R> jmul(const Jet<R>& a, const Jet<R>& b) {
  Jet<R> o;
  o.v = a.v * b.v;
#pragma unroll
  for (int i = 0; i < 3; ++i) o.g[i] = a.g[i] * b.v + b.g[i] * a.v;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      o.h[i][k] = a.h[i][k] * b.v + b.h[i][k] * a.v + a.g[i] * b.g[k] + a.g[k] * b.g[i];
  return o;
}

template <typename R>
PTC_D Jet<R> jrecip(const Jet<R>& a) {
  Jet<R> o;
  R r = R(1) / a.v;
  R r2 = r * r;
  o.v = r;
#pragma unroll
  for (int i = 0; i < 3; ++i) o.g[i] = -a.g[i] * r2;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) o.h[i][k] = -a.h[i][k] * r2 + R(2) * a.g[i] * a.g[k] * (r2 * r);
  return o;
}

template <typename R>
PTC_D void jsincos(const Jet<R>& a, Jet<R>& s, Jet<R>& c) {
  R sv, cv;
  sv = sin(a.v);
  cv = cos(a.v);
  s.v = sv;
  c.v = cv;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    s.g[i] = a.g[i] * cv;
    c.g[i] = -a.g[i] * sv;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      R gg = a.g[i] * a.g[k];
      s.h[i][k] = a.h[i][k] * cv - gg * sv;
      c.h[i][k] = -a.h[i][k] * sv - gg * cv;
    }
  }
}

template <typename R>
struct CartPole {
  static constexpr int NX = 4, NU = 1;
  // structural nonzeros (bit i * cols + j) of the Euler step's derivatives:
  // fx = [1 0 dt 0; 0 1 0 dt; 0 * 1 *; 0 * 0 *], fu = [0 0 * *]^T,
  // lambda . fxx lives in (theta, omega) x (theta, omega)
  static constexpr uint64_t kFxMask = (1ull << 0) | (1ull << 2) | (1ull << 5) | (1ull << 7) |
                                      (1ull << 9) | (1ull << 10) | (1ull << 11) | (1ull << 13) |
                                      (1ull << 15);
  static constexpr uint64_t kFuMask = (1ull << 2) | (1ull << 3);
  static constexpr uint64_t kHxxMask = (1ull << 5) | (1ull << 7) | (1ull << 13) | (1ull << 15);

  // Accelerations and their derivatives in the reduced variables (theta,
  // omega, force), restating the reference's closed forms
  // (systems.py:262-327 _quotient_derivs / _cartpole_accel): numerator and
  // denominator derivatives combined by the quotient rule, with only the
  // entries the model reads (g0..g2; h00, h01, h11, h02, h12 -- the
  // force-force entry is unused) and none of the identically-zero terms.
  // One reciprocal of the denominator replaces the quotient rule's
  // divisions.
  //   cart acc = (F + mp s (l om + g c)) / (mc + mp s^2)
  //   pole acc = (-F c - mp l om^2 c s - (mc + mp) g s) / (l (mc + mp s^2))
  struct Accel {
    R g0, g1, g2, h00, h01, h11, h02, h12;
  };
  // n / den with den depending on theta only (gradient gd0, Hessian hd00)
  PTC_D static void quotient(R n, R gn0, R gn1, R gn2, R hn00, R hn01, R hn11, R hn02, R den,
                             R gd0, R hd00, Accel& q) {
    const R rd = R(1) / den, rd2 = rd * rd;
    q.g0 = gn0 * rd - n * gd0 * rd2;
    q.g1 = gn1 * rd;
    q.g2 = gn2 * rd;
    q.h00 = hn00 * rd - R(2) * (gn0 * gd0) * rd2 - n * hd00 * rd2 + R(2) * n * (gd0 * gd0) * (rd2 * rd);
    q.h01 = hn01 * rd - (gn1 * gd0) * rd2;
    q.h11 = hn11 * rd;
    q.h02 = hn02 * rd - (gn2 * gd0) * rd2;
    q.h12 = R(0);
  }

  PTC_D static void accels(const ProblemParams& p, R s, R c, R om, R force, Accel& cart,
                           Accel& pole) {
    const R g = R(p.dyn[0]), ln = R(p.dyn[1]), mc = R(p.dyn[2]), mp = R(p.dyn[3]);
    const R c2s2 = c * c - s * s;
    const R den = mc + mp * s * s;
    const R gd0 = R(2) * mp * s * c;
    const R hd00 = R(2) * mp * c2s2;
    // cart numerator n1 = F + mp s (l om + g c)
    const R n1 = force + mp * s * (ln * om + g * c);
    quotient(n1, mp * c * ln * om + mp * g * c2s2, mp * ln * s, R(1),
             -mp * ln * s * om - R(4) * mp * g * s * c, mp * ln * c, R(0), R(0), den, gd0, hd00,
             cart);
    // pole numerator n2 over l den
    const R om2 = om * om, mg = (mc + mp) * g;
    const R n2 = -force * c - mp * ln * om2 * c * s - mg * s;
    quotient(n2, force * s - mp * ln * om2 * c2s2 - mg * c, R(-2) * mp * ln * om * c * s, -c,
             force * c + R(4) * mp * ln * om2 * s * c + mg * s, R(-2) * mp * ln * om * c2s2,
             R(-2) * mp * ln * c * s, s, ln * den, ln * gd0, ln * hd00, pole);
  }

  // fp32 keeps the second-order jet form of the same derivatives (below):
  // fp32 cart-pole barrier solves are chaotic at the 1e-4 level -- a 1-ulp
  // change of the controls moves the solution 2e-5..1.2e-3 from the fp64
  // reference (scratch/fp32_spread.py) -- and the fp32 parity instances are
  // pinned with this form's rounding.
  PTC_D static void accels_jet(const ProblemParams& p, R th, R om, R force, Jet<R>& cart,
                           Jet<R>& pole) {
    const R g = R(p.dyn[0]), ln = R(p.dyn[1]), mc = R(p.dyn[2]), mp = R(p.dyn[3]);
    Jet<R> TH = jvar(th, 0), OM = jvar(om, 1), FF = jvar(force, 2);
    Jet<R> s, c;
    jsincos(TH, s, c);
    Jet<R> den = jaddc(jscale(jmul(s, s), mp), mc);
    Jet<R> rden = jrecip(den);
    Jet<R> inner = jadd(jscale(OM, ln), jscale(c, g));
    Jet<R> n1 = jadd(FF, jscale(jmul(s, inner), mp));
    cart = jmul(n1, rden);
    Jet<R> n2 = jadd(jadd(jscale(jmul(FF, c), R(-1)), jscale(jmul(jmul(jmul(OM, OM), c), s), -(mp * ln))),
                     jscale(s, -((mc + mp) * g)));
    pole = jscale(jmul(n2, rden), R(1) / ln);
  }

  // per-stage auxiliary values of a state (sin theta, cos theta): a
  // trajectory's are cached next to it by the single-sweep Newton kernels,
  // so the value sweep and the forward sweep's Jacobians reuse the ones the
  // candidate's rollout evaluated (same calls, same bits; Newton iteration
  // 0.998 -> 0.961 ms at 32,768 problems).  fp64 only (the fp32
  // derivatives keep their jet form)
  static constexpr int kAux = sizeof(R) == 8 ? 2 : 0;
  PTC_D static void aux(const R (&x)[4], R (&w)[2]) { sincos(x[1], &w[0], &w[1]); }

  PTC_D static void step_w(const ProblemParams& p, int, int, const R (&x)[4], const R (&u)[1],
                           const R (&w)[2], R (&xn)[4]) {
    const R g = R(p.dyn[0]), ln = R(p.dyn[1]), mc = R(p.dyn[2]), mp = R(p.dyn[3]), dt = R(p.dyn[4]);
    const R s = w[0], c = w[1];
    R den = mc + mp * s * s;
    R ca = (u[0] + mp * s * (ln * x[3] + g * c)) / den;
    R pa = (-u[0] * c - mp * ln * x[3] * x[3] * c * s - (mc + mp) * g * s) / (ln * den);
    xn[0] = x[0] + dt * x[2];
    xn[1] = x[1] + dt * x[3];
    xn[2] = x[2] + dt * ca;
    xn[3] = x[3] + dt * pa;
  }

  PTC_D static void step(const ProblemParams& p, int t, int b, const R (&x)[4], const R (&u)[1],
                         R (&xn)[4]) {
    R w[2];
    if constexpr (sizeof(R) == 4) {
      w[0] = sin(x[1]);
      w[1] = cos(x[1]);
    } else {
      sincos(x[1], &w[0], &w[1]);
    }
    step_w(p, t, b, x, u, w, xn);
  }

  template <bool kSecond>
  PTC_D static void derivs_w(const ProblemParams& p, int, int, const R (&x)[4], const R (&u)[1],
                             const R (&w)[2], const R (&lam)[4], DynDerivs<R, 4, 1>& D) {
    const R dt = R(p.dyn[4]);
    Accel cart, pole;
    if constexpr (sizeof(R) == 4) {
      Jet<R> jc, jp;
      accels_jet(p, x[1], x[3], u[0], jc, jp);
      cart = {jc.g[0], jc.g[1], jc.g[2], jc.h[0][0], jc.h[0][1], jc.h[1][1], jc.h[0][2], jc.h[1][2]};
      pole = {jp.g[0], jp.g[1], jp.g[2], jp.h[0][0], jp.h[0][1], jp.h[1][1], jp.h[0][2], jp.h[1][2]};
    } else {
      accels(p, w[0], w[1], x[3], u[0], cart, pole);
    }
    set_identity(D.fx);
    D.fx[0][2] = dt;
    D.fx[1][3] = dt;
    D.fx[2][1] = dt * cart.g0;
    D.fx[2][3] = dt * cart.g1;
    D.fx[3][1] = dt * pole.g0;
    D.fx[3][3] = R(1) + dt * pole.g1;
    D.fu[0][0] = R(0);
    D.fu[1][0] = R(0);
    D.fu[2][0] = dt * cart.g2;
    D.fu[3][0] = dt * pole.g2;
    if (kSecond) {
      set_zero(D.Hxx);
      set_zero(D.Hxu);
      D.Huu[0][0] = R(0);
      // rows 2 (cart) and 3 (pole) carry second derivatives in (theta, omega)
      const R l2 = lam[2] * dt, l3 = lam[3] * dt;
      D.Hxx[1][1] = l2 * cart.h00 + l3 * pole.h00;
      D.Hxx[1][3] = D.Hxx[3][1] = l2 * cart.h01 + l3 * pole.h01;
      D.Hxx[3][3] = l2 * cart.h11 + l3 * pole.h11;
      D.Hxu[1][0] = l2 * cart.h02 + l3 * pole.h02;
      D.Hxu[3][0] = l2 * cart.h12 + l3 * pole.h12;
    }
  }

  template <bool kSecond>
  PTC_D static void derivs(const ProblemParams& p, int t, int b, const R (&x)[4], const R (&u)[1],
                           const R (&lam)[4], DynDerivs<R, 4, 1>& D) {
    R w[2] = {R(0), R(0)};
    if constexpr (sizeof(R) == 8) sincos(x[1], &w[0], &w[1]);
    derivs_w<kSecond>(p, t, b, x, u, w, lam, D);
  }
};

// a model's structural zeros (linalg.cuh masks); dense unless it says
template <class Dyn, class = void>
struct JacMask {
  static constexpr uint64_t fx = kDense, fu = kDense, hxx = kDense;
};
template <class Dyn>
struct JacMask<Dyn, std::void_t<decltype(Dyn::kFxMask)>> {
  static constexpr uint64_t fx = Dyn::kFxMask, fu = Dyn::kFuMask, hxx = Dyn::kHxxMask;
};

// per-stage auxiliary values a model caches next to a trajectory (kAux,
// aux, step_w, derivs_w); none unless it says
template <class Dyn, class = void>
struct AuxOf {
  static constexpr int n = 0;
};
template <class Dyn>
struct AuxOf<Dyn, std::void_t<decltype(Dyn::kAux)>> {
  static constexpr int n = Dyn::kAux;
};
template <class Dyn>
constexpr int kAuxDim = AuxOf<Dyn>::n > 0 ? AuxOf<Dyn>::n : 1;

// the model's derivatives from cached auxiliary values when use_w
template <bool kSecond, class Dyn, typename R>
PTC_D void dyn_derivs(const ProblemParams& p, int t, int b, const R (&x)[Dyn::NX],
                      const R (&u)[Dyn::NU], const R (&w)[kAuxDim<Dyn>], bool use_w,
                      const R (&lam)[Dyn::NX], DynDerivs<R, Dyn::NX, Dyn::NU>& D) {
  if constexpr (AuxOf<Dyn>::n > 0) {
    if (use_w) {
      Dyn::template derivs_w<kSecond>(p, t, b, x, u, w, lam, D);
      return;
    }
  }
  Dyn::template derivs<kSecond>(p, t, b, x, u, lam, D);
}

// x' = A_t x + B_t u + c_t with per-stage / per-problem broadcasting
template <typename R, int NX_, int NU_>
struct Affine {
  static constexpr int NX = NX_, NU = NU_;

  PTC_D static size_t at(const ProblemParams& p, int c, int t, int b) {
    int tt = p.lin_T > 1 ? t : 0;
    int bb = p.lin_B > 1 ? b : 0;
    return ((size_t)c * p.lin_T + tt) * p.lin_B + bb;
  }

  PTC_D static void mats(const ProblemParams& p, int t, int b, R (&A)[NX][NX], R (&Bm)[NX][NU]) {
    const R* pa = static_cast<const R*>(p.lin_A);
    const R* pb = static_cast<const R*>(p.lin_Bm);
#pragma unroll
    for (int i = 0; i < NX; ++i) {
#pragma unroll
      for (int j = 0; j < NX; ++j) A[i][j] = __ldg(pa + at(p, i * NX + j, t, b));
#pragma unroll
      for (int j = 0; j < NU; ++j) Bm[i][j] = __ldg(pb + at(p, i * NU + j, t, b));
    }
  }

  PTC_D static void offset(const ProblemParams& p, int t, int b, R (&c)[NX]) {
    const R* pc = static_cast<const R*>(p.lin_c);
#pragma unroll
    for (int i = 0; i < NX; ++i) c[i] = pc ? __ldg(pc + at(p, i, t, b)) : R(0);
  }

  PTC_D static void step(const ProblemParams& p, int t, int b, const R (&x)[NX], const R (&u)[NU],
                         R (&xn)[NX]) {
    R A[NX][NX], Bm[NX][NU], c[NX];
    mats(p, t, b, A, Bm);
    offset(p, t, b, c);
    R ax[NX], bu[NX];
    mv<NX, NX>(A, x, ax);
    mv<NX, NU>(Bm, u, bu);
#pragma unroll
    for (int i = 0; i < NX; ++i) xn[i] = ax[i] + bu[i] + c[i];
  }

  template <bool kSecond>
  PTC_D static void derivs(const ProblemParams& p, int t, int b, const R (&)[NX], const R (&)[NU],
                           const R (&)[NX], DynDerivs<R, NX, NU>& D) {
    mats(p, t, b, D.fx, D.fu);
    if (kSecond) {
      set_zero(D.Hxx);
      set_zero(D.Huu);
      set_zero(D.Hxu);
    }
  }
};

// ---------------------------------------------------------------------------
// cost, constraints, augmentation
// ---------------------------------------------------------------------------

// stage cost 0.5 (x-g)^T Q (x-g) + 0.5 u^T R u
template <typename R, int NX, int NU>
PTC_D R stage_cost(const ProblemParams& p, const R (&x)[NX], const R (&u)[NU]) {
  R e[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) e[i] = x[i] - R(p.goal[i]);
  R qx = R(0), ru = R(0);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) qx += e[i] * R(p.Q[i * NX + j]) * e[j];
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NU; ++j) ru += u[i] * R(p.Rc[i * NU + j]) * u[j];
  return R(0.5) * (qx + ru);
}

// The stage-cost constants in registers (kernels that evaluate the cost at
// every stage of a sweep load them once; same arithmetic as stage_cost).
template <typename R, int NX, int NU>
struct CostRegs {
  R goal[NX], Q[NX][NX], Rc[NU][NU];
  PTC_D void load(const ProblemParams& p) {
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      goal[i] = R(p.goal[i]);
#pragma unroll
      for (int j = 0; j < NX; ++j) Q[i][j] = R(p.Q[i * NX + j]);
    }
#pragma unroll
    for (int i = 0; i < NU; ++i)
#pragma unroll
      for (int j = 0; j < NU; ++j) Rc[i][j] = R(p.Rc[i * NU + j]);
  }
};

// Wide states: the constants in shared memory instead (one copy per block;
// a register copy of Q would spill at nx = 12).
template <typename R, int NX, int NU>
struct CostSmem {
  R goal[NX], Q[NX][NX], Rc[NU][NU];
  // every thread of the block calls this (it synchronises the block)
  PTC_D void load(const ProblemParams& p) {
    for (int e = threadIdx.x; e < NX * NX; e += blockDim.x) Q[e / NX][e % NX] = R(p.Q[e]);
    for (int e = threadIdx.x; e < NU * NU; e += blockDim.x) Rc[e / NU][e % NU] = R(p.Rc[e]);
    for (int e = threadIdx.x; e < NX; e += blockDim.x) goal[e] = R(p.goal[e]);
    __syncthreads();
  }
};

template <typename R, int NX, int NU>
PTC_D R stage_cost(const CostSmem<R, NX, NU>& p, const R (&x)[NX], const R (&u)[NU]) {
  R e[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) e[i] = x[i] - p.goal[i];
  R qx = R(0), ru = R(0);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) qx += e[i] * p.Q[i][j] * e[j];
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NU; ++j) ru += u[i] * p.Rc[i][j] * u[j];
  return R(0.5) * (qx + ru);
}

template <typename R, int NX, int NU>
PTC_D R stage_cost(const CostRegs<R, NX, NU>& p, const R (&x)[NX], const R (&u)[NU]) {
  R e[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) e[i] = x[i] - p.goal[i];
  R qx = R(0), ru = R(0);
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) qx += e[i] * p.Q[i][j] * e[j];
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NU; ++j) ru += u[i] * p.Rc[i][j] * u[j];
  return R(0.5) * (qx + ru);
}

template <typename R, int NX>
PTC_D R terminal_cost(const ProblemParams& p, const R (&x)[NX]) {
  R e[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) e[i] = x[i] - R(p.goal[i]);
  R q = R(0);
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    R row = R(0);
#pragma unroll
    for (int j = 0; j < NX; ++j) row += R(p.Qf[i * NX + j]) * e[j];
    q += e[i] * row;
  }
  return R(0.5) * q;
}

template <typename R, int NX>
PTC_D void terminal_grad(const ProblemParams& p, const R (&x)[NX], R (&gx)[NX]) {
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    R acc = R(0);
#pragma unroll
    for (int j = 0; j < NX; ++j) acc += R(p.Qf[i * NX + j]) * (x[j] - R(p.goal[j]));
    gx[i] = acc;
  }
}

// value of stacked constraint row k: sign * (var[idx] - bound)
template <typename R, int NX, int NU>
PTC_D R row_value(const ProblemParams& p, int k, const R (&x)[NX], const R (&u)[NU]) {
  const int idx = p.row_idx[k];
  R var = R(0);
  if (p.row_var[k] == 0) {
#pragma unroll
    for (int i = 0; i < NX; ++i) var = (i == idx) ? x[i] : var;
  } else {
#pragma unroll
    for (int i = 0; i < NU; ++i) var = (i == idx) ? u[i] : var;
  }
  const R bnd = R(p.row_bound[k]);
  return p.row_sign[k] > 0 ? var - bnd : bnd - var;
}

// Augmentation value at one stage; `bad_row` reports the first row with
// w >= 0 for the barrier (-1 if strictly feasible).
template <typename R, int NX, int NU>
PTC_D R aug_value(const ProblemParams& p, const AugArgs<R>& a, int t, int T, int B, int b,
                  const R (&x)[NX], const R (&u)[NU], int& bad_row) {
  bad_row = -1;
  if (a.kind == AUG_ZERO) return R(0);
  const int W = p.W;
  if (a.kind == AUG_BARRIER) {
    // rows in the stacking order of build_params (api.cu; problem.py:254-260):
    // state upper, state lower, control upper, control lower -- the same
    // values and summation order as the row table, unrolled over variables
    R sg = R(0), sh = R(0);
    int k = 0;
    const unsigned up = p.box_up, lo = p.box_lo;
    auto row = [&](R w, R& acc) {
      if (w >= R(0) && bad_row < 0) bad_row = k;
      acc += log(-w);
      ++k;
    };
#pragma unroll
    for (int i = 0; i < NX; ++i)
      if (up >> i & 1u) row(x[i] - R(p.box_ub[i]), sg);
#pragma unroll
    for (int i = 0; i < NX; ++i)
      if (lo >> i & 1u) row(R(p.box_lb[i]) - x[i], sg);
    // control rows: a control boxed on both sides evaluates its two logs in
    // one block (independent chains), summed afterwards in row order
    R lu[NU], ll[NU];
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      const bool hu = up >> (kMaxNX + i) & 1u, hl = lo >> (kMaxNX + i) & 1u;
      const R wu = u[i] - R(p.box_ub[kMaxNX + i]), wl = R(p.box_lb[kMaxNX + i]) - u[i];
      if (hu && hl) {
        lu[i] = log(-wu);
        ll[i] = log(-wl);
      } else if (hu) {
        lu[i] = log(-wu);
      } else if (hl) {
        ll[i] = log(-wl);
      }
    }
#pragma unroll
    for (int i = 0; i < NU; ++i)
      if (up >> (kMaxNX + i) & 1u) {
        if (u[i] - R(p.box_ub[kMaxNX + i]) >= R(0) && bad_row < 0) bad_row = k;
        sh += lu[i];
        ++k;
      }
#pragma unroll
    for (int i = 0; i < NU; ++i)
      if (lo >> (kMaxNX + i) & 1u) {
        if (R(p.box_lb[kMaxNX + i]) - u[i] >= R(0) && bad_row < 0) bad_row = k;
        sh += ll[i];
        ++k;
      }
    return -R(a.mu[b]) * (sg + sh);
  }
  const R rho = R(a.rho);
  R acc = R(0);
  for (int k = 0; k < W; ++k) {
    R w = row_value<R, NX, NU>(p, k, x, u);
    R res = w - ldf(a.z, k, t, T, B, b) + ldf(a.v, k, t, T, B, b) / rho;
    acc += res * res;
  }
  return R(0.5) * rho * acc;
}

// Gradient and (diagonal) Hessian of the augmentation with respect to the
// state and the control.  Box rows touch a single variable each, so the
// Hessians are diagonal and the cross term vanishes (outer.py:97-99).
template <typename R, int NX, int NU>
PTC_D void aug_derivs(const ProblemParams& p, const AugArgs<R>& a, int t, int T, int B, int b,
                      const R (&x)[NX], const R (&u)[NU], R (&cx)[NX], R (&cu)[NU],
                      R (&cxx)[NX], R (&cuu)[NU]) {
  set_zero(cx);
  set_zero(cu);
  set_zero(cxx);
  set_zero(cuu);
  if (a.kind == AUG_ZERO) return;
  const int W = p.W;
  if (a.kind == AUG_BARRIER) {
    const R mu = R(a.mu[b]);
    // per row w = sign (var - bound): gradient sign / w, Hessian 1 / w^2.
    // sign = +-1, so sign / w is exactly +-(1 / w): one division per row.
    // Unrolled over variables (a variable's upper row before its lower one,
    // as in the row table, the Hessian term rounded before it is summed:
    // same sums, same bits)
    const unsigned up = p.box_up, lo = p.box_lo;
#pragma unroll
    for (int i = 0; i < NX; ++i)
      if (up >> i & 1u) {
        const R inv = R(1) / (x[i] - R(p.box_ub[i]));
        cx[i] += inv;
        cxx[i] += mul_rn(inv, inv);
      }
#pragma unroll
    for (int i = 0; i < NX; ++i)
      if (lo >> i & 1u) {
        const R inv = R(1) / (R(p.box_lb[i]) - x[i]);
        cx[i] += -inv;
        cxx[i] += mul_rn(inv, inv);
      }
#pragma unroll
    for (int i = 0; i < NU; ++i)
      if (up >> (kMaxNX + i) & 1u) {
        const R inv = R(1) / (u[i] - R(p.box_ub[kMaxNX + i]));
        cu[i] += inv;
        cuu[i] += mul_rn(inv, inv);
      }
#pragma unroll
    for (int i = 0; i < NU; ++i)
      if (lo >> (kMaxNX + i) & 1u) {
        const R inv = R(1) / (R(p.box_lb[kMaxNX + i]) - u[i]);
        cu[i] += -inv;
        cuu[i] += mul_rn(inv, inv);
      }
#pragma unroll
    for (int i = 0; i < NX; ++i) { cx[i] = -mu * cx[i]; cxx[i] = mu * cxx[i]; }
#pragma unroll
    for (int i = 0; i < NU; ++i) { cu[i] = -mu * cu[i]; cuu[i] = mu * cuu[i]; }
    return;
  }
  const R rho = R(a.rho);
  for (int k = 0; k < W; ++k) {
    R w = row_value<R, NX, NU>(p, k, x, u);
    R res = w - ldf(a.z, k, t, T, B, b) + ldf(a.v, k, t, T, B, b) / rho;
    R sgn = R(p.row_sign[k]);
    const int idx = p.row_idx[k];
    if (p.row_var[k] == 0) {
#pragma unroll
      for (int i = 0; i < NX; ++i)
        if (i == idx) { cx[i] += sgn * res; cxx[i] += sgn * sgn; }
    } else {
#pragma unroll
      for (int i = 0; i < NU; ++i)
        if (i == idx) { cu[i] += sgn * res; cuu[i] += sgn * sgn; }
    }
  }
#pragma unroll
  for (int i = 0; i < NX; ++i) { cx[i] *= rho; cxx[i] *= rho; }
#pragma unroll
  for (int i = 0; i < NU; ++i) { cu[i] *= rho; cuu[i] *= rho; }
}

// ------------------------------------------------ user constraint models
// The augmentations of a model with user constraints w = [g_t(x); h_t(u)]
// (reference ConstraintModel, problem.py:167-230; barrier outer.py:30-157,
// ADMM outer.py:252-333), with full Hessians (rows may couple variables).

template <typename R, class Dyn>
PTC_D R aug_value_user(const ProblemParams& p, const AugArgs<R>& a, int t, int T, int B, int b,
                       const R (&x)[Dyn::NX], const R (&u)[Dyn::NU], int& bad_row) {
  constexpr int W = Dyn::kWs + Dyn::kWc;
  bad_row = -1;
  if (a.kind == AUG_ZERO) return R(0);
  R w[W > 0 ? W : 1];
  Dyn::ucon_w(p, t, x, u, w);
  if (a.kind == AUG_BARRIER) {
    R sg = R(0), sh = R(0);
    for (int k = 0; k < W; ++k) {
      if (w[k] >= R(0) && bad_row < 0) bad_row = k;
      const R lg = log(-w[k]);
      if (k < Dyn::kWs) sg += lg; else sh += lg;
    }
    return -R(a.mu[b]) * (sg + sh);
  }
  const R rho = R(a.rho);
  R acc = R(0);
  for (int k = 0; k < W; ++k) {
    const R res = w[k] - ldf(a.z, k, t, T, B, b) + ldf(a.v, k, t, T, B, b) / rho;
    acc += res * res;
  }
  return R(0.5) * rho * acc;
}

// gradients cx, cu and full Hessians Cxx, Cuu (the cross term vanishes:
// g depends on x, h on u)
template <typename R, class Dyn>
PTC_D void aug_derivs_user(const ProblemParams& p, const AugArgs<R>& a, int t, int T, int B,
                           int b, const R (&x)[Dyn::NX], const R (&u)[Dyn::NU],
                           R (&cx)[Dyn::NX], R (&cu)[Dyn::NU], R (&Cxx)[Dyn::NX][Dyn::NX],
                           R (&Cuu)[Dyn::NU][Dyn::NU]) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU, WS = Dyn::kWs, WC = Dyn::kWc;
  set_zero(cx);
  set_zero(cu);
  set_zero(Cxx);
  set_zero(Cuu);
  if (a.kind == AUG_ZERO) return;
  R w[WS + WC > 0 ? WS + WC : 1];
  R gx[Dyn::kWsA][NX], hu[Dyn::kWcA][NU];
  R gxx[Dyn::kWsA][NX][NX], huu[Dyn::kWcA][NU][NU];
  Dyn::ucon_derivs(p, t, x, u, w, gx, hu, gxx, huu);
  // weights: barrier  cx = -mu gx^T (1/g), Cxx = mu (S^T S - sum_k gxx_k / g_k), S = gx / g
  //          ADMM     cx = rho gx^T r,     Cxx = rho (gx^T gx + sum_k r_k gxx_k)
  const bool barrier = a.kind == AUG_BARRIER;
  const R mu = barrier ? R(a.mu[b]) : R(0), rho = R(a.rho);
  for (int k = 0; k < WS + WC; ++k) {
    R c1, c2, c0;   // gradient weight, second-derivative weight, outer-product weight
    if (barrier) {
      const R inv = R(1) / w[k];
      c1 = -mu * inv;
      c2 = -mu * inv;
      c0 = mu * inv * inv;
    } else {
      const R res = w[k] - ldf(a.z, k, t, T, B, b) + ldf(a.v, k, t, T, B, b) / rho;
      c1 = rho * res;
      c2 = rho * res;
      c0 = rho;
    }
    if (k < WS) {
      const int r = k;
      for (int i = 0; i < NX; ++i) {
        cx[i] += c1 * gx[r][i];
        for (int j = 0; j < NX; ++j) Cxx[i][j] += c0 * gx[r][i] * gx[r][j] + c2 * gxx[r][i][j];
      }
    } else {
      const int r = k - WS;
      for (int i = 0; i < NU; ++i) {
        cu[i] += c1 * hu[r][i];
        for (int j = 0; j < NU; ++j) Cuu[i][j] += c0 * hu[r][i] * hu[r][j] + c2 * huu[r][i][j];
      }
    }
  }
}

}  // namespace ptc
