// Kernels of one device-resident Newton iteration (reference newton.py:129-215)
// and of the two outer loops (outer.py:221-245 barrier, outer.py:392-435 ADMM).
//
// Every problem of a batch carries its own trust-region state (alpha, nu),
// iteration counter, history and outer-loop state in HBM; the control kernel
// replays the reference's accept/reject logic per problem, so a batch of
// independent MPC problems advances without any host round trip and a
// single problem reproduces the reference iteration sequence.
#pragma once

#include "lqr_kernels.cuh"
#include "models.cuh"

namespace ptc {

constexpr double kAlphaMax = 1e12;

enum : int { METHOD_NEWTON = 0, METHOD_BARRIER = 1, METHOD_ADMM = 2 };

struct Options {
  int method;
  double alpha0, nu0, inner_tol;
  int max_iters;
  double mu0, zeta, mu_tol;
  double rho, residual_tol;
  int max_outer;
  int hist_cap, round_cap;
  int keep_round_controls;
};

template <typename R>
struct NewtonArgs {
  int B, T;
  Plan plan;
  Options opt;
  const ProblemParams* pp;
  int aug_kind;            // AUG_* used inside the Newton solve
  // trajectories, double buffered: buffer q at X + q * xsz
  R *X, *U;
  size_t xsz, usz;
  // per-problem state [B]
  int *status, *phase, *parity, *flags, *iters, *term, *round, *hist_len, *bad_index, *n_running;
  double *alpha, *nu, *cur_cost, *cand_cost, *mu;
  double* bad_value;        // [B] w at bad_index (InfeasibleError.value)
  double* hist;            // (hist_cap, 5, B)
  double *round_mu, *round_cost, *round_rp, *round_rd;   // (round_cap, B)
  int *round_iters, *round_term;                          // (round_cap, B)
  R* round_U;              // (round_cap, nu, T, B) or null
  // ADMM consensus variables (W, T, B)
  R *z, *v;
  // expansion
  R *lam, *P, *Rm, *M, *d, *Fx, *Fu, *PT;
  // co-state scan tree
  R* cagg[kMaxLevels + 1];
  R* ccar[kMaxLevels + 1];
  // partial reductions per level-0 unit
  double* cpart[2];        // (3, P0, B): sum l, sum c, first infeasible index
  double* apart;           // (2, P0, B): ADMM primal / dual residual maxima
  double* red;             // (3, P0, B) from the propagation sweep
  // candidate rollout (see k_roll_gate / the parallel rollout below)
  int* rstate;             // [B] bit 0 skip, bit 1 converged, bit 2 result in xr
  double* rres;            // (P0, B) residual maxima of the rollout guess
  R* xr;                   // second state buffer of the parallel rollout (xsz)
  int pr_iters;            // Newton sweeps of the parallel rollout (0 = sequential)
  // time-block mode (ptc_solver_block_phase): stages [t_base, t_base + T) of
  // a longer horizon; blk_last = the block ends it (terminal cost / gradient)
  int blk, blk_last, t_base;
  int uterm;               // user-defined cost: the terminal cost is in the partials
  R* lam_in;               // (nx, 1, B) co-state entering at the block end
  R* x_in;                 // (nx, 1, B) state at the block start (rollout carry)
  const R* x0g;            // (nx, 1, B) the horizon's initial state (phase argument)
  // per-stage auxiliary values of each trajectory buffer (models with kAux,
  // single-sweep plans): buffer q at aux + q * auxsz, (kAux, T, B); aux_ok
  // [B] bit q = buffer q's values belong to its current states (cleared by
  // every host entry that writes the states)
  R* aux;
  size_t auxsz;
  int* aux_ok;
};

template <typename R>
PTC_D AugArgs<R> aug_of(const NewtonArgs<R>& a) {
  AugArgs<R> g;
  g.kind = a.aug_kind;
  g.mu = a.mu;
  g.rho = a.opt.rho;
  g.z = a.z;
  g.v = a.v;
  return g;
}

template <typename R, int NX>
PTC_D void ld_x(const NewtonArgs<R>& a, int q, int t, int b, R (&x)[NX]) {
  ld_vec(a.X + q * a.xsz, t, a.T + 1, a.B, b, x);
}

template <typename R, int NU>
PTC_D void ld_u(const NewtonArgs<R>& a, int q, int t, int b, R (&u)[NU]) {
  ld_vec(a.U + q * a.usz, t, a.T, a.B, b, u);
}

template <typename R>
PTC_D bool running(const NewtonArgs<R>& a, int b) { return a.status[b] == ST_RUNNING; }

// Per-problem partials (P0 rows per field) are folded by k_reduce_partials
// into row 0 when there are many of them (long horizons, small batches);
// consumers then read one row instead of looping over P0 in one thread.
constexpr int kReduceMin = 64;
PTC_HD int partial_rows(int P0) { return P0 > kReduceMin ? 1 : P0; }

enum : int { RED_SUM = 0, RED_MAX = 1, RED_FIRST = 2 };

// One block per problem: fold fields f of part[(f * P0 + j) * B + b] over j
// into row 0.  ops: 2 bits per field (RED_SUM, RED_MAX = NaN-propagating
// max, RED_FIRST = smallest non-negative value or -1, i.e. the first
// infeasible index since rows follow the stage order).
static __global__ void k_reduce_partials(double* part, int nf, int ops, int P0, int B) {
  __shared__ double sh[256];
  const int b = blockIdx.x;
  for (int f = 0; f < nf; ++f) {
    const int op = (ops >> (2 * f)) & 3;
    double acc = op == RED_SUM ? 0.0 : (op == RED_MAX ? 0.0 : -1.0);
    for (int j = threadIdx.x; j < P0; j += blockDim.x) {
      const double v = part[((size_t)f * P0 + j) * B + b];
      if (op == RED_SUM) acc += v;
      else if (op == RED_MAX) acc = nanmax(acc, v);
      else if (v >= 0.0 && (acc < 0.0 || v < acc)) acc = v;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
        const double o = sh[threadIdx.x + w];
        double& m = sh[threadIdx.x];
        if (op == RED_SUM) m += o;
        else if (op == RED_MAX) m = nanmax(m, o);
        else if (o >= 0.0 && (m < 0.0 || o < m)) m = o;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) part[((size_t)f * P0) * B + b] = sh[0];
    __syncthreads();
  }
}

// ------------------------------------------------------------ initialisation

template <typename R>
__global__ void k_init_state(NewtonArgs<R> a) {
  const int b = unit_id();
  if (b >= a.B) return;
  a.status[b] = ST_RUNNING;
  a.phase[b] = PH_NEED_COST | PH_NEED_EXP;
  a.parity[b] = 0;
  a.flags[b] = 0;
  a.iters[b] = 0;
  a.term[b] = TERM_NONE;
  a.round[b] = 0;
  a.hist_len[b] = 0;
  a.bad_index[b] = -1;
  a.bad_value[b] = NAN;
  a.alpha[b] = a.opt.alpha0;
  a.nu[b] = a.opt.nu0;
  a.cur_cost[b] = 0.0;
  a.cand_cost[b] = 0.0;
  a.mu[b] = a.opt.mu0;
  // outer-round records of rounds that never run read as zero
  for (int r = 0; r < a.opt.round_cap; ++r) {
    const size_t o = (size_t)r * a.B + b;
    a.round_iters[o] = 0;
    a.round_term[o] = TERM_NONE;
    a.round_mu[o] = 0.0;
    a.round_cost[o] = 0.0;
    a.round_rp[o] = 0.0;
    a.round_rd[o] = 0.0;
  }
  if (a.opt.method == METHOD_BARRIER && !(a.opt.mu0 > a.opt.mu_tol)) a.status[b] = ST_DONE;
}

// x_{t+1} == f_t(x_t, u_t) check of the initial trajectory (newton.py:118-126)
template <typename R, class Dyn>
__global__ void k_check_consistent(NewtonArgs<R> a, int* bad_t) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  const int i = unit_id();
  if (i >= a.T * a.B) return;
  const int b = i % a.B, t = i / a.B;
  R x[NX], u[NU], xn[NX], p[NX];
  ld_x(a, 0, t, b, x);
  ld_u(a, 0, t, b, u);
  ld_x(a, 0, t + 1, b, xn);
  Dyn::step(*a.pp, t, b, x, u, p);
  double gap = 0.0, mag = 0.0;
#pragma unroll
  for (int k = 0; k < NX; ++k) {
    gap = nanmax(gap, double(fabs(p[k] - xn[k])));
    mag = nanmax(mag, double(fabs(p[k])));
  }
  const double tol = (sizeof(R) == 8 ? 1e-8 : 1e-4) * (1.0 + mag);
  if (gap > tol || gap != gap) atomicMin(bad_t + b, t);
}

// ADMM start: z = Pi_C(w(x, u)), v = 0   (outer.py:409-410)
template <typename R, int NX, int NU, class Dyn = void>
__global__ void k_admm_init(NewtonArgs<R> a) {
  const int i = unit_id();
  if (i >= a.T * a.B) return;
  const int b = i % a.B, t = i / a.B;
  const ProblemParams& p = *a.pp;
  R x[NX], u[NU];
  ld_x(a, 0, t, b, x);
  ld_u(a, 0, t, b, u);
  if constexpr (!std::is_void_v<Dyn> && kUserCon<Dyn>) {
    constexpr int W = Dyn::kWs + Dyn::kWc;
    R w[W > 0 ? W : 1];
    Dyn::ucon_w(p, t, x, u, w);
    for (int k = 0; k < W; ++k) {
      stf(a.z, k, t, a.T, a.B, b, w[k] < R(0) ? w[k] : R(0));
      stf(a.v, k, t, a.T, a.B, b, R(0));
    }
    return;
  }
  for (int k = 0; k < p.W; ++k) {
    R w = row_value<R, NX, NU>(p, k, x, u);
    stf(a.z, k, t, a.T, a.B, b, w < R(0) ? w : R(0));
    stf(a.v, k, t, a.T, a.B, b, R(0));
  }
}

// ------------------------------------------------------- cost of a trajectory

// which = 0: current trajectory (only when PH_NEED_COST), 1: the candidate.
template <typename R, int NX, int NU, class Dyn = void>
__global__ void __launch_bounds__(128) k_cost_partials(NewtonArgs<R> a, int which) {
  // cost constants: registers for small states, the block's shared copy for
  // wide ones (loaded before any thread leaves)
  __shared__ CostSmem<R, NX, NU> cs_shared;
  if constexpr (NX >= 8) cs_shared.load(*a.pp);
  const int P0 = a.plan.units0();
  const int u0 = unit_id();
  if (u0 >= P0 * a.B) return;
  const int b = u0 % a.B, j = u0 / a.B;
  if (!running(a, b)) return;
  if (which == 0 && !(a.phase[b] & PH_NEED_COST)) return;
  const int q = which == 0 ? a.parity[b] : 1 - a.parity[b];
  const int T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const ProblemParams& p = *a.pp;
  const AugArgs<R> g = aug_of(a);
  double sl = 0.0, sc = 0.0;
  int bad = -1;
  CostRegs<R, NX, NU> cr;
  if constexpr (NX < 8) cr.load(p);
  for (int t = t0; t < t1; ++t) {
    R x[NX], u[NU];
    ld_x(a, q, t, b, x);
    ld_u(a, q, t, b, u);
    if constexpr (!std::is_void_v<Dyn> && kUserCost<Dyn>) sl += double(Dyn::ucost(p, t, x, u));
    else if constexpr (NX < 8) sl += double(stage_cost<R, NX, NU>(cr, x, u));
    else sl += double(stage_cost<R, NX, NU>(cs_shared, x, u));
    int br;
    if constexpr (!std::is_void_v<Dyn> && kUserCon<Dyn>)
      sc += double(aug_value_user<R, Dyn>(p, g, t, T, B, b, x, u, br));
    else
      sc += double(aug_value<R, NX, NU>(p, g, t, T, B, b, x, u, br));
    if (br >= 0 && bad < 0) bad = t * p.W + br;
  }
  if constexpr (!std::is_void_v<Dyn> && kUserCost<Dyn>) {
    if (j == P0 - 1) {   // the terminal cost rides in the last unit's partial
      R xT[NX];
      ld_x(a, q, T, b, xT);
      sl += double(Dyn::uterm(p, xT));
    }
  }
  double* cp = a.cpart[which];
  cp[((size_t)0 * P0 + j) * B + b] = sl;
  cp[((size_t)1 * P0 + j) * B + b] = sc;
  cp[((size_t)2 * P0 + j) * B + b] = double(bad);
}

// ------------------------------------------------------------ co-state scan

// level-0 up-sweep: fold the reverse maps lambda_t = q_t + fx_t^T lambda_{t+1}
// over a chunk (the last stage absorbs the terminal gradient, F = 0)
template <typename R, class Dyn>
__global__ void __launch_bounds__(128) k_costate_up0(NewtonArgs<R> a) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  const int P0 = a.plan.units0();
  const int u0 = unit_id();
  if (u0 >= P0 * a.B) return;
  const int b = u0 % a.B, j = u0 / a.B;
  if (!running(a, b) || !(a.phase[b] & PH_NEED_EXP)) return;
  const int q = a.parity[b];
  const int T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const ProblemParams& p = *a.pp;
  const AugArgs<R> g = aug_of(a);
  Aff<R, NX> acc;
  aff_identity(acc);
  for (int t = t1 - 1; t >= t0; --t) {
    R x[NX], u[NU], lam0[NX];
    ld_x(a, q, t, b, x);
    ld_u(a, q, t, b, u);
    set_zero(lam0);
    DynDerivs<R, NX, NU> D;
    Dyn::template derivs<false>(p, t, b, x, u, lam0, D);
    R cx[NX], cu[NU];
    if constexpr (kUserCon<Dyn>) {
      R Cxx[NX][NX], Cuu[NU][NU];
      aug_derivs_user<R, Dyn>(p, g, t, T, B, b, x, u, cx, cu, Cxx, Cuu);
    } else {
      R cxx[NX], cuu[NU];
      aug_derivs<R, NX, NU>(p, g, t, T, B, b, x, u, cx, cu, cxx, cuu);
    }
    Aff<R, NX> m;
    R ulx[NX];
    if constexpr (kUserCost<Dyn>) Dyn::ucost_grad(p, t, x, u, ulx);
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      R lx = R(0);
      if constexpr (kUserCost<Dyn>) {
        lx = ulx[i];
      } else {
#pragma unroll
        for (int k = 0; k < NX; ++k) lx += (x[k] - R(p.goal[k])) * R(p.Q[i * NX + k]);
      }
      m.e[i] = lx + cx[i];
#pragma unroll
      for (int k = 0; k < NX; ++k) m.F[i][k] = D.fx[k][i];
    }
    if (t == T - 1) {
      R xT[NX], lT[NX], fl[NX];
      ld_x(a, q, T, b, xT);
      if constexpr (kUserCost<Dyn>) Dyn::uterm_grad(p, xT, lT);
      else terminal_grad(p, xT, lT);
      mv<NX, NX>(m.F, lT, fl);
#pragma unroll
      for (int i = 0; i < NX; ++i) {
        m.e[i] += fl[i];
#pragma unroll
        for (int k = 0; k < NX; ++k) m.F[i][k] = R(0);
      }
    }
    Aff<R, NX> o;
    aff_compose(m, acc, o);
    acc = o;
  }
  st_aff(a.cagg[1], j, a.plan.n[1], B, b, acc);
}

// generic affine tree kernels shared by the co-state (reverse) scan
template <typename R, int NX>
__global__ void __launch_bounds__(128) k_costate_up(NewtonArgs<R> a, int l) {
  const int nl = a.plan.n[l], nu = a.plan.n[l + 1];
  const int u0 = unit_id();
  if (u0 >= nu * a.B) return;
  const int b = u0 % a.B, j = u0 / a.B;
  if (!running(a, b) || !(a.phase[b] & PH_NEED_EXP)) return;
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  Aff<R, NX> acc;
  ld_aff(a.cagg[l], last, nl, a.B, b, acc);
  for (int i = last - 1; i >= first; --i) {
    Aff<R, NX> m, o;
    ld_aff(a.cagg[l], i, nl, a.B, b, m);
    aff_compose(m, acc, o);
    acc = o;
  }
  st_aff(a.cagg[l + 1], j, nu, a.B, b, acc);
}

template <typename R, int NX>
__global__ void __launch_bounds__(128) k_costate_top(NewtonArgs<R> a) {
  const int b = unit_id();
  if (b >= a.B) return;
  if (!running(a, b) || !(a.phase[b] & PH_NEED_EXP)) return;
  const int L = a.plan.L, nL = a.plan.n[L];
  R c[NX];
  set_zero(c);
  for (int i = nL - 1; i >= 0; --i) {
    st_vec(a.ccar[L], i, nL, a.B, b, c);
    Aff<R, NX> m;
    ld_aff(a.cagg[L], i, nL, a.B, b, m);
    R y[NX];
    aff_apply(m, c, y);
#pragma unroll
    for (int k = 0; k < NX; ++k) c[k] = y[k];
  }
}

template <typename R, int NX>
__global__ void __launch_bounds__(128) k_costate_down(NewtonArgs<R> a, int l) {
  const int nl = a.plan.n[l], nu = a.plan.n[l + 1];
  const int u0 = unit_id();
  if (u0 >= nu * a.B) return;
  const int b = u0 % a.B, j = u0 / a.B;
  if (!running(a, b) || !(a.phase[b] & PH_NEED_EXP)) return;
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  R c[NX];
  ld_vec(a.ccar[l + 1], j, nu, a.B, b, c);
  for (int i = last; i >= first; --i) {
    st_vec(a.ccar[l], i, nl, a.B, b, c);
    Aff<R, NX> m;
    ld_aff(a.cagg[l], i, nl, a.B, b, m);
    R y[NX];
    aff_apply(m, c, y);
#pragma unroll
    for (int k = 0; k < NX; ++k) c[k] = y[k];
  }
}

// Second-order data of stage t of the augmented Lagrangian at (x_t, u_t)
// with the next co-state lambda_{t+1} (passes.py:155-185): P, R, M, d, Fx,
// Fu, plus lambda_t = lx + cx + fx^T lambda_{t+1}.  Shared by the co-state
// sweep (which stores it) and the fused value sweep (which consumes it in
// registers), so both paths produce identical bits.
template <typename R, class Dyn>
PTC_D void stage_expansion(const NewtonArgs<R>& a, const ProblemParams& p, const AugArgs<R>& g,
                           int t, int b, const R (&x)[Dyn::NX], const R (&u)[Dyn::NU],
                           const R (&w)[kAuxDim<Dyn>], bool use_w,
                           const R (&ln)[Dyn::NX], Stage<R, Dyn::NX, Dyn::NU>& st,
                           R (&lt)[Dyn::NX]) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  constexpr uint64_t FxM = JacMask<Dyn>::fx, FuM = JacMask<Dyn>::fu, HxxM = JacMask<Dyn>::hxx;
  DynDerivs<R, NX, NU> D;
  dyn_derivs<true, Dyn>(p, t, b, x, u, w, use_w, ln, D);
  if constexpr (kUserCost<Dyn> || kUserCon<Dyn>) {
    // a user cost and / or user constraints: l's and the augmentation's
    // derivatives as full matrices (passes.py:171-181 adds lxx + cxx +
    // lambda fxx etc. in this order)
    R lx[NX], lu[NU], lxx[NX][NX], luu[NU][NU], lxu[NX][NU];
    if constexpr (kUserCost<Dyn>) {
      Dyn::ucost_derivs(p, t, x, u, lx, lu, lxx, luu, lxu);
    } else {
      set_zero(lxu);
      for (int i = 0; i < NX; ++i) {
        R acc = R(0);
        for (int k = 0; k < NX; ++k) {
          acc += (x[k] - R(p.goal[k])) * R(p.Q[i * NX + k]);
          lxx[i][k] = R(p.Q[i * NX + k]);
        }
        lx[i] = acc;
      }
      for (int i = 0; i < NU; ++i) {
        R acc = R(0);
        for (int k = 0; k < NU; ++k) {
          acc += u[k] * R(p.Rc[i * NU + k]);
          luu[i][k] = R(p.Rc[i * NU + k]);
        }
        lu[i] = acc;
      }
    }
    R cx[NX], cu[NU], Cxx[NX][NX], Cuu[NU][NU];
    if constexpr (kUserCon<Dyn>) {
      aug_derivs_user<R, Dyn>(p, g, t, a.T, a.B, b, x, u, cx, cu, Cxx, Cuu);
    } else {
      R cxx[NX], cuu[NU];
      aug_derivs<R, NX, NU>(p, g, t, a.T, a.B, b, x, u, cx, cu, cxx, cuu);
      set_zero(Cxx);
      set_zero(Cuu);
      for (int i = 0; i < NX; ++i) Cxx[i][i] = cxx[i];
      for (int i = 0; i < NU; ++i) Cuu[i][i] = cuu[i];
    }
    for (int i = 0; i < NX; ++i)
      for (int k = 0; k < NX; ++k) st.P[i][k] = (lxx[i][k] + Cxx[i][k]) + D.Hxx[i][k];
    symmetrize<NX>(st.P);
    for (int i = 0; i < NU; ++i)
      for (int k = 0; k < NU; ++k) st.Rr[i][k] = (luu[i][k] + Cuu[i][k]) + D.Huu[i][k];
    symmetrize<NU>(st.Rr);
    R ftl[NU], fxl[NX];
    mtv<NU, NX, R, FuM>(D.fu, ln, ftl);
    mtv<NX, NX, R, FxM>(D.fx, ln, fxl);
    for (int i = 0; i < NU; ++i) st.d[i] = (lu[i] + cu[i]) + ftl[i];
    for (int i = 0; i < NX; ++i) lt[i] = (lx[i] + cx[i]) + fxl[i];
    for (int i = 0; i < NX; ++i) {
      for (int k = 0; k < NU; ++k) {
        st.M[i][k] = lxu[i][k] + D.Hxu[i][k];
        st.Fu[i][k] = D.fu[i][k];
      }
      for (int k = 0; k < NX; ++k) st.Fx[i][k] = D.fx[i][k];
    }
    return;
  }
  R cx[NX], cu[NU], cxx[NX], cuu[NU];
  aug_derivs<R, NX, NU>(p, g, t, a.T, a.B, b, x, u, cx, cu, cxx, cuu);
  // (terms that are structurally zero are left out: a + 0 = a)
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int k = 0; k < NX; ++k) {
      R v = i == k ? R(p.Q[i * NX + k]) + cxx[i] : R(p.Q[i * NX + k]);
      st.P[i][k] = may_nz(HxxM, i * NX + k) ? v + D.Hxx[i][k] : v;
    }
  symmetrize<NX>(st.P);
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int k = 0; k < NU; ++k)
      st.Rr[i][k] = (R(p.Rc[i * NU + k]) + (i == k ? cuu[i] : R(0))) + D.Huu[i][k];
  symmetrize<NU>(st.Rr);
  R ftl[NU];
  mtv<NU, NX, R, FuM>(D.fu, ln, ftl);
#pragma unroll
  for (int i = 0; i < NU; ++i) {
    R ru = R(0);
#pragma unroll
    for (int k = 0; k < NU; ++k) ru += u[k] * R(p.Rc[i * NU + k]);
    st.d[i] = (ru + cu[i]) + ftl[i];
  }
  R fxl[NX];
  mtv<NX, NX, R, FxM>(D.fx, ln, fxl);
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    R lx = R(0);
#pragma unroll
    for (int k = 0; k < NX; ++k) lx += (x[k] - R(p.goal[k])) * R(p.Q[i * NX + k]);
    lt[i] = (lx + cx[i]) + fxl[i];
  }
#pragma unroll
  for (int i = 0; i < NX; ++i) {
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      st.M[i][k] = D.Hxu[i][k];
      st.Fu[i][k] = D.fu[i][k];
    }
#pragma unroll
    for (int k = 0; k < NX; ++k) st.Fx[i][k] = D.fx[i][k];
  }
}

// level-0 down-sweep fused with the Hamiltonian expansion (passes.py:155-185):
// with lambda_{t+1} in registers, evaluate every model derivative at
// (x_t, u_t) once and emit P, R, M, d, Fx, Fu and lambda_t.
// kExp: store the expansion (pass-level API, tree plans); without it only
// the co-states are stored and the fused value sweep re-derives the stage
// data in registers (the 2nx^2 + nu^2 + 2nx nu + nu words never touch HBM).
template <typename R, class Dyn, bool kExp = true>
__global__ void __launch_bounds__(128) k_costate_down0(NewtonArgs<R> a) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  const int P0 = a.plan.units0();
  const int u0 = unit_id();
  if (u0 >= P0 * a.B) return;
  const int b = u0 % a.B, j = u0 / a.B;
  if (!running(a, b) || !(a.phase[b] & PH_NEED_EXP)) return;
  const int q = a.parity[b];
  const int T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const ProblemParams& p = *a.pp;
  const AugArgs<R> g = aug_of(a);
  R ln[NX];
  if (j == P0 - 1) {
    R xT[NX];
    ld_x(a, q, T, b, xT);
    R PT[NX][NX];
    if constexpr (kUserCost<Dyn>) {
      Dyn::uterm_grad(p, xT, ln);
      Dyn::uterm_hess(p, xT, PT);
    } else {
      terminal_grad(p, xT, ln);
#pragma unroll
      for (int i = 0; i < NX; ++i)
#pragma unroll
        for (int k = 0; k < NX; ++k) PT[i][k] = R(p.Qf[i * NX + k]);
    }
    st_vec(a.lam, T, T + 1, B, b, ln);
    symmetrize<NX>(PT);
    st_mat(a.PT, 0, 1, B, b, PT);
  } else {
    ld_vec(a.ccar[1], j, a.plan.n[1], B, b, ln);
  }
  R x[NX], u[NU];
  ld_x(a, q, t1 - 1 >= t0 ? t1 - 1 : t0, b, x);
  ld_u(a, q, t1 - 1 >= t0 ? t1 - 1 : t0, b, u);
  for (int t = t1 - 1; t >= t0; --t) {
    // software pipeline: stage t-1's state and control load while stage t runs
    R xn[NX], un[NU];
    const int tp = t > t0 ? t - 1 : t;
    ld_x(a, q, tp, b, xn);
    ld_u(a, q, tp, b, un);
    R lt[NX];
    if constexpr (!kExp) {
      // co-states only: first derivatives suffice (bitwise the same lambda
      // as stage_expansion computes)
      DynDerivs<R, NX, NU> D;
      Dyn::template derivs<false>(p, t, b, x, u, ln, D);
      R cx[NX], cu[NU];
      if constexpr (kUserCon<Dyn>) {
        R Cxx[NX][NX], Cuu[NU][NU];
        aug_derivs_user<R, Dyn>(p, g, t, T, B, b, x, u, cx, cu, Cxx, Cuu);
      } else {
        R cxx[NX], cuu[NU];
        aug_derivs<R, NX, NU>(p, g, t, T, B, b, x, u, cx, cu, cxx, cuu);
      }
      R fxl[NX], ulx[NX];
      mtv<NX, NX>(D.fx, ln, fxl);
      if constexpr (kUserCost<Dyn>) Dyn::ucost_grad(p, t, x, u, ulx);
#pragma unroll
      for (int i = 0; i < NX; ++i) {
        R lx = R(0);
        if constexpr (kUserCost<Dyn>) {
          lx = ulx[i];
        } else {
#pragma unroll
          for (int k = 0; k < NX; ++k) lx += (x[k] - R(p.goal[k])) * R(p.Q[i * NX + k]);
        }
        lt[i] = (lx + cx[i]) + fxl[i];
      }
    } else {
      Stage<R, NX, NU> st;
      const R w0[kAuxDim<Dyn>] = {};
      stage_expansion<R, Dyn>(a, p, g, t, b, x, u, w0, false, ln, st, lt);
      st_mat(a.P, t, T, B, b, st.P);
      st_mat(a.Rm, t, T, B, b, st.Rr);
      st_mat(a.M, t, T, B, b, st.M);
      st_vec(a.d, t, T, B, b, st.d);
      st_mat(a.Fx, t, T, B, b, st.Fx);
      st_mat(a.Fu, t, T, B, b, st.Fu);
    }
    st_vec(a.lam, t, T + 1, B, b, lt);
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      ln[i] = lt[i];
      x[i] = xn[i];
    }
#pragma unroll
    for (int i = 0; i < NU; ++i) u[i] = un[i];
  }
}

// ----------------------------------------------- fused single-sweep LQR
// For single-sweep plans (one level-0 unit per problem: the large-batch
// schedule) the Newton iteration's value and propagation sweeps re-derive
// every stage's expansion from (x_t, u_t, lambda_{t+1}) in registers
// instead of reading the stored one: same functions, same bits, ~1/4 of
// the HBM traffic of the unfused iteration.

template <typename R, class Dyn>
__global__ void __launch_bounds__(128) k_value_fused(NewtonArgs<R> a, LqrArgs<R> la) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  const int b = unit_id();
  if (b >= a.B) return;
  if (!running(a, b)) return;
  const int q = a.parity[b];
  const int T = a.T, B = a.B;
  const ProblemParams& p = *a.pp;
  const AugArgs<R> g = aug_of(a);
  const R alpha = R(a.alpha[b]);
  // the co-state recursion runs inside this sweep: stage_expansion returns
  // lambda_t = l_x + f_x^T lambda_{t+1} (passes.py:122-148) next to the
  // stage's expansion, so the co-states never touch HBM.  Boundary:
  // lambda_T = terminal gradient, P_T = sym(Qf) (passes.py:140-148).
  VCarry<R, NX> c;
  int fl = 0;
  R ln[NX], x[NX], u[NU];
  {
    R xT[NX];
    ld_x(a, q, T, b, xT);
    if constexpr (kUserCost<Dyn>) {
      Dyn::uterm_grad(p, xT, ln);
      Dyn::uterm_hess(p, xT, c.Y);
    } else {
      terminal_grad(p, xT, ln);
#pragma unroll
      for (int i = 0; i < NX; ++i)
#pragma unroll
        for (int k = 0; k < NX; ++k) c.Y[i][k] = R(p.Qf[i * NX + k]);
    }
  }
  symmetrize<NX>(c.Y);
  set_zero(c.eta);
  // the trajectory's cached auxiliary values (sin / cos of the angle) when
  // the forward sweep that built it left them, else evaluated and cached
  constexpr int kA = AuxOf<Dyn>::n;
  const bool aux_on = kA > 0 && a.aux != nullptr;
  const bool have = aux_on && ((a.aux_ok[b] >> q) & 1);
  R* auxq = aux_on ? a.aux + q * a.auxsz : nullptr;
  R w[kAuxDim<Dyn>] = {};
  ld_x(a, q, T - 1, b, x);
  ld_u(a, q, T - 1, b, u);
  if (have) ld_vec(auxq, T - 1, T, B, b, w);
  for (int t = T - 1; t >= 0; --t) {
    // software pipeline: stage t-1's state and control are in flight while
    // stage t is expanded and folded
    R xn[NX], un[NU], wn[kAuxDim<Dyn>];
    const int tp = t > 0 ? t - 1 : 0;
    ld_x(a, q, tp, b, xn);
    ld_u(a, q, tp, b, un);
    if (have) ld_vec(auxq, tp, T, B, b, wn);
    if constexpr (kA > 0) {
      if (aux_on && !have) {
        Dyn::aux(x, w);
        st_vec(auxq, t, T, B, b, w);
      }
    }
    Stage<R, NX, NU> st;
    R lt[NX];
    stage_expansion<R, Dyn>(a, p, g, t, b, x, u, w, aux_on, ln, st, lt);
#pragma unroll
    for (int i = 0; i < NU; ++i) st.Rr[i][i] += alpha;
    R Gam[NU][NX], gam[NU];
    VCarry<R, NX> o;
    fl |= riccati_step<R, NX, NU, true, JacMask<Dyn>::fx, JacMask<Dyn>::fu>(st, c, Gam, gam, o);
    st_mat(la.Gam, t, T, B, b, Gam);
    st_vec(la.gam, t, T, B, b, gam);
    st_vec(a.d, t, T, B, b, st.d);
    c = o;
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      ln[i] = lt[i];
      x[i] = xn[i];
    }
#pragma unroll
    for (int i = 0; i < NU; ++i) u[i] = un[i];
    if (have) {
#pragma unroll
      for (int i = 0; i < kAuxDim<Dyn>; ++i) w[i] = wn[i];
    }
  }
  if (aux_on && !have) a.aux_ok[b] |= 1 << q;
  if (fl) atomicOr(a.flags + b, fl);
}

// --------------------------------------------------------------- rollout

enum : int { RS_SKIP = 1, RS_CONV = 2, RS_IN_XR = 4 };

// Which problems need the candidate rollout this iteration: k_control never
// looks at the candidate of a problem that is not running, whose subproblem
// failed (R/Q definiteness, singular combine) or whose step is below
// inner_tol (newton.py:166-181), so those skip it.
template <typename R>
__global__ void k_roll_gate(NewtonArgs<R> a) {
  const int b = unit_id();
  if (b >= a.B) return;
  int st = 0;
  if (!running(a, b) || (a.flags[b] & (FLAG_DEF_R | FLAG_DEF_Q | FLAG_COND))) {
    st = RS_SKIP;
  } else {
    const int P0 = a.plan.units0();
    double step = 0.0;
    for (int j = 0; j < partial_rows(P0); ++j) step = nanmax(step, a.red[((size_t)2 * P0 + j) * a.B + b]);
    if (step <= a.opt.inner_tol) st = RS_SKIP;
  }
  a.rstate[b] = st;
}

// candidate u + du rolled through the nonlinear dynamics (problem.py:449-473)
// -- sequential in time, parallel over the batch; controls are prefetched
// kRing steps ahead so the recurrence runs at the dynamics' latency, not
// the memory's.  With kFromUc the candidate controls are already in place.
// kCost: also accumulate the candidate's stage and augmentation costs (the
// partials k_cost_partials(a, 1) would produce, single-unit plans only), so
// the candidate trajectory is not read back a second time.
template <typename R, class Dyn, bool kFromUc, bool kCost = false>
__global__ void __launch_bounds__(128) k_rollout(NewtonArgs<R> a, const R* dU) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  constexpr int kRing = 8;
  const int b = unit_id();
  if (b >= a.B) return;
  if (a.rstate[b] & (RS_SKIP | RS_CONV)) return;
  const int q = a.parity[b], c = 1 - q;
  const int T = a.T, B = a.B;
  // the model constants in registers: loop-invariant divisions hoist out of
  // the recurrence (the parameters live in global memory, which the stores
  // below could alias as far as the compiler knows)
  ProblemParams p;
  const ProblemParams& gp = *a.pp;
  p.dyn_kind = gp.dyn_kind;
#pragma unroll
  for (int i = 0; i < 8; ++i) p.dyn[i] = gp.dyn[i];
  p.lin_T = gp.lin_T;
  p.lin_B = gp.lin_B;
  p.lin_A = gp.lin_A;
  p.lin_Bm = gp.lin_Bm;
  p.lin_c = gp.lin_c;
  p.lin_st = gp.lin_st;
  p.user_data = gp.user_data;
  R* Xc = a.X + c * a.xsz;
  R* Uc = a.U + c * a.usz;
  R x[NX];
  ld_x(a, q, 0, b, x);
  st_vec(Xc, 0, T + 1, B, b, x);
  bool finite = true;
  double sl = 0.0, sc = 0.0;
  int bad = -1;
  const AugArgs<R> g = aug_of(a);
  CostRegs<R, NX, NU> cr;
  if constexpr (kCost && NX < 8) cr.load(gp);
  R ring[kRing][NU];
  auto fetch = [&](int t, R (&u)[NU]) {
    if (t < T) {
      if (kFromUc) {
        ld_vec(Uc, t, T, B, b, u);
      } else {
        R du[NU];
        ld_u(a, q, t, b, u);
        ld_vec(dU, t, T, B, b, du);
#pragma unroll
        for (int i = 0; i < NU; ++i) u[i] += du[i];
      }
    }
  };
#pragma unroll
  for (int k = 0; k < kRing; ++k) fetch(k, ring[k]);
  for (int t0 = 0; t0 < T; t0 += kRing) {
#pragma unroll
    for (int k = 0; k < kRing; ++k) {
      const int t = t0 + k;
      if (t < T) {
        R u[NU];
#pragma unroll
        for (int i = 0; i < NU; ++i) u[i] = ring[k][i];
        fetch(t + kRing, ring[k]);
        if (!kFromUc) st_vec(Uc, t, T, B, b, u);
        if constexpr (kCost) {
          if constexpr (kUserCost<Dyn>) sl += double(Dyn::ucost(gp, t, x, u));
          else if constexpr (NX < 8) sl += double(stage_cost<R, NX, NU>(cr, x, u));
          else sl += double(stage_cost<R, NX, NU>(gp, x, u));
          int br;
          if constexpr (kUserCon<Dyn>) sc += double(aug_value_user<R, Dyn>(gp, g, t, T, B, b, x, u, br));
          else sc += double(aug_value<R, NX, NU>(gp, g, t, T, B, b, x, u, br));
          if (br >= 0 && bad < 0) bad = t * gp.W + br;
        }
        R xn[NX];
        Dyn::step(p, t, b, x, u, xn);
#pragma unroll
        for (int i = 0; i < NX; ++i) {
          finite = finite && isfinite(xn[i]);
          x[i] = xn[i];
        }
        st_vec(Xc, t + 1, T + 1, B, b, x);
      }
    }
  }
  if (!finite) atomicOr(a.flags + b, FLAG_DIVERGED);
  if constexpr (kCost) {
    if constexpr (kUserCost<Dyn>) sl += double(Dyn::uterm(gp, x));   // x = x_T
    double* cp = a.cpart[1];  // P0 == 1
    cp[(size_t)0 * B + b] = sl;
    cp[(size_t)1 * B + b] = sc;
    cp[(size_t)2 * B + b] = double(bad);
  }
}

// ------------------------------------ fused forward sweep (single-sweep plans)
//
// The propagation sweep (passes.py:330-361, Jacobians re-derived from x, u
// like k_value_fused) and the candidate rollout (k_rollout) both walk the
// horizon forwards, one thread per problem, and both are
// latency-bound chains (the 4x4 closed-loop recurrence; the model's step).
// Here one thread runs them side by side, stage by stage: du_t is formed
// from the deviation recurrence and at once added to u_t to drive the
// candidate's step, so the two independent chains fill each other's latency
// and du, dx never touch HBM.  newton.py:190-197 rolls out only when the
// step norm exceeds inner_tol; the thread knows its norm only at the end, so
// the candidate is built speculatively and its outcome (divergence flag)
// is kept only when the gate passes -- k_control never reads the candidate
// of a gated problem (same decisions and bits as prop + gate + rollout).
// kCost: the candidate's stage / augmentation costs accumulate in the same
// sweep (otherwise k_cost_partials(a, 1) runs after).
template <typename R, class Dyn, bool kCost>
__global__ void __launch_bounds__(128) k_forward_fused(NewtonArgs<R> a, LqrArgs<R> la) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  const int b = unit_id();
  if (b >= a.B) return;
  if (!running(a, b)) return;
  if (a.flags[b] & (FLAG_DEF_R | FLAG_DEF_Q | FLAG_COND)) {
    a.rstate[b] = RS_SKIP;  // no law: k_control escalates alpha
    return;
  }
  const int q = a.parity[b], c = 1 - q;
  const int T = a.T, B = a.B;
  ProblemParams p;   // model constants in registers (see k_rollout)
  const ProblemParams& gp = *a.pp;
  p.dyn_kind = gp.dyn_kind;
#pragma unroll
  for (int i = 0; i < 8; ++i) p.dyn[i] = gp.dyn[i];
  p.lin_T = gp.lin_T;
  p.lin_B = gp.lin_B;
  p.lin_A = gp.lin_A;
  p.lin_Bm = gp.lin_Bm;
  p.lin_c = gp.lin_c;
  p.lin_st = gp.lin_st;
  p.user_data = gp.user_data;
  R* Xc = a.X + c * a.xsz;
  R* Uc = a.U + c * a.usz;
  const AugArgs<R> g = aug_of(a);
  CostRegs<R, NX, NU> cr;
  if constexpr (kCost && NX < 8) cr.load(gp);
  R x[NX], xc[NX], lam0[NX];
  set_zero(x);
  set_zero(lam0);
  double s2 = 0.0, sd = 0.0, mx = 0.0, sl = 0.0, sc = 0.0;
  int bad = -1;
  bool finite = true;
  // cached auxiliary values: the current trajectory's (left by the value
  // sweep) feed its Jacobians; the candidate's, evaluated for its steps,
  // are cached next to it
  constexpr int kA = AuxOf<Dyn>::n;
  const bool aux_on = kA > 0 && a.aux != nullptr;
  const bool have = aux_on && ((a.aux_ok[b] >> q) & 1);
  const R* auxq = aux_on ? a.aux + q * a.auxsz : nullptr;
  R* auxc = aux_on ? a.aux + c * a.auxsz : nullptr;
  R xs[NX], us[NU], Gam[NU][NX], gam[NU], dd[NU], ws[kAuxDim<Dyn>] = {};
  ld_x(a, q, 0, b, xs);
  ld_u(a, q, 0, b, us);
  ld_mat(la.Gam, 0, T, B, b, Gam);
  ld_vec(la.gam, 0, T, B, b, gam);
  ld_vec(a.d, 0, T, B, b, dd);
  if (have) ld_vec(auxq, 0, T, B, b, ws);
#pragma unroll
  for (int i = 0; i < NX; ++i) xc[i] = xs[i];
  st_vec(Xc, 0, T + 1, B, b, xc);
  for (int t = 0; t < T; ++t) {
    // software pipeline: stage t+1's inputs load while stage t runs
    R xs_n[NX], us_n[NU], Gam_n[NU][NX], gam_n[NU], dd_n[NU], ws_n[kAuxDim<Dyn>];
    const int tn = t + 1 < T ? t + 1 : t;
    ld_x(a, q, tn, b, xs_n);
    ld_u(a, q, tn, b, us_n);
    ld_mat(la.Gam, tn, T, B, b, Gam_n);
    ld_vec(la.gam, tn, T, B, b, gam_n);
    ld_vec(a.d, tn, T, B, b, dd_n);
    if (have) ld_vec(auxq, tn, T, B, b, ws_n);
    R du[NU], uc[NU];
    mv<NU, NX>(Gam, x, du);
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      du[i] += gam[i];
      s2 += double(du[i]) * double(du[i]);
      sd += double(du[i]) * double(dd[i]);
      mx = nanmax(mx, double(fabs(du[i])));
      uc[i] = us[i] + du[i];   // the candidate control u + du (problem.py:449)
    }
    st_vec(Uc, t, T, B, b, uc);
    // candidate chain: stage cost at (xc_t, uc_t), then xc_{t+1} = f(xc_t, uc_t)
    if constexpr (kCost) {
      if constexpr (kUserCost<Dyn>) sl += double(Dyn::ucost(gp, t, xc, uc));
      else if constexpr (NX < 8) sl += double(stage_cost<R, NX, NU>(cr, xc, uc));
      else sl += double(stage_cost<R, NX, NU>(gp, xc, uc));
      int br;
      if constexpr (kUserCon<Dyn>) sc += double(aug_value_user<R, Dyn>(gp, g, t, T, B, b, xc, uc, br));
      else sc += double(aug_value<R, NX, NU>(gp, g, t, T, B, b, xc, uc, br));
      if (br >= 0 && bad < 0) bad = t * gp.W + br;
    }
    R xcn[NX];
    if constexpr (kA > 0) {
      if (aux_on) {
        R wc[kAuxDim<Dyn>];
        Dyn::aux(xc, wc);
        st_vec(auxc, t, T, B, b, wc);
        Dyn::step_w(p, t, b, xc, uc, wc, xcn);
      } else {
        Dyn::step(p, t, b, xc, uc, xcn);
      }
    } else {
      Dyn::step(p, t, b, xc, uc, xcn);
    }
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      finite = finite && isfinite(xcn[i]);
      xc[i] = xcn[i];
    }
    st_vec(Xc, t + 1, T + 1, B, b, xc);
    // deviation chain: dx_{t+1} = (fx + fu Gamma) dx_t + fu gamma at the
    // current trajectory
    DynDerivs<R, NX, NU> D;
    dyn_derivs<false, Dyn>(p, t, b, xs, us, ws, have, lam0, D);
    constexpr uint64_t FxM = JacMask<Dyn>::fx, FuM = JacMask<Dyn>::fu;
    constexpr uint64_t FM = plus_rows_mask<NX, NX, NU>(FxM, FuM);
    R F[NX][NX], e[NX], y[NX];
    mm<NX, NU, NX, R, kDense, FuM>(D.fu, Gam, F);
#pragma unroll
    for (int i = 0; i < NX; ++i)
#pragma unroll
      for (int k = 0; k < NX; ++k) {
        const bool fu_row = may_nz(plus_rows_mask<NX, NX, NU>(0, FuM), i * NX + k);
        const R v = !fu_row ? D.fx[i][k] : (may_nz(FxM, i * NX + k) ? F[i][k] + D.fx[i][k] : F[i][k]);
        F[i][k] = (t == 0) ? R(0) : v;
      }
    mv<NX, NU, R, FuM>(D.fu, gam, e);
    mv<NX, NX, R, FM>(F, x, y);
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      x[i] = y[i] + e[i];
      xs[i] = xs_n[i];
    }
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      us[i] = us_n[i];
      gam[i] = gam_n[i];
      dd[i] = dd_n[i];
#pragma unroll
      for (int k = 0; k < NX; ++k) Gam[i][k] = Gam_n[i][k];
    }
    if (have) {
#pragma unroll
      for (int i = 0; i < kAuxDim<Dyn>; ++i) ws[i] = ws_n[i];
    }
  }
  if (aux_on) a.aux_ok[b] |= 1 << c;
  la.red[(size_t)0 * B + b] = s2;
  la.red[(size_t)1 * B + b] = sd;
  la.red[(size_t)2 * B + b] = mx;
  // the rollout gate of newton.py:181 (k_roll_gate): only a step above
  // inner_tol is rolled out, so only then does the candidate's outcome count
  const bool gated = mx <= a.opt.inner_tol;
  a.rstate[b] = gated ? RS_SKIP : 0;
  if (!gated && !finite) atomicOr(a.flags + b, FLAG_DIVERGED);
  if constexpr (kCost) {
    if constexpr (kUserCost<Dyn>) sl += double(Dyn::uterm(gp, xc));   // xc = x_T
    double* cp = a.cpart[1];  // P0 == 1
    cp[(size_t)0 * B + b] = sl;
    cp[(size_t)1 * B + b] = sc;
    cp[(size_t)2 * B + b] = double(bad);
  }
}

// ------------------------------------------------ parallel (log-depth) rollout
//
// For small batches with long horizons the rollout is solved as a nonlinear
// system  x_{t+1} = f_t(x_t, u_t)  by Newton's method on the whole
// trajectory: linearised at a guess x^k, the recurrence becomes the affine
// scan  x_{t+1} = f(x^k_t) + Fx(x^k_t) (x_t - x^k_t),  solved with the same
// blocked tree as the other scans.  The first guess x + dx is the LQR
// propagation pass's prediction (itself the first Newton iterate from the
// dynamically consistent current trajectory), so convergence is quadratic
// from the start; a problem stops as soon as every step of its guess
// satisfies the recurrence to 1e-13 relative (fp64; fp32 1e-5).  A problem that has not converged
// after pr_iters sweeps (or meets a non-finite state) is rolled out by the
// sequential kernel, so the result and the divergence report never depend
// on the parallel path's convergence.

template <typename R>
PTC_D R* pr_buf(const NewtonArgs<R>& a, int b, int which) {
  // which 0: the candidate buffer (1 - parity), 1: xr
  return which == 0 ? a.X + (1 - a.parity[b]) * a.xsz : a.xr;
}

template <typename R, int NX, int NU>
__global__ void k_pr_init(NewtonArgs<R> a, const R* dX, const R* dU) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)(a.T + 1) * a.B) return;
  const int b = (int)(i % a.B), t = (int)(i / a.B);
  if (a.rstate[b] & RS_SKIP) return;
  const int q = a.parity[b];
  R x[NX], d[NX];
  ld_x(a, q, t, b, x);
  ld_vec(dX, t, a.T + 1, a.B, b, d);
#pragma unroll
  for (int k = 0; k < NX; ++k) x[k] += d[k];
  st_vec(pr_buf(a, b, 0), t, a.T + 1, a.B, b, x);
  if (t < a.T) {
    R u[NU], du[NU];
    ld_u(a, q, t, b, u);
    ld_vec(dU, t, a.T, a.B, b, du);
#pragma unroll
    for (int k = 0; k < NU; ++k) u[k] += du[k];
    st_vec(a.U + (1 - q) * a.usz, t, a.T, a.B, b, u);
  }
}

// level-0: affine elements of the linearised recurrence folded over a chunk,
// and the residual of the current guess
template <typename R, class Dyn>
__global__ void __launch_bounds__(128) k_pr_up0(NewtonArgs<R> a, int k) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  const int P0 = a.plan.units0();
  const int u0 = unit_id();
  if (u0 >= P0 * a.B) return;
  const int b = u0 % a.B, j = u0 / a.B;
  if (a.rstate[b] & (RS_SKIP | RS_CONV)) return;
  const int T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const ProblemParams& p = *a.pp;
  const R* g = pr_buf(a, b, k & 1);
  const R* Uc = a.U + (1 - a.parity[b]) * a.usz;
  Aff<R, NX> acc;
  aff_identity(acc);
  double res = 0.0;
  R lam0[NX];
  set_zero(lam0);
  for (int t = t0; t < t1; ++t) {
    R x[NX], u[NU], xn[NX], fn[NX];
    ld_vec(g, t, T + 1, B, b, x);
    ld_vec(Uc, t, T, B, b, u);
    ld_vec(g, t + 1, T + 1, B, b, xn);
    Dyn::step(p, t, b, x, u, fn);
    DynDerivs<R, NX, NU> D;
    Dyn::template derivs<false>(p, t, b, x, u, lam0, D);
    double mag = 1.0, gap = 0.0;
    Aff<R, NX> m, o;
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      gap = nanmax(gap, double(fabs(xn[i] - fn[i])));
      mag = nanmax(mag, double(fabs(fn[i])));
      R fxx = R(0);
#pragma unroll
      for (int c = 0; c < NX; ++c) {
        m.F[i][c] = D.fx[i][c];
        fxx = fma(D.fx[i][c], x[c], fxx);
      }
      m.e[i] = fn[i] - fxx;
    }
    res = nanmax(res, gap / mag);
    if (!(gap == gap) || !(mag == mag)) res = INFINITY;
    aff_compose(m, acc, o);
    acc = o;
  }
  if (a.plan.L >= 1) st_aff(a.cagg[1], j, a.plan.n[1], B, b, acc);
  a.rres[(size_t)j * B + b] = res;
}

template <typename R>
__global__ void k_pr_check(NewtonArgs<R> a, int k) {
  const int b = unit_id();
  if (b >= a.B) return;
  int st = a.rstate[b];
  if (st & (RS_SKIP | RS_CONV)) return;
  const int P0 = a.plan.units0();
  double r = 0.0;
  for (int j = 0; j < partial_rows(P0); ++j) r = nanmax(r, a.rres[(size_t)j * a.B + b]);
  // per-step consistency |x_{t+1} - f(x_t, u_t)| / max(1, |f|): the scan's
  // own rounding (tree carries compose many steps) sits at a few hundred
  // ulp for long horizons, so fp64 accepts 1e-13 (fp32 1e-5)
  const double tol = sizeof(R) == 8 ? 1e-13 : 1e-5;
  if (r <= tol) a.rstate[b] = st | RS_CONV | ((k & 1) ? RS_IN_XR : 0);
}

template <typename R, int NX>
__global__ void __launch_bounds__(128) k_pr_up(NewtonArgs<R> a, int l) {
  const int nl = a.plan.n[l], nn = a.plan.n[l + 1];
  const int u0 = unit_id();
  if (u0 >= nn * a.B) return;
  const int b = u0 % a.B, j = u0 / a.B;
  if (a.rstate[b] & (RS_SKIP | RS_CONV)) return;
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  Aff<R, NX> acc;
  ld_aff(a.cagg[l], first, nl, a.B, b, acc);
  for (int i = first + 1; i <= last; ++i) {
    Aff<R, NX> m, o;
    ld_aff(a.cagg[l], i, nl, a.B, b, m);
    aff_compose(m, acc, o);
    acc = o;
  }
  st_aff(a.cagg[l + 1], j, nn, a.B, b, acc);
}

template <typename R, int NX>
__global__ void __launch_bounds__(128) k_pr_top(NewtonArgs<R> a, int k) {
  const int b = unit_id();
  if (b >= a.B) return;
  if (a.rstate[b] & (RS_SKIP | RS_CONV)) return;
  const int L = a.plan.L, nL = a.plan.n[L];
  R x[NX];
  ld_vec(pr_buf(a, b, k & 1), 0, a.T + 1, a.B, b, x);  // x_0, identical in both buffers
  for (int i = 0; i < nL; ++i) {
    st_vec(a.ccar[L], i, nL, a.B, b, x);
    Aff<R, NX> m;
    ld_aff(a.cagg[L], i, nL, a.B, b, m);
    R y[NX];
    aff_apply(m, x, y);
#pragma unroll
    for (int c = 0; c < NX; ++c) x[c] = y[c];
  }
}

template <typename R, int NX>
__global__ void __launch_bounds__(128) k_pr_down(NewtonArgs<R> a, int l) {
  const int nl = a.plan.n[l], nn = a.plan.n[l + 1];
  const int u0 = unit_id();
  if (u0 >= nn * a.B) return;
  const int b = u0 % a.B, j = u0 / a.B;
  if (a.rstate[b] & (RS_SKIP | RS_CONV)) return;
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  R x[NX];
  ld_vec(a.ccar[l + 1], j, nn, a.B, b, x);
  for (int i = first; i <= last; ++i) {
    st_vec(a.ccar[l], i, nl, a.B, b, x);
    Aff<R, NX> m;
    ld_aff(a.cagg[l], i, nl, a.B, b, m);
    R y[NX];
    aff_apply(m, x, y);
#pragma unroll
    for (int c = 0; c < NX; ++c) x[c] = y[c];
  }
}

// level-0 forward sweep: the next guess x^{k+1} from the chunk's carry
template <typename R, class Dyn>
__global__ void __launch_bounds__(128) k_pr_down0(NewtonArgs<R> a, int k) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  const int P0 = a.plan.units0();
  const int u0 = unit_id();
  if (u0 >= P0 * a.B) return;
  const int b = u0 % a.B, j = u0 / a.B;
  if (a.rstate[b] & (RS_SKIP | RS_CONV)) return;
  const int T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const ProblemParams& p = *a.pp;
  const R* g = pr_buf(a, b, k & 1);
  R* n = pr_buf(a, b, (k + 1) & 1);
  const R* Uc = a.U + (1 - a.parity[b]) * a.usz;
  R x[NX];
  if (j == 0) {
    ld_vec(g, 0, T + 1, B, b, x);
    st_vec(n, 0, T + 1, B, b, x);
  } else {
    ld_vec(a.ccar[1], j, a.plan.n[1], B, b, x);
  }
  R lam0[NX];
  set_zero(lam0);
  for (int t = t0; t < t1; ++t) {
    R xg[NX], u[NU], fn[NX];
    ld_vec(g, t, T + 1, B, b, xg);
    ld_vec(Uc, t, T, B, b, u);
    Dyn::step(p, t, b, xg, u, fn);
    DynDerivs<R, NX, NU> D;
    Dyn::template derivs<false>(p, t, b, xg, u, lam0, D);
    R dxv[NX], y[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) dxv[i] = x[i] - xg[i];
    mv<NX, NX>(D.fx, dxv, y);
#pragma unroll
    for (int i = 0; i < NX; ++i) x[i] = fn[i] + y[i];
    st_vec(n, t + 1, T + 1, B, b, x);
  }
}

// a converged guess left in xr moves to the candidate buffer
template <typename R, int NX>
__global__ void k_pr_finish(NewtonArgs<R> a) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)(a.T + 1) * a.B) return;
  const int b = (int)(i % a.B), t = (int)(i / a.B);
  if ((a.rstate[b] & (RS_SKIP | RS_CONV | RS_IN_XR)) != (RS_CONV | RS_IN_XR)) return;
  R x[NX];
  ld_vec(a.xr, t, a.T + 1, a.B, b, x);
  st_vec(a.X + (1 - a.parity[b]) * a.xsz, t, a.T + 1, a.B, b, x);
}

// ------------------------------------------------------- trust-region control

template <typename R>
PTC_D void record(const NewtonArgs<R>& a, int b, double cost, double alpha, double ratio,
                  double step, double acc) {
  const int k = a.hist_len[b];
  if (k < a.opt.hist_cap) {
    double* h = a.hist + (size_t)k * 5 * a.B + b;
    h[0 * a.B] = cost;
    h[1 * a.B] = alpha;
    h[2 * a.B] = ratio;
    h[3 * a.B] = step;
    h[4 * a.B] = acc;
  }
  a.hist_len[b] = k + 1;
}

template <typename R, int NX>
PTC_D double finalize_cost(const NewtonArgs<R>& a, int which, int q, int b, int& bad) {
  const int P0 = a.plan.units0();
  const double* cp = a.cpart[which];
  double sl = 0.0, sc = 0.0;
  bad = -1;
  for (int j = 0; j < partial_rows(P0); ++j) {
    sl += cp[((size_t)0 * P0 + j) * a.B + b];
    sc += cp[((size_t)1 * P0 + j) * a.B + b];
    int bj = int(cp[((size_t)2 * P0 + j) * a.B + b]);
    if (bad < 0 && bj >= 0) bad = bj;
  }
  // block mode / user cost: the terminal cost is in the (reduced) partials
  if (a.blk || a.uterm) return sl + sc;
  R xT[NX];
  ld_x(a, q, a.T, b, xT);
  double term = double(terminal_cost(*a.pp, xT));
  return term + (sl + sc);
}

// Constraint value w at the flat index stage * W + row of buffer q: the
// `value` the reference's InfeasibleError carries (outer.py:47-52).
template <typename R, int NX, int NU>
PTC_D double infeasible_value(const NewtonArgs<R>& a, int q, int b, int bad) {
  const int W = a.pp->W > 0 ? a.pp->W : 1;
  const int t = bad / W - a.t_base, k = bad % W;
  if (t < 0 || t >= a.T) return NAN;
  R x[NX], u[NU];
  ld_x(a, q, t, b, x);
  ld_u(a, q, t, b, u);
  return double(row_value<R, NX, NU>(*a.pp, k, x, u));
}

// User constraints: the InfeasibleError value k_control could not evaluate
// (its row tables describe boxes only) from the model's own rows.
template <typename R, class Dyn>
__global__ void k_user_bad_value(NewtonArgs<R> a) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU, W = Dyn::kWs + Dyn::kWc;
  const int b = unit_id();
  if (b >= a.B) return;
  const int bad = a.bad_index[b];
  if (bad < 0 || W == 0) return;
  const int t = bad / W, k = bad % W;
  if (t >= a.T) return;
  R x[NX], u[NU], w[W > 0 ? W : 1];
  ld_x(a, a.parity[b], t, b, x);
  ld_u(a, a.parity[b], t, b, u);
  Dyn::ucon_w(*a.pp, t, x, u, w);
  a.bad_value[b] = double(w[k]);
}

// One step of newton.py:157-208 for every running problem.
template <typename R, int NX, int NU>
__global__ void k_control(NewtonArgs<R> a) {
  const int b = unit_id();
  if (b >= a.B) return;
  if (!running(a, b)) return;
  int ph = a.phase[b];
  const bool barrier = a.aug_kind == AUG_BARRIER;
  double cur = a.cur_cost[b];
  if (ph & PH_NEED_COST) {
    int bad;
    cur = finalize_cost<R, NX>(a, 0, a.parity[b], b, bad);
    if (barrier && bad >= 0) {
      a.status[b] = ST_ERR_INFEASIBLE;
      a.bad_index[b] = bad;
      a.bad_value[b] = infeasible_value<R, NX, NU>(a, a.parity[b], b, bad);
      return;
    }
    ph &= ~PH_NEED_COST;
  }
  ph &= ~PH_NEED_EXP;  // consumed by this iteration's co-state pass
  double alpha = a.alpha[b], nu = a.nu[b];
  const int fl = a.flags[b];
  a.flags[b] = 0;
  int it = a.iters[b];
  bool finished = false;
  int term = TERM_NONE;
  const double tol = a.opt.inner_tol;
  if (fl & (FLAG_DEF_R | FLAG_DEF_Q | FLAG_COND)) {
    if (alpha > kAlphaMax) {
      a.status[b] = ST_ERR_STALLED;
      a.alpha[b] = alpha;
      a.phase[b] = ph;
      a.cur_cost[b] = cur;
      return;
    }
    record(a, b, cur, alpha, -INFINITY, NAN, 0.0);
    alpha = alpha > 0.0 ? alpha * nu : 1e-6;
    nu = 2.0 * nu;
    ++it;
  } else {
    const int P0 = a.plan.units0();
    double s2 = 0.0, sd = 0.0, step = 0.0;
    for (int j = 0; j < partial_rows(P0); ++j) {
      s2 += a.red[((size_t)0 * P0 + j) * a.B + b];
      sd += a.red[((size_t)1 * P0 + j) * a.B + b];
      step = nanmax(step, a.red[((size_t)2 * P0 + j) * a.B + b]);
    }
    if (step <= tol) {
      record(a, b, cur, alpha, NAN, step, 0.0);
      ++it;
      finished = true;
      term = TERM_STEP;
    } else {
      const double pred = 0.5 * (alpha * s2 - sd);
      int bad;
      const double cand = finalize_cost<R, NX>(a, 1, 1 - a.parity[b], b, bad);
      double ratio;
      double newc = INFINITY;
      if ((fl & FLAG_DIVERGED) || (barrier && bad >= 0)) {
        ratio = -INFINITY;
      } else {
        newc = cand;
        ratio = (pred <= 0.0) ? -INFINITY : (cur - newc) / pred;
      }
      a.cand_cost[b] = newc;   // the candidate's cost (readable: "cand_cost")
      const double used = alpha;
      // fp32 solver only: a model decrease below the float32 resolution of
      // the cost (2^-20 |cost|, 16 ulps) cannot be judged by the gain ratio
      // -- both costs carry that much rounding from the fp32 rollouts -- so
      // a feasible candidate is accepted and ends the solve as converged
      // (the relative cost change it makes is below fp32 resolution too).
      // The fp64 solver never takes this branch: it follows newton.py.
      const bool below32 = sizeof(R) == 4 && pred > 0.0 && newc < INFINITY &&
                           pred <= 0x1p-20 * fabs(cur);
      if (ratio > 0.0 || below32) {
        const double f = 1.0 - pow(2.0 * ratio - 1.0, 3.0);
        alpha = alpha * (f > 1.0 / 3.0 ? f : 1.0 / 3.0);
        nu = 2.0;
        const double rel = fabs(cur - newc) / fmax(1.0, fabs(cur));
        record(a, b, newc, used, ratio, step, 1.0);
        a.parity[b] ^= 1;
        cur = newc;
        ph |= PH_NEED_EXP;
        ++it;
        if (rel <= tol || below32) {
          finished = true;
          term = TERM_COST;
        }
      } else {
        alpha = alpha * nu;
        nu = 2.0 * nu;
        record(a, b, cur, used, ratio, step, 0.0);
        ++it;
        if (alpha > kAlphaMax) {
          finished = true;
          term = TERM_STALLED;
        }
      }
    }
  }
  if (!finished && it >= a.opt.max_iters) {
    finished = true;
    term = TERM_MAX_ITERS;
  }
  if (finished) {
    ph |= PH_ROUND_DONE;
    a.term[b] = term;
  }
  a.iters[b] = it;
  a.alpha[b] = alpha;
  a.nu[b] = nu;
  a.cur_cost[b] = cur;
  a.phase[b] = ph;
}

// --------------------------------------------------------------- outer loops

// per-stage work at the end of a Newton round: copy the round's controls
// (barrier report) or run the ADMM consensus/dual update with residual maxima
template <typename R, int NX, int NU, class Dyn = void>
__global__ void __launch_bounds__(128) k_round_end(NewtonArgs<R> a) {
  const int P0 = a.plan.units0();
  const int u0 = unit_id();
  if (u0 >= P0 * a.B) return;
  const int b = u0 % a.B, j = u0 / a.B;
  if (!running(a, b) || !(a.phase[b] & PH_ROUND_DONE)) return;
  const int T = a.T, B = a.B, q = a.parity[b];
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  if (a.opt.method == METHOD_BARRIER) {
    const int r = a.round[b];
    if (a.round_U && r < a.opt.round_cap) {
      R* dst = a.round_U + (size_t)r * NU * T * B;
      for (int t = t0; t < t1; ++t) {
        R u[NU];
        ld_u(a, q, t, b, u);
        st_vec(dst, t, T, B, b, u);
      }
    }
    return;
  }
  if (a.opt.method != METHOD_ADMM) return;
  const ProblemParams& p = *a.pp;
  const R rho = R(a.opt.rho);
  double rp = 0.0, rd = 0.0;
  for (int t = t0; t < t1; ++t) {
    R x[NX], u[NU];
    ld_x(a, q, t, b, x);
    ld_u(a, q, t, b, u);
    R wu[kMaxRows];
    if constexpr (!std::is_void_v<Dyn> && kUserCon<Dyn>) {
      constexpr int W = Dyn::kWs + Dyn::kWc;
      R w_[W > 0 ? W : 1];
      Dyn::ucon_w(p, t, x, u, w_);
      for (int k = 0; k < W; ++k) wu[k] = w_[k];
    }
    for (int k = 0; k < p.W; ++k) {
      R w;
      if constexpr (!std::is_void_v<Dyn> && kUserCon<Dyn>) w = wu[k];
      else w = row_value<R, NX, NU>(p, k, x, u);
      R zp = ldf(a.z, k, t, T, B, b);
      R vv = ldf(a.v, k, t, T, B, b);
      R zs = w + vv / rho;
      R zn = zs < R(0) ? zs : R(0);
      if (zs != zs) zn = zs;
      R vn = vv + rho * (w - zn);
      stf(a.z, k, t, T, B, b, zn);
      stf(a.v, k, t, T, B, b, vn);
      rp = nanmax(rp, double(fabs(w - zn)));
      rd = nanmax(rd, double(fabs(zn - zp)));
    }
  }
  a.apart[((size_t)0 * P0 + j) * B + b] = rp;
  a.apart[((size_t)1 * P0 + j) * B + b] = rd;
}

template <typename R>
__global__ void k_outer(NewtonArgs<R> a) {
  const int b = unit_id();
  if (b >= a.B) return;
  if (running(a, b) && (a.phase[b] & PH_ROUND_DONE)) {
    const int r = a.round[b];
    const int m = a.opt.method;
    if (r < a.opt.round_cap) {
      const size_t o = (size_t)r * a.B + b;
      a.round_mu[o] = a.mu[b];
      a.round_cost[o] = a.cur_cost[b];
      a.round_iters[o] = a.iters[b];
      a.round_term[o] = a.term[b];
      a.round_rp[o] = 0.0;
      a.round_rd[o] = 0.0;
    }
    a.round[b] = r + 1;
    bool again = false;
    if (m == METHOD_BARRIER) {
      const double mu = a.mu[b] * a.opt.zeta;
      a.mu[b] = mu;
      again = mu > a.opt.mu_tol;
    } else if (m == METHOD_ADMM) {
      const int P0 = a.plan.units0();
      double rp = 0.0, rd = 0.0;
      for (int j = 0; j < partial_rows(P0); ++j) {
        rp = nanmax(rp, a.apart[((size_t)0 * P0 + j) * a.B + b]);
        rd = nanmax(rd, a.apart[((size_t)1 * P0 + j) * a.B + b]);
      }
      if (r < a.opt.round_cap) {
        a.round_rp[(size_t)r * a.B + b] = rp;
        a.round_rd[(size_t)r * a.B + b] = rd;
      }
      const bool conv = rp <= a.opt.residual_tol && rd <= a.opt.residual_tol;
      again = !conv && (r + 1) < a.opt.max_outer;
    }
    if (again) {
      a.alpha[b] = a.opt.alpha0;
      a.nu[b] = a.opt.nu0;
      a.iters[b] = 0;
      a.phase[b] = PH_NEED_COST | PH_NEED_EXP;
    } else {
      a.status[b] = ST_DONE;
      a.phase[b] &= ~PH_ROUND_DONE;
    }
  }
  if (running(a, b)) atomicAdd(a.n_running, 1);
}

}  // namespace ptc
