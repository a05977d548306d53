// Warp-cooperative Newton kernels for wide affine models (nx >= 8).
//
// The thread-per-unit co-state / expansion / rollout kernels of
// newton_kernels.cuh hold an nx x nx affine map per thread; at nx = 12 the
// co-state aggregates (156 words) spill and one 12x12x12 composition is a
// serial chain of 1,728 FMAs per stage.  As for the LQR scans (wide.cuh),
// one WARP owns one scan unit here: stage data is gathered into a per-warp
// shared-memory slab with the next stage's loads already in flight
// (WGather), lanes split every product over output entries, and the
// compositions run on the DMMA path of w_mm.  Kernels:
//
//   kwn_costate_up0 / kwn_tree_* / kwn_costate_down0   co-state scan + the
//       fused Hamiltonian expansion (passes.py:122-185) for affine dynamics
//       (fx = A_t, fu = B_t, no second-order dynamics terms)
//   kwn_roll_up0 / kwn_tree_* / kwn_roll_down0   candidate rollout of an
//       affine model as an exact forward affine scan (problem.py:449-473):
//       x_{t+1} = A_t x_t + (B_t u_t + c_t), so one up/down sweep replaces
//       the log-depth Newton iterations the nonlinear models need
//   kwn_rollout_seq   the sequential recurrence, one warp per problem, the
//       stage data streamed through a 16-deep cp.async ring so the
//       recurrence runs at the FMA chain's latency (~0.1 us / stage)
//       instead of the global-load latency of the thread kernel
#pragma once

#include <type_traits>

#include "newton_kernels.cuh"
#include "wide.cuh"

namespace ptc {

enum : int { RS_FALLBACK = 8 };   // parallel rollout met a non-finite state

template <class Dyn>
struct IsAffine : std::false_type {};
template <typename R, int NX, int NU>
struct IsAffine<Affine<R, NX, NU>> : std::true_type {};

// affine models with nx >= 8 take the warp-cooperative Newton kernels
template <class Dyn>
constexpr bool kWideNewton = IsAffine<Dyn>::value && Dyn::NX >= 8;

// problems up to this batch size roll out one warp each (larger batches keep
// one thread per problem: enough independent recurrences to hide latency)
constexpr int kWarpRolloutMaxB = 2048;

// ------------------------------------------------------------ gathers

// element (c, t) of a field at base[c * cs + t * ts]; null base reads 0
template <typename R>
struct GField {
  const R* base;
  size_t cs, ts;
};

// SoA trajectory field (comps x rows x B), problem b
template <typename R>
PTC_D GField<R> gf_traj(const R* f, int rows, int B, int b) {
  return GField<R>{f ? f + b : nullptr, (size_t)rows * B, (size_t)B};
}

// affine model field `which` (0 A, 1 Bm, 2 c): the stage-major copy
// [t][A | Bm | c] when the solver keeps one (one contiguous row per stage),
// else the component-major data (comps x lin_T x lin_B), broadcast over
// stages / problems
template <typename R, int NX, int NU>
PTC_D GField<R> gf_model(const ProblemParams& p, int b, int which) {
  constexpr int NC = NX * NX + NX * NU + NX;
  const int off = which == 0 ? 0 : which == 1 ? NX * NX : NX * NX + NX * NU;
  if (p.lin_st) return GField<R>{static_cast<const R*>(p.lin_st) + off, 1, (size_t)NC};
  const void* f = which == 0 ? p.lin_A : which == 1 ? p.lin_Bm : p.lin_c;
  const R* r = static_cast<const R*>(f);
  return GField<R>{r ? r + (p.lin_B > 1 ? b : 0) : nullptr, (size_t)p.lin_T * p.lin_B,
                   p.lin_T > 1 ? (size_t)p.lin_B : (size_t)0};
}

// Register prefetch of one stage of up to five fields with their own
// strides: lane l holds components l, l+32, ... of the concatenation.
template <typename R, int N0, int N1 = 0, int N2 = 0, int N3 = 0, int N4 = 0>
struct WGather {
  static constexpr int TOTAL = N0 + N1 + N2 + N3 + N4;
  static constexpr int PER = (TOTAL + 31) / 32;
  const R* p[PER];
  size_t ts[PER];
  R v[PER];
  PTC_D void init(GField<R> f0, GField<R> f1 = GField<R>{nullptr, 0, 0},
                  GField<R> f2 = GField<R>{nullptr, 0, 0}, GField<R> f3 = GField<R>{nullptr, 0, 0},
                  GField<R> f4 = GField<R>{nullptr, 0, 0}) {
    const int ln = lane_id();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      int c = ln + 32 * k;
      GField<R> f{nullptr, 0, 0};
      if (c < N0) f = f0;
      else if ((c -= N0) < N1) f = f1;
      else if ((c -= N1) < N2) f = f2;
      else if ((c -= N2) < N3) f = f3;
      else if ((c -= N3) < N4) f = f4;
      p[k] = f.base ? f.base + (size_t)c * f.cs : nullptr;
      ts[k] = f.ts;
    }
  }
  PTC_D void load(int t) {
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = p[k] ? __ldg(p[k] + (size_t)t * ts[k]) : R(0);
  }
  PTC_D void store(R* dst) const {
    const int ln = lane_id();
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (ln + 32 * k < TOTAL) dst[ln + 32 * k] = v[k];
    __syncwarp();
  }
};

// ------------------------------------------------------------ cp.async

template <typename R>
PTC_D void cp_async(R* smem, const R* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if constexpr (sizeof(R) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}

PTC_D void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int N>
PTC_D void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ------------------------------------------------------------ stage algebra

// The stacked constraint rows on one lane's variable (lane v < NX: x_v,
// NX <= v < NX + NU: u_{v-NX}), collected once per kernel in row order:
// box constraints put at most an upper and a lower row on a variable.
template <typename R>
struct LaneRows {
  static constexpr int kMax = 4;
  int n;             // rows on this variable; > kMax: use the general loop
  int k[kMax];
  R sgn[kMax], bnd[kMax];
};

template <typename R, int NX, int NU>
PTC_D LaneRows<R> lane_rows(const ProblemParams& p) {
  LaneRows<R> r;
  r.n = 0;
  const int v = lane_id();
  const int var = v < NX ? 0 : 1, idx = v < NX ? v : v - NX;
  for (int k = 0; k < p.W && v < NX + NU; ++k) {
    if (p.row_var[k] != var || p.row_idx[k] != idx) continue;
#pragma unroll
    for (int q = 0; q < LaneRows<R>::kMax; ++q)
      if (q == r.n) {
        r.k[q] = k;
        r.sgn[q] = R(p.row_sign[k]);
        r.bnd[q] = R(p.row_bound[k]);
      }
    ++r.n;
  }
  return r;
}

// Augmentation derivatives (models.cuh aug_derivs), one lane per variable,
// each folding the rows on its variable in row order (same arithmetic: the
// row signs are +-1, so sgn / w == sgn * (1 / w) exactly).
// out = [cx | cu | cxx | cuu].
template <typename R, int NX, int NU>
PTC_D void w_aug_derivs(const ProblemParams& p, const AugArgs<R>& g, const LaneRows<R>& lr, int t,
                        int T, int B, int b, const R* x, const R* u, R* out) {
  const int v = lane_id();
  if (v < NX + NU) {
    const int var = v < NX ? 0 : 1, idx = v < NX ? v : v - NX;
    const R val = v < NX ? x[v] : u[v - NX];
    R gs = R(0), hs = R(0);
    if (g.kind == AUG_BARRIER) {
      if (lr.n <= LaneRows<R>::kMax) {
#pragma unroll
        for (int q = 0; q < LaneRows<R>::kMax; ++q) {
          if (q >= lr.n) break;
          const R w = lr.sgn[q] > 0 ? val - lr.bnd[q] : lr.bnd[q] - val;
          const R inv = R(1) / w;
          const R sc = lr.sgn[q] * inv;
          gs += lr.sgn[q] * inv;
          hs += sc * sc;
        }
      } else {
        for (int k = 0; k < p.W; ++k) {
          if (p.row_var[k] != var || p.row_idx[k] != idx) continue;
          const R bnd = R(p.row_bound[k]);
          const R w = p.row_sign[k] > 0 ? val - bnd : bnd - val;
          const R inv = R(1) / w;
          const R sgn = R(p.row_sign[k]);
          const R sc = sgn / w;
          gs += sgn * inv;
          hs += sc * sc;
        }
      }
      const R mu = R(g.mu[b]);
      gs = -mu * gs;
      hs = mu * hs;
    } else if (g.kind == AUG_ADMM) {
      const R rho = R(g.rho);
      for (int k = 0; k < p.W; ++k) {
        if (p.row_var[k] != var || p.row_idx[k] != idx) continue;
        const R bnd = R(p.row_bound[k]);
        const R w = p.row_sign[k] > 0 ? val - bnd : bnd - val;
        const R res = w - ldf(g.z, k, t, T, B, b) + ldf(g.v, k, t, T, B, b) / rho;
        const R sgn = R(p.row_sign[k]);
        gs += sgn * res;
        hs += sgn * sgn;
      }
      gs *= rho;
      hs *= rho;
    }
    if (v < NX) {
      out[v] = gs;
      out[NX + NU + v] = hs;
    } else {
      out[NX + (v - NX)] = gs;
      out[2 * NX + NU + (v - NX)] = hs;
    }
  }
  __syncwarp();
}

// the warp's copy of the stage-cost constants [Q | goal | Rc]
template <typename R, int NX, int NU>
PTC_D void w_cost_consts(const ProblemParams& p, R* ck) {
  for (int e = lane_id(); e < NX * NX; e += 32) ck[e] = R(p.Q[e]);
  for (int e = lane_id(); e < NX; e += 32) ck[NX * NX + e] = R(p.goal[e]);
  for (int e = lane_id(); e < NU * NU; e += 32) ck[NX * NX + NX + e] = R(p.Rc[e]);
  __syncwarp();
}

template <typename R>
PTC_D bool nw_skip(const NewtonArgs<R>& a, int b, int gate) {
  if (gate == 1) return !running(a, b) || !(a.phase[b] & PH_NEED_EXP);
  if (gate == 2) return (a.rstate[b] & RS_SKIP) != 0;
  return false;
}

template <typename R, int NX, int NU>
struct NSlab {
  static constexpr int CC = NX * NX + NX;
  static constexpr int AUG = 2 * NX + 2 * NU;
  static constexpr int CK = NX * NX + NX + NU * NU;   // Q, goal, Rc copies
  static constexpr int kCoUp0 = 3 * CC + (NX * NX + NX + NU) + AUG + 2 * NX + CK;
  static constexpr int kTree = 3 * CC;
  static constexpr int kCoDown0 = (NX * NX + NX * NU + NX + NU) + 2 * NX + AUG + CK;
  static constexpr int ROLL = CC + NX * NU + 2 * NU;   // [A | c | Bm | u | du]
  static constexpr int kRollUp0 = 2 * CC + ROLL;
  static constexpr int kRollDown0 = 2 * NX + ROLL;
  static constexpr int kCost = NX + NU + CK;
};

#define PTC_NW_PROLOGUE(count, gate, ...)        \
  const int u = warp_unit();                     \
  if (u >= (count) * a.B) return;                \
  const int b = u % a.B, j = u / a.B;            \
  (void)j;                                       \
  if (nw_skip(a, b, (gate))) return;             \
  using N = NSlab<R, NX, NU>;                    \
  R* slab = warp_slab<R>((__VA_ARGS__));

// ------------------------------------------------------------ co-state scan

// level-0 up-sweep: fold lambda_t = q_t + A_t^T lambda_{t+1} over a chunk
// (k_costate_up0; the last stage absorbs the terminal gradient, F = 0)
template <typename R, int NX, int NU>
__global__ void __launch_bounds__(64) kwn_costate_up0(NewtonArgs<R> a) {
  PTC_NW_PROLOGUE(a.plan.units0(), 1, NSlab<R, NX, NU>::kCoUp0)
  const int q = a.parity[b], T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const ProblemParams& p = *a.pp;
  const AugArgs<R> g = aug_of(a);
  const LaneRows<R> lr = lane_rows<R, NX, NU>(p);
  R* acc = slab;
  R* m = acc + N::CC;
  R* o = m + N::CC;
  R* F = o + N::CC;           // [A | x | u]
  R* x = F + NX * NX;
  R* uu = x + NX;
  R* aug = uu + NU;
  R* v0 = aug + N::AUG;
  R* v1 = v0 + NX;
  R* Qs = v1 + NX;             // [Q | goal | Rc]
  const R* gs = Qs + NX * NX;
  const int ln = lane_id();
  w_cost_consts<R, NX, NU>(p, Qs);
  w_identity<NX>(acc);
  w_fill<NX>(acc + NX * NX, R(0));
  WGather<R, NX * NX, NX, NU> pf;
  pf.init(gf_model<R, NX, NU>(p, b, 0), gf_traj(a.X + q * a.xsz, T + 1, B, b),
          gf_traj(a.U + q * a.usz, T, B, b));
  if (t0 < t1) pf.load(t1 - 1);
  for (int t = t1 - 1; t >= t0; --t) {
    pf.store(F);
    if (t - 1 >= t0) pf.load(t - 1);
    w_aug_derivs<R, NX, NU>(p, g, lr, t, T, B, b, x, uu, aug);
    for (int e = ln; e < NX * NX; e += 32) {
      const int i = e / NX, k = e - (e / NX) * NX;
      m[e] = F[k * NX + i];
    }
    for (int i = ln; i < NX; i += 32) {
      R lx = R(0);
#pragma unroll
      for (int k = 0; k < NX; ++k) lx += (x[k] - gs[k]) * Qs[i * NX + k];
      m[NX * NX + i] = lx + aug[i];
    }
    __syncwarp();
    if (t == T - 1 && (!a.blk || a.blk_last)) {
      w_ld<NX>(a.X + q * a.xsz, T, T + 1, B, b, v0);
      for (int i = ln; i < NX; i += 32) {
        R s = R(0);
#pragma unroll
        for (int k = 0; k < NX; ++k) s += R(p.Qf[i * NX + k]) * (v0[k] - R(p.goal[k]));
        v1[i] = s;
      }
      __syncwarp();
      w_mv<NX, NX, false, 0>(m, v1, v0);
      for (int i = ln; i < NX; i += 32) m[NX * NX + i] += v0[i];
      for (int e = ln; e < NX * NX; e += 32) m[e] = R(0);
      __syncwarp();
    }
    w_aff_compose<R, NX>(m, acc, o);
    R* sw = acc;
    acc = o;
    o = sw;
  }
  w_st<N::CC>(a.cagg[1], j, a.plan.n[1], B, b, acc);
}

// generic affine tree kernels on cagg / ccar: kRev = reverse (co-state)
// direction, else forward (rollout).  gate as nw_skip.
template <typename R, int NX, int NU, bool kRev>
__global__ void __launch_bounds__(64) kwn_tree_up(NewtonArgs<R> a, int l, int gate) {
  PTC_NW_PROLOGUE(a.plan.n[l + 1], gate, NSlab<R, NX, NU>::kTree)
  const int nl = a.plan.n[l], nn = a.plan.n[l + 1];
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  R* acc = slab;
  R* m = acc + N::CC;
  R* o = m + N::CC;
  w_ld<N::CC>(a.cagg[l], kRev ? last : first, nl, a.B, b, acc);
  const int n = last - first;
  for (int s = 1; s <= n; ++s) {
    const int i = kRev ? last - s : first + s;
    w_ld<N::CC>(a.cagg[l], i, nl, a.B, b, m);
    w_aff_compose<R, NX>(m, acc, o);
    R* sw = acc;
    acc = o;
    o = sw;
  }
  w_st<N::CC>(a.cagg[l + 1], j, nn, a.B, b, acc);
}

template <typename R, int NX>
PTC_D void w_aff_apply_inplace(const R* m, R* x, R* y) {
  w_mv<NX, NX, false, 0>(m, x, y);
  for (int k = lane_id(); k < NX; k += 32) x[k] = y[k] + m[NX * NX + k];
  __syncwarp();
}

template <typename R, int NX, int NU, bool kRev>
__global__ void __launch_bounds__(64) kwn_tree_top(NewtonArgs<R> a, int gate, int xbuf) {
  PTC_NW_PROLOGUE(1, gate, NSlab<R, NX, NU>::kTree)
  const int L = a.plan.L, nL = a.plan.n[L];
  R* x = slab;
  R* m = x + N::CC;
  R* y = m + N::CC;
  if (kRev) {
    // co-state entering at the horizon end: 0 (the last chunk absorbed the
    // terminal gradient), or the later blocks' carry in block mode
    if (a.blk && !a.blk_last) w_ld<NX>(a.lam_in, 0, 1, a.B, b, x);
    else w_fill<NX>(x, R(0));
  } else if (a.blk) {
    w_ld<NX>(a.x_in, 0, 1, a.B, b, x);   // state at the block start
  } else {
    w_ld<NX>(a.X + (xbuf < 0 ? a.parity[b] : xbuf) * a.xsz, 0, a.T + 1, a.B, b, x);  // x_0
  }
  for (int s = 0; s < nL; ++s) {
    const int i = kRev ? nL - 1 - s : s;
    w_st<NX>(a.ccar[L], i, nL, a.B, b, x);
    w_ld<N::CC>(a.cagg[L], i, nL, a.B, b, m);
    w_aff_apply_inplace<R, NX>(m, x, y);
  }
}

template <typename R, int NX, int NU, bool kRev>
__global__ void __launch_bounds__(64) kwn_tree_down(NewtonArgs<R> a, int l, int gate) {
  PTC_NW_PROLOGUE(a.plan.n[l + 1], gate, NSlab<R, NX, NU>::kTree)
  const int nl = a.plan.n[l], nn = a.plan.n[l + 1];
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  R* x = slab;
  R* m = x + N::CC;
  R* y = m + N::CC;
  w_ld<NX>(a.ccar[l + 1], j, nn, a.B, b, x);
  for (int s = 0; s <= last - first; ++s) {
    const int i = kRev ? last - s : first + s;
    w_st<NX>(a.ccar[l], i, nl, a.B, b, x);
    w_ld<N::CC>(a.cagg[l], i, nl, a.B, b, m);
    w_aff_apply_inplace<R, NX>(m, x, y);
  }
}

// level-0 down-sweep fused with the expansion (k_costate_down0 /
// stage_expansion for affine dynamics): with lambda_{t+1} in the slab,
// emit P, R, M, d, Fx, Fu and lambda_t of every stage of the chunk.
// xst: write the expansion as stage-major rows [P R M d Fx Fu] (the wide
// LQR's staged layout, wide.cuh) instead of the component-major fields.
template <typename R, int NX, int NU>
__global__ void __launch_bounds__(64) kwn_costate_down0(NewtonArgs<R> a, R* xst) {
  PTC_NW_PROLOGUE(a.plan.units0(), 1, NSlab<R, NX, NU>::kCoDown0)
  using WS = WSlab<R, NX, NU>;
  const int P0 = a.plan.units0();
  const int q = a.parity[b], T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const ProblemParams& p = *a.pp;
  const AugArgs<R> g = aug_of(a);
  const LaneRows<R> lr = lane_rows<R, NX, NU>(p);
  R* F = slab;                 // [A | Bm | x | u]
  R* Bm = F + NX * NX;
  R* x = Bm + NX * NU;
  R* uu = x + NX;
  R* lnx = uu + NU;            // lambda_{t+1}
  R* lt = lnx + NX;            // lambda_t
  R* aug = lt + NX;
  R* Qs = aug + N::AUG;        // [Q | goal | Rc]
  const R* gs = Qs + NX * NX;
  const R* Rcs = gs + NX;
  const int ln = lane_id();
  const R* X = a.X + q * a.xsz;
  w_cost_consts<R, NX, NU>(p, Qs);
  if (j == P0 - 1 && a.blk && !a.blk_last) {
    w_ld<NX>(a.lam_in, 0, 1, B, b, lnx);   // carry from the later blocks
    w_st<NX>(a.lam, T, T + 1, B, b, lnx);
  } else if (j == P0 - 1) {
    w_ld<NX>(X, T, T + 1, B, b, lt);
    for (int i = ln; i < NX; i += 32) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < NX; ++k) s += R(p.Qf[i * NX + k]) * (lt[k] - R(p.goal[k]));
      lnx[i] = s;
    }
    __syncwarp();
    w_st<NX>(a.lam, T, T + 1, B, b, lnx);
    for (int e = ln; e < NX * NX; e += 32) {
      const int i = e / NX, k = e - (e / NX) * NX;
      const R v = i == k ? R(p.Qf[e]) : R(0.5) * (R(p.Qf[i * NX + k]) + R(p.Qf[k * NX + i]));
      a.PT[(size_t)e * B + b] = v;
    }
  } else {
    w_ld<NX>(a.ccar[1], j, a.plan.n[1], B, b, lnx);
  }
  WGather<R, NX * NX, NX * NU, NX, NU> pf;
  pf.init(gf_model<R, NX, NU>(p, b, 0), gf_model<R, NX, NU>(p, b, 1), gf_traj(X, T + 1, B, b),
          gf_traj(a.U + q * a.usz, T, B, b));
  if (t0 < t1) pf.load(t1 - 1);
  const R* cxx = aug + NX + NU;
  const R* cuu = cxx + NX;
  for (int t = t1 - 1; t >= t0; --t) {
    pf.store(F);
    if (t - 1 >= t0) pf.load(t - 1);
    w_aug_derivs<R, NX, NU>(p, g, lr, t, T, B, b, x, uu, aug);
    if (ln < NX) {
      const int i = ln;
      R lx = R(0);
#pragma unroll
      for (int k = 0; k < NX; ++k) lx += (x[k] - gs[k]) * Qs[i * NX + k];
      R fxl = F[i] * lnx[0];
#pragma unroll
      for (int k = 1; k < NX; ++k) fxl = fma(F[k * NX + i], lnx[k], fxl);
      lt[i] = (lx + aug[i]) + fxl;
    } else if (ln < NX + NU) {
      const int i = ln - NX;
      R ftl = Bm[i] * lnx[0];
#pragma unroll
      for (int k = 1; k < NX; ++k) ftl = fma(Bm[k * NU + i], lnx[k], ftl);
      R ru = R(0);
#pragma unroll
      for (int k = 0; k < NU; ++k) ru += uu[k] * Rcs[i * NU + k];
      const R di = (ru + aug[NX + i]) + ftl;
      if (xst) xst[(size_t)t * WS::SC + WS::sd + i] = di;
      else a.d[((size_t)i * T + t) * B + b] = di;
    }
    // P = sym(Q + diag cxx), R = sym(Rc + diag cuu), M = 0, Fx = A, Fu = B
    constexpr int nP = NX * NX, nR = NU * NU, nM = NX * NU;
    R* row = xst ? xst + (size_t)t * WS::SC : nullptr;
    for (int e = ln; e < 2 * nP + nR + 2 * nM; e += 32) {
      if (e < nP) {
        const int i = e / NX, k = e - (e / NX) * NX;
        const R pik = (Qs[i * NX + k] + (i == k ? cxx[i] : R(0))) + R(0);
        const R pki = (Qs[k * NX + i] + (i == k ? cxx[i] : R(0))) + R(0);
        const R v = i == k ? pik : R(0.5) * (pik + pki);
        if (row) row[WS::sP + e] = v;
        else a.P[((size_t)e * T + t) * B + b] = v;
      } else if (e < nP + nR) {
        const int c = e - nP, i = c / NU, k = c - (c / NU) * NU;
        const R rik = (Rcs[i * NU + k] + (i == k ? cuu[i] : R(0))) + R(0);
        const R rki = (Rcs[k * NU + i] + (i == k ? cuu[i] : R(0))) + R(0);
        const R v = i == k ? rik : R(0.5) * (rik + rki);
        if (row) row[WS::sR + c] = v;
        else a.Rm[((size_t)c * T + t) * B + b] = v;
      } else if (e < nP + nR + nM) {
        const int c = e - nP - nR;
        if (row) row[WS::sM + c] = R(0);
        else a.M[((size_t)c * T + t) * B + b] = R(0);
      } else if (e < 2 * nP + nR + nM) {
        const int c = e - nP - nR - nM;
        if (row) row[WS::sFx + c] = F[c];
        else a.Fx[((size_t)c * T + t) * B + b] = F[c];
      } else {
        const int c = e - 2 * nP - nR - nM;
        if (row) row[WS::sFu + c] = Bm[c];
        else a.Fu[((size_t)c * T + t) * B + b] = Bm[c];
      }
    }
    __syncwarp();
    for (int i = ln; i < NX; i += 32) {
      a.lam[((size_t)i * (T + 1) + t) * B + b] = lt[i];
      lnx[i] = lt[i];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------ rollout scan

// candidate controls u + du of stage t into the slab's u slot
template <typename R, int NX, int NU>
PTC_D void w_cand_controls(R* uu, const R* du) {
  for (int i = lane_id(); i < NU; i += 32) uu[i] += du[i];
  __syncwarp();
}

// Affine-scan rollout, kMode 1: the Newton candidate u + du of buffer parity
// into 1 - parity (gated by k_roll_gate); kMode 0: problem.py `rollout` of
// buffer 0 in place.
// level-0 up-sweep: fold (A_t, B_t u_t + c_t) over the chunk
template <typename R, int NX, int NU, int kMode>
__global__ void __launch_bounds__(64) kwn_roll_up0(NewtonArgs<R> a, const R* dU) {
  PTC_NW_PROLOGUE(a.plan.units0(), (kMode == 1 ? 2 : 0), NSlab<R, NX, NU>::kRollUp0)
  const int q = kMode == 1 ? a.parity[b] : 0, T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const ProblemParams& p = *a.pp;
  R* acc = slab;
  R* o = acc + N::CC;
  R* F = o + N::CC;            // [A | c | Bm | u | du]; [A | e] is the stage map
  R* Bm = F + N::CC;
  R* uu = Bm + NX * NU;
  R* du = uu + NU;
  w_identity<NX>(acc);
  w_fill<NX>(acc + NX * NX, R(0));
  WGather<R, NX * NX, NX, NX * NU, NU, NU> pf;
  pf.init(gf_model<R, NX, NU>(p, b, 0), gf_model<R, NX, NU>(p, b, 2), gf_model<R, NX, NU>(p, b, 1),
          gf_traj(a.U + q * a.usz, T, B, b), gf_traj(dU, T, B, b));
  if (t0 < t1) pf.load(t0);
  for (int t = t0; t < t1; ++t) {
    pf.store(F);
    if (t + 1 < t1) pf.load(t + 1);
    if (kMode == 1) w_cand_controls<R, NX, NU>(uu, du);
    for (int i = lane_id(); i < NX; i += 32) {
      R bu = Bm[i * NU] * uu[0];
#pragma unroll
      for (int k = 1; k < NU; ++k) bu = fma(Bm[i * NU + k], uu[k], bu);
      F[NX * NX + i] = bu + F[NX * NX + i];
    }
    __syncwarp();
    w_aff_compose<R, NX>(F, acc, o);
    R* sw = acc;
    acc = o;
    o = sw;
  }
  w_st<N::CC>(a.cagg[1], j, a.plan.n[1], B, b, acc);
}

// level-0 down-sweep: x_{t+1} = (A_t x_t + B_t u_t) + c_t from the chunk's
// carry (the sequential recurrence's own arithmetic), candidate controls and
// states stored; a non-finite state flags the problem for the sequential
// fallback (overflowing aggregates must not decide divergence)
template <typename R, int NX, int NU, int kMode>
__global__ void __launch_bounds__(64) kwn_roll_down0(NewtonArgs<R> a, const R* dU) {
  PTC_NW_PROLOGUE(a.plan.units0(), (kMode == 1 ? 2 : 0), NSlab<R, NX, NU>::kRollDown0)
  const int q = kMode == 1 ? a.parity[b] : 0, T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const ProblemParams& p = *a.pp;
  R* Xc = a.X + (kMode == 1 ? 1 - q : 0) * a.xsz;
  R* Uc = a.U + (1 - q) * a.usz;
  R* x = slab;
  R* y = x + NX;
  R* F = y + NX;               // [A | c | Bm | u | du]
  R* c = F + NX * NX;
  R* Bm = c + NX;
  R* uu = Bm + NX * NU;
  R* du = uu + NU;
  const int ln = lane_id();
  if (j == 0 && a.blk) {
    w_ld<NX>(a.x_in, 0, 1, B, b, x);
    w_st<NX>(Xc, 0, T + 1, B, b, x);
  } else if (j == 0) {
    w_ld<NX>(a.X + q * a.xsz, 0, T + 1, B, b, x);
    if (kMode == 1) w_st<NX>(Xc, 0, T + 1, B, b, x);
  } else {
    w_ld<NX>(a.ccar[1], j, a.plan.n[1], B, b, x);
  }
  WGather<R, NX * NX, NX, NX * NU, NU, NU> pf;
  pf.init(gf_model<R, NX, NU>(p, b, 0), gf_model<R, NX, NU>(p, b, 2), gf_model<R, NX, NU>(p, b, 1),
          gf_traj(a.U + q * a.usz, T, B, b), gf_traj(dU, T, B, b));
  if (t0 < t1) pf.load(t0);
  bool finite = true;
  int first_bad = -1;
  for (int t = t0; t < t1; ++t) {
    pf.store(F);
    if (t + 1 < t1) pf.load(t + 1);
    if (kMode == 1) {
      w_cand_controls<R, NX, NU>(uu, du);
      if (ln < NU) Uc[((size_t)ln * T + t) * B + b] = uu[ln];
    }
    if (ln < NX) {
      const int i = ln;
      R ax = F[i * NX] * x[0];
#pragma unroll
      for (int k = 1; k < NX; ++k) ax = fma(F[i * NX + k], x[k], ax);
      R bu = Bm[i * NU] * uu[0];
#pragma unroll
      for (int k = 1; k < NU; ++k) bu = fma(Bm[i * NU + k], uu[k], bu);
      const R xn = (ax + bu) + c[i];
      if (finite && !isfinite(xn)) first_bad = t + 1;
      finite = finite && isfinite(xn);
      y[i] = xn;
      Xc[((size_t)i * (T + 1) + t + 1) * B + b] = xn;
    }
    __syncwarp();
    if (ln < NX) x[ln] = y[ln];
    __syncwarp();
  }
  if (!a.blk) {
    if (__any_sync(0xffffffffu, !finite) && ln == 0) atomicOr(a.rstate + b, RS_FALLBACK);
  } else if (kMode == 1) {
    // block mode has no sequential fallback (the recurrence crosses ranks):
    // a non-finite candidate is a rejected step, as the reference's
    // DivergenceError inside newton_solve
    if (__any_sync(0xffffffffu, !finite) && ln == 0) atomicOr(a.flags + b, FLAG_DIVERGED);
  } else if (!finite) {
    // rollout API: first non-finite global state index (min over chunks)
    atomicMin(reinterpret_cast<unsigned*>(a.bad_index + b), unsigned(a.t_base + first_bad));
  }
}

// ------------------------------------------------------------ sequential

// One warp per problem: x_{t+1} = (A_t x_t + B_t u_t) + c_t, lane i < NX
// owning state i (bitwise the thread kernel's Affine::step arithmetic), the
// stage data [A | Bm | c | u (| du)] streamed kDepth stages ahead through a
// cp.async ring in shared memory.
//   kMode 0: problem.py `rollout` of buffer 0 in place (first non-finite
//            stage + 1 in bad_index, as k_rollout_inplace)
//   kMode 1: the Newton candidate u + du from buffer parity into 1 - parity
//            (k_rollout<.., false>); only_flagged: just the problems the
//            parallel rollout flagged RS_FALLBACK
template <typename R, int NX, int NU, int kMode>
__global__ void __launch_bounds__(32) kwn_rollout_seq(NewtonArgs<R> a, const R* dU,
                                                      int only_flagged) {
  constexpr int kDepth = 16;
  constexpr int NC = NX * NX + NX * NU + NX + NU + (kMode == 1 ? NU : 0);
  constexpr int oB = NX * NX, oC = oB + NX * NU, oU = oC + NX, oD = oU + NU;
  const int b = blockIdx.x;
  if (b >= a.B) return;
  if (kMode == 1 && (a.rstate[b] & RS_SKIP)) return;
  if (only_flagged && !(a.rstate[b] & RS_FALLBACK)) return;
  extern __shared__ __align__(16) unsigned char w_smem[];
  R* ring = reinterpret_cast<R*>(w_smem);
  const int T = a.T, B = a.B;
  const int q = kMode == 1 ? a.parity[b] : 0;
  const ProblemParams& p = *a.pp;
  WGather<R, NX * NX, NX * NU, NX, NU, (kMode == 1 ? NU : 0)> g;
  g.init(gf_model<R, NX, NU>(p, b, 0), gf_model<R, NX, NU>(p, b, 1), gf_model<R, NX, NU>(p, b, 2),
         gf_traj(a.U + q * a.usz, T, B, b), gf_traj(dU, T, B, b));
  const int ln = lane_id();
  auto issue = [&](int t) {
    R* slot = ring + (t % kDepth) * NC;
#pragma unroll
    for (int k = 0; k < g.PER; ++k) {
      const int c = ln + 32 * k;
      if (c < NC) {
        if (g.p[k]) cp_async(slot + c, g.p[k] + (size_t)t * g.ts[k]);
        else slot[c] = R(0);
      }
    }
  };
#pragma unroll 1
  for (int s = 0; s < kDepth; ++s) {
    if (s < T) issue(s);
    cp_async_commit();
  }
  R* Xo = a.X + (kMode == 1 ? (1 - q) * a.xsz : 0);
  R* Uc = a.U + (1 - q) * a.usz;
  R xi = ln < NX ? a.X[((size_t)ln * (T + 1)) * B + b + q * a.xsz] : R(0);
  if (kMode == 1 && ln < NX) Xo[((size_t)ln * (T + 1)) * B + b] = xi;
  bool finite = true, reported = false;
  for (int t = 0; t < T; ++t) {
    cp_async_wait<kDepth - 1>();
    __syncwarp();
    const R* S = ring + (t % kDepth) * NC;
    R xs[NX];
#pragma unroll
    for (int k = 0; k < NX; ++k) xs[k] = __shfl_sync(0xffffffffu, xi, k);
    R uk[NU];
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      uk[k] = S[oU + k];
      if (kMode == 1) uk[k] += S[oD + k];
    }
    R xn = R(0);
    if (ln < NX) {
      R ax = S[ln * NX] * xs[0];
#pragma unroll
      for (int k = 1; k < NX; ++k) ax = fma(S[ln * NX + k], xs[k], ax);
      R bu = S[oB + ln * NU] * uk[0];
#pragma unroll
      for (int k = 1; k < NU; ++k) bu = fma(S[oB + ln * NU + k], uk[k], bu);
      xn = (ax + bu) + S[oC + ln];
    }
    __syncwarp();
    if (t + kDepth < T) issue(t + kDepth);
    cp_async_commit();
    if (kMode == 1) {
#pragma unroll
      for (int k = 0; k < NU; ++k)
        if (ln == k) Uc[((size_t)k * T + t) * B + b] = uk[k];
    }
    const bool bad = ln < NX && !isfinite(xn);
    if (kMode == 0 && !reported && __any_sync(0xffffffffu, bad)) {
      reported = true;
      if (ln == 0) a.bad_index[b] = t + 1;
    }
    finite = finite && !bad;
    if (ln < NX) {
      xi = xn;
      Xo[((size_t)ln * (T + 1) + t + 1) * B + b] = xn;
    }
  }
  cp_async_wait<0>();
  if (kMode == 1 && __any_sync(0xffffffffu, !finite) && ln == 0) atomicOr(a.flags + b, FLAG_DIVERGED);
}

// ------------------------------------------------------------ time blocks

// the block's whole map: fold the top tree level (kRev: reverse order) into
// one affine aggregate, out (CC, 1, B)
template <typename R, int NX, int NU, bool kRev>
__global__ void __launch_bounds__(64) kwn_tree_block(NewtonArgs<R> a, R* out, int gate) {
  PTC_NW_PROLOGUE(1, gate, NSlab<R, NX, NU>::kTree)
  const int L = a.plan.L, nL = a.plan.n[L];
  R* acc = slab;
  R* m = acc + N::CC;
  R* o = m + N::CC;
  w_ld<N::CC>(a.cagg[L], kRev ? nL - 1 : 0, nL, a.B, b, acc);
  for (int s = 1; s < nL; ++s) {
    w_ld<N::CC>(a.cagg[L], kRev ? nL - 1 - s : s, nL, a.B, b, m);
    w_aff_compose<R, NX>(m, acc, o);
    R* sw = acc;
    acc = o;
    o = sw;
  }
  w_st<N::CC>(out, 0, 1, a.B, b, acc);
}

// carry entering this rank's block from the gathered block maps
// g (world, CC, 1, B): kRev: co-state at the block end = maps of ranks
// world-1 .. rank+1 applied to 0 (the last block's map is constant);
// forward: state at the block start = maps of ranks 0 .. rank-1 applied to x0
template <typename R, int NX, int NU, bool kRev>
__global__ void __launch_bounds__(64) kwn_blk_carry(NewtonArgs<R> a, const R* g, int rank,
                                                    int world, int gate) {
  PTC_NW_PROLOGUE(1, gate, NSlab<R, NX, NU>::kTree)
  if (kRev && a.blk_last) return;
  R* x = slab;
  R* m = x + N::CC;
  R* y = m + N::CC;
  const size_t stride = (size_t)N::CC * a.B;
  if (kRev) {
    w_fill<NX>(x, R(0));
    for (int k = world - 1; k > rank; --k) {
      w_ld<N::CC>(g + k * stride, 0, 1, a.B, b, m);
      w_aff_apply_inplace<R, NX>(m, x, y);
    }
    w_st<NX>(a.lam_in, 0, 1, a.B, b, x);
  } else {
    w_ld<NX>(a.x0g, 0, 1, a.B, b, x);
    for (int k = 0; k < rank; ++k) {
      w_ld<N::CC>(g + k * stride, 0, 1, a.B, b, m);
      w_aff_apply_inplace<R, NX>(m, x, y);
    }
    w_st<NX>(a.x_in, 0, 1, a.B, b, x);
  }
}

// Cost partials of one chunk (k_cost_partials, models.cuh stage_cost /
// aug_value) with the work spread over the warp: lane i < NX accumulates
// row i of (x - g)^T Q (x - g) over the chunk's stages, lanes NX..NX+NU-1 the
// control rows of u^T Rc u, lane k < W constraint row k's barrier log /
// ADMM residual square and its first infeasible stage; one warp reduction
// per chunk instead of a serial per-stage sum on one thread.
template <typename R, int NX, int NU>
__global__ void __launch_bounds__(64) kwn_cost_partials(NewtonArgs<R> a, int which) {
  const int u = warp_unit();
  if (u >= a.plan.units0() * a.B) return;
  const int b = u % a.B, j = u / a.B;
  if (!running(a, b)) return;
  if (which == 0 && !(a.phase[b] & PH_NEED_COST)) return;
  using N = NSlab<R, NX, NU>;
  R* slab = warp_slab<R>(N::kCost);
  R* xu = slab;                 // [x | u] of the stage
  R* ck = xu + NX + NU;         // [Q | goal | Rc]
  const int P0 = a.plan.units0(), T = a.T, B = a.B;
  const int q = which == 0 ? a.parity[b] : 1 - a.parity[b];
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const ProblemParams& p = *a.pp;
  const AugArgs<R> g = aug_of(a);
  const int ln = lane_id();
  w_cost_consts<R, NX, NU>(p, ck);
  const R* Qs = ck;
  const R* gs = ck + NX * NX;
  const R* Rcs = gs + NX;
  // this lane's constraint row
  const int W = p.W;
  const bool has_row = ln < W && g.kind != AUG_ZERO;
  int rvar = 0, ridx = 0;
  R rsgn = R(0), rbnd = R(0);
  if (has_row) {
    rvar = p.row_var[ln];
    ridx = p.row_idx[ln];
    rsgn = R(p.row_sign[ln]);
    rbnd = R(p.row_bound[ln]);
  }
  const R rho = R(g.rho);
  double aq = 0.0, ac = 0.0;
  int first_bad = -1;
  WGather<R, NX, NU> pf;
  pf.init(gf_traj(a.X + q * a.xsz, T + 1, B, b), gf_traj(a.U + q * a.usz, T, B, b));
  if (t0 < t1) pf.load(t0);
  for (int t = t0; t < t1; ++t) {
    pf.store(xu);
    if (t + 1 < t1) pf.load(t + 1);
    if (ln < NX) {
      const R ei = xu[ln] - gs[ln];
      R r = R(0);
#pragma unroll
      for (int k = 0; k < NX; ++k) r += ei * Qs[ln * NX + k] * (xu[k] - gs[k]);
      aq += double(r);
    } else if (ln < NX + NU) {
      const int i = ln - NX;
      R r = R(0);
#pragma unroll
      for (int k = 0; k < NU; ++k) r += xu[NX + i] * Rcs[i * NU + k] * xu[NX + k];
      aq += double(r);
    }
    if (has_row) {
      R var = R(0);
#pragma unroll
      for (int i = 0; i < NX; ++i) var = (rvar == 0 && i == ridx) ? xu[i] : var;
#pragma unroll
      for (int i = 0; i < NU; ++i) var = (rvar == 1 && i == ridx) ? xu[NX + i] : var;
      const R w = rsgn > 0 ? var - rbnd : rbnd - var;
      if (g.kind == AUG_BARRIER) {
        if (w >= R(0) && first_bad < 0) first_bad = t;
        ac += double(log(-w));
      } else {
        const R res = w - ldf(g.z, ln, t, T, B, b) + ldf(g.v, ln, t, T, B, b) / rho;
        ac += double(res * res);
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    aq += __shfl_xor_sync(0xffffffffu, aq, off);
    ac += __shfl_xor_sync(0xffffffffu, ac, off);
  }
  // first infeasible (stage, row) in stage-major order
  int bad = first_bad >= 0 ? first_bad * W + ln : 0x7fffffff;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, off));
  if (ln == 0) {
    double sc = 0.0;
    if (g.kind == AUG_BARRIER) sc = -a.mu[b] * ac;
    else if (g.kind == AUG_ADMM) sc = 0.5 * double(rho) * ac;
    double* cp = a.cpart[which];
    cp[((size_t)0 * P0 + j) * B + b] = 0.5 * aq;
    cp[((size_t)1 * P0 + j) * B + b] = sc;
    cp[((size_t)2 * P0 + j) * B + b] = bad == 0x7fffffff ? -1.0 : double(bad);
  }
}

#undef PTC_NW_PROLOGUE

// Reduction vectors exchanged between ranks (ptc_solver_block_phase): each
// folds the per-chunk partial rows into one value per problem (export) and
// writes the all-reduced value back as row 0 with identity rows after it
// (import), so k_control / k_outer read the horizon-wide numbers.
template <typename R>
__global__ void k_blk_export_red(NewtonArgs<R> a, double* out) {
  const int b = unit_id();
  if (b >= a.B) return;
  const int P0 = a.plan.units0(), B = a.B;
  double s2 = 0.0, sd = 0.0, mx = 0.0;
  for (int j = 0; j < partial_rows(P0); ++j) {
    s2 += a.red[((size_t)0 * P0 + j) * B + b];
    sd += a.red[((size_t)1 * P0 + j) * B + b];
    mx = nanmax(mx, a.red[((size_t)2 * P0 + j) * B + b]);
  }
  const int fl = a.flags[b];
  out[0 * B + b] = s2;
  out[1 * B + b] = sd;
  out[2 * B + b] = mx;
  out[3 * B + b] = (fl & FLAG_DEF_R) ? 1.0 : 0.0;
  out[4 * B + b] = (fl & FLAG_DEF_Q) ? 1.0 : 0.0;
  out[5 * B + b] = (fl & FLAG_COND) ? 1.0 : 0.0;
}

template <typename R>
__global__ void k_blk_import_red(NewtonArgs<R> a, const double* in) {
  const int b = unit_id();
  if (b >= a.B) return;
  const int P0 = a.plan.units0(), B = a.B;
  for (int f = 0; f < 3; ++f)
    for (int j = 0; j < partial_rows(P0); ++j)
      a.red[((size_t)f * P0 + j) * B + b] = j == 0 ? in[f * B + b] : 0.0;
  int fl = a.flags[b];
  if (in[3 * B + b] > 0.0) fl |= FLAG_DEF_R;
  if (in[4 * B + b] > 0.0) fl |= FLAG_DEF_Q;
  if (in[5 * B + b] > 0.0) fl |= FLAG_COND;
  a.flags[b] = fl;
}

template <typename R, int NX>
__global__ void k_blk_export_cost(NewtonArgs<R> a, double* out) {
  const int b = unit_id();
  if (b >= a.B) return;
  const int P0 = a.plan.units0(), B = a.B, W = a.pp->W;
  for (int w = 0; w < 2; ++w) {
    const double* cp = a.cpart[w];
    double sl = 0.0, sc = 0.0;
    int bad = -1;
    for (int j = 0; j < partial_rows(P0); ++j) {
      sl += cp[((size_t)0 * P0 + j) * B + b];
      sc += cp[((size_t)1 * P0 + j) * B + b];
      const int bj = int(cp[((size_t)2 * P0 + j) * B + b]);
      if (bad < 0 && bj >= 0) bad = bj;
    }
    if (a.blk_last) {
      R xT[NX];
      ld_x(a, w == 0 ? a.parity[b] : 1 - a.parity[b], a.T, b, xT);
      sl += double(terminal_cost(*a.pp, xT));
    }
    out[(2 * w + 0) * B + b] = sl;
    out[(2 * w + 1) * B + b] = sc;
    out[(5 + w) * B + b] = bad >= 0 ? double(bad) + double(a.t_base) * W : 1e300;
  }
  out[4 * B + b] = (a.flags[b] & FLAG_DIVERGED) ? 1.0 : 0.0;
}

template <typename R>
__global__ void k_blk_import_cost(NewtonArgs<R> a, const double* in) {
  const int b = unit_id();
  if (b >= a.B) return;
  const int P0 = a.plan.units0(), B = a.B;
  for (int w = 0; w < 2; ++w) {
    double* cp = a.cpart[w];
    const double bad = in[(5 + w) * B + b];
    for (int j = 0; j < partial_rows(P0); ++j) {
      cp[((size_t)0 * P0 + j) * B + b] = j == 0 ? in[(2 * w + 0) * B + b] : 0.0;
      cp[((size_t)1 * P0 + j) * B + b] = j == 0 ? in[(2 * w + 1) * B + b] : 0.0;
      cp[((size_t)2 * P0 + j) * B + b] = (j == 0 && bad < 1e299) ? bad : -1.0;
    }
  }
  if (in[4 * B + b] > 0.0) a.flags[b] |= FLAG_DIVERGED;
}

template <typename R>
__global__ void k_blk_export_apart(NewtonArgs<R> a, double* out) {
  const int b = unit_id();
  if (b >= a.B) return;
  const int P0 = a.plan.units0(), B = a.B;
  double rp = 0.0, rd = 0.0;
  if (a.apart)
    for (int j = 0; j < partial_rows(P0); ++j) {
      rp = nanmax(rp, a.apart[((size_t)0 * P0 + j) * B + b]);
      rd = nanmax(rd, a.apart[((size_t)1 * P0 + j) * B + b]);
    }
  out[0 * B + b] = rp;
  out[1 * B + b] = rd;
}

template <typename R>
__global__ void k_blk_import_apart(NewtonArgs<R> a, const double* in) {
  const int b = unit_id();
  if (b >= a.B || !a.apart) return;
  const int P0 = a.plan.units0(), B = a.B;
  for (int f = 0; f < 2; ++f)
    for (int j = 0; j < partial_rows(P0); ++j)
      a.apart[((size_t)f * P0 + j) * B + b] = j == 0 ? in[f * B + b] : 0.0;
}

// ------------------------------------------------------------ launchers

template <typename R, int NX, int NU>
struct WideNewton {
  using N = NSlab<R, NX, NU>;
  using W = Wide<R, NX, NU>;
  static constexpr int kSeqSmem =
      16 * (NX * NX + NX * NU + NX + 2 * NU) * (int)sizeof(R);

  static void costate(const NewtonArgs<R>& a, cudaStream_t s, R* xst = nullptr) {
    const Plan& pl = a.plan;
    const long long B = a.B, P0 = pl.units0();
    if (pl.L >= 1) {
      kwn_costate_up0<R, NX, NU><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kCoUp0), s>>>(a);
      tree<true>(a, 1, s);
    }
    kwn_costate_down0<R, NX, NU><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kCoDown0), s>>>(a, xst);
  }

  template <bool kRev>
  static void tree(const NewtonArgs<R>& a, int gate, cudaStream_t s, int xbuf = -1) {
    const Plan& pl = a.plan;
    const long long B = a.B;
    const int sm = W::smem(N::kTree);
    for (int l = 1; l < pl.L; ++l)
      kwn_tree_up<R, NX, NU, kRev><<<W::grid(pl.n[l + 1] * B), 32 * kWarpsPerBlock, sm, s>>>(a, l, gate);
    kwn_tree_top<R, NX, NU, kRev><<<W::grid(B), 32 * kWarpsPerBlock, sm, s>>>(a, gate, xbuf);
    for (int l = pl.L - 1; l >= 1; --l)
      kwn_tree_down<R, NX, NU, kRev><<<W::grid(pl.n[l + 1] * B), 32 * kWarpsPerBlock, sm, s>>>(a, l, gate);
  }

  // candidate rollout as an exact affine scan (tree plans), sequential
  // fallback for problems whose scan met a non-finite state
  template <int kMode>
  static void scan(const NewtonArgs<R>& a, const R* dU, cudaStream_t s) {
    const long long B = a.B, P0 = a.plan.units0();
    kwn_roll_up0<R, NX, NU, kMode><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kRollUp0), s>>>(a, dU);
    tree<false>(a, kMode == 1 ? 2 : 0, s, kMode == 1 ? -1 : 0);
    kwn_roll_down0<R, NX, NU, kMode><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kRollDown0), s>>>(a, dU);
    kwn_rollout_seq<R, NX, NU, kMode><<<(unsigned)B, 32, kSeqSmem, s>>>(a, dU, 1);
  }

  static void rollout_scan(const NewtonArgs<R>& a, const R* dU, cudaStream_t s) {
    scan<1>(a, dU, s);
  }

  static void cost_partials(const NewtonArgs<R>& a, int which, cudaStream_t s) {
    kwn_cost_partials<R, NX, NU><<<W::grid((long long)a.plan.units0() * a.B), 32 * kWarpsPerBlock,
                                   W::smem(N::kCost), s>>>(a, which);
  }

  static void rollout_seq(const NewtonArgs<R>& a, const R* dU, cudaStream_t s) {
    kwn_rollout_seq<R, NX, NU, 1><<<(unsigned)a.B, 32, kSeqSmem, s>>>(a, dU, 0);
  }

  // One phase of a time-sharded iteration (include/pintoc_b200.h
  // ptc_solver_block_phase); the caller exchanges `out` between ranks.
  template <class LqrBlock>
  static void block_phase(const NewtonArgs<R>& a, const LqrArgs<R>& la, LqrBlock lqr_block,
                          int phase, const void* in, void* out, int rank, int world,
                          cudaStream_t s) {
    const Plan& pl = a.plan;
    const long long B = a.B, P0 = pl.units0();
    const int tb = W::smem(N::kTree);
    const dim3 g1 = W::grid(B);
    const unsigned gB = (unsigned)((B + 127) / 128);
    const bool fold = partial_rows((int)P0) < (int)P0;
    constexpr int kOpsRed = RED_SUM | (RED_SUM << 2) | (RED_MAX << 4);
    constexpr int kOpsCost = RED_SUM | (RED_SUM << 2) | (RED_FIRST << 4);
    LqrArgs<R> l2 = la;
    l2.prestaged = (la.xst && B == 1) ? 1 : 0;
    l2.gains_in_gst = l2.prestaged;
    R* o = static_cast<R*>(out);
    const R* gin = static_cast<const R*>(in);
    const double* din = static_cast<const double*>(in);
    double* dout = static_cast<double*>(out);
    auto up_levels = [&](auto kRevTag, int gate) {
      constexpr bool kRev = decltype(kRevTag)::value;
      for (int l = 1; l < pl.L; ++l)
        kwn_tree_up<R, NX, NU, kRev><<<W::grid(pl.n[l + 1] * B), 32 * kWarpsPerBlock, tb, s>>>(a, l, gate);
      kwn_tree_block<R, NX, NU, kRev><<<g1, 32 * kWarpsPerBlock, tb, s>>>(a, o, gate);
    };
    auto down_levels = [&](auto kRevTag, int gate) {
      constexpr bool kRev = decltype(kRevTag)::value;
      kwn_blk_carry<R, NX, NU, kRev><<<g1, 32 * kWarpsPerBlock, tb, s>>>(a, gin, rank, world, gate);
      kwn_tree_top<R, NX, NU, kRev><<<g1, 32 * kWarpsPerBlock, tb, s>>>(a, gate, -1);
      for (int l = pl.L - 1; l >= 1; --l)
        kwn_tree_down<R, NX, NU, kRev><<<W::grid(pl.n[l + 1] * B), 32 * kWarpsPerBlock, tb, s>>>(a, l, gate);
    };
    using Rev = std::true_type;
    using Fwd = std::false_type;
    switch (phase) {
      case 0:
        cudaMemsetAsync(a.n_running, 0, sizeof(int), s);
        kwn_cost_partials<R, NX, NU><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kCost), s>>>(a, 0);
        kwn_costate_up0<R, NX, NU><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kCoUp0), s>>>(a);
        up_levels(Rev{}, 1);
        break;
      case 1:
        down_levels(Rev{}, 1);
        kwn_costate_down0<R, NX, NU><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kCoDown0), s>>>(
            a, l2.prestaged ? la.xst : nullptr);
        lqr_block(&l2, 0, nullptr, out, rank, world, s);
        break;
      case 2:
        lqr_block(&l2, 1, in, out, rank, world, s);
        break;
      case 3:
        lqr_block(&l2, 2, in, nullptr, rank, world, s);
        if (fold) k_reduce_partials<<<(unsigned)B, 256, 0, s>>>(a.red, 3, kOpsRed, (int)P0, (int)B);
        k_blk_export_red<R><<<gB, 128, 0, s>>>(a, dout);
        break;
      case 4:
        k_blk_import_red<R><<<gB, 128, 0, s>>>(a, din);
        k_roll_gate<R><<<gB, 128, 0, s>>>(a);
        kwn_roll_up0<R, NX, NU, 1><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kRollUp0), s>>>(a, la.dU);
        up_levels(Fwd{}, 2);
        break;
      case 5:
        down_levels(Fwd{}, 2);
        kwn_roll_down0<R, NX, NU, 1><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kRollDown0), s>>>(a, la.dU);
        kwn_cost_partials<R, NX, NU><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kCost), s>>>(a, 1);
        if (fold) {
          k_reduce_partials<<<(unsigned)B, 256, 0, s>>>(a.cpart[0], 3, kOpsCost, (int)P0, (int)B);
          k_reduce_partials<<<(unsigned)B, 256, 0, s>>>(a.cpart[1], 3, kOpsCost, (int)P0, (int)B);
        }
        k_blk_export_cost<R, NX><<<gB, 128, 0, s>>>(a, dout);
        break;
      case 6:
        k_blk_import_cost<R><<<gB, 128, 0, s>>>(a, din);
        k_control<R, NX, NU><<<gB, 128, 0, s>>>(a);
        k_round_end<R, NX, NU><<<(unsigned)((P0 * B + 127) / 128), 128, 0, s>>>(a);
        if (fold && a.apart && a.opt.method == METHOD_ADMM)
          k_reduce_partials<<<(unsigned)B, 256, 0, s>>>(a.apart, 2, RED_MAX | (RED_MAX << 2), (int)P0, (int)B);
        k_blk_export_apart<R><<<gB, 128, 0, s>>>(a, dout);
        break;
      case 7:
        k_blk_import_apart<R><<<gB, 128, 0, s>>>(a, din);
        k_outer<R><<<gB, 128, 0, s>>>(a);
        break;
      case 8:
        cudaMemsetAsync(a.bad_index, 0xff, sizeof(int) * B, s);
        kwn_roll_up0<R, NX, NU, 0><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kRollUp0), s>>>(a, nullptr);
        up_levels(Fwd{}, 0);
        break;
      case 9:
        down_levels(Fwd{}, 0);
        kwn_roll_down0<R, NX, NU, 0><<<W::grid(P0 * B), 32 * kWarpsPerBlock, W::smem(N::kRollDown0), s>>>(a, nullptr);
        break;
      default:
        break;
    }
  }

  // problem.py `rollout`: the affine scan on tree plans with the log-depth
  // rollout enabled (sequential recurrence for problems it flags), else the
  // warp-per-problem recurrence
  static void rollout_inplace(const NewtonArgs<R>& a, cudaStream_t s) {
    if (a.pr_iters > 0 && a.plan.L >= 1) {
      cudaMemsetAsync(a.rstate, 0, sizeof(int) * a.B, s);
      scan<0>(a, nullptr, s);
    } else {
      kwn_rollout_seq<R, NX, NU, 0><<<(unsigned)a.B, 32, kSeqSmem, s>>>(a, nullptr, 0);
    }
  }
};

}  // namespace ptc
