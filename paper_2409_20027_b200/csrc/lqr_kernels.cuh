// LQR subproblem kernels: blocked reverse scan over value elements (Alg. 2)
// and blocked forward scan over closed-loop affine maps (Alg. 3).
//
// Scan structure:
//   up-sweep   level 0: each thread folds K0 consecutive stages into one
//              aggregate (each stage combined in Woodbury form,
//              vcombine_stage, so the dual elements never touch HBM);
//              level l: each thread folds K aggregates of level l.
//   top        one thread per problem walks the <= K top items.
//   down-sweep level l: carries flow back down; at level 0 the carry is the
//              cost-to-go (S_{t+1}, s_{t+1}) and the thread sweeps its chunk
//              with the Riccati-form step (riccati_step), emitting the gains
//              and (fused) the level-1 aggregates of the propagation scan.
// With K0 >= T (large batches) the tree vanishes and every problem is one
// sequential sweep per pass -- the work-optimal schedule when the batch
// alone fills the GPU.
#pragma once

#include <cooperative_groups.h>

#include "elements.cuh"

namespace ptc {

template <typename R>
struct LqrArgs {
  int B, T;
  Plan plan;
  // expansion (T rows unless noted), SoA (comp, rows, B)
  const R *P, *Rm, *M, *d, *Fx, *Fu;
  const R* PT;             // (nx*nx, 1, B)
  const double* alpha;     // [B]
  const int* status;       // [B] or null; only ST_RUNNING problems are processed
  // outputs
  R *S, *s;                // (nx*nx | nx, T+1, B), optional (null = skip)
  R *Gam, *gam;            // (nu*nx | nu, T, B)
  R *dX, *dU;              // (nx, T+1, B), (nu, T, B)
  int* flags;              // [B] OR of FLAG_*
  double* red;             // (3, P0, B): sum du^2, sum du.d, max |du|
  // time-block mode (horizon sharded across ranks, see sharded.py):
  //   t_base       global index of local stage 0 (the head element of the
  //                propagation scan, F = 0, exists only at global stage 0)
  //   no_terminal  this block does not end with the terminal element
  //   vcarry_in    (nx*nx + nx, 1, B) cost-to-go (Y, eta) entering the block
  //                from the later blocks, or null (= zero)
  //   x_in         (nx, 1, B) deviation dx at the block's first stage, or null
  //   block_mode   emit block aggregates (level-1 scratch always carved)
  int t_base, no_terminal, block_mode;
  const R* vcarry_in;
  const R* x_in;
  R* vcin_buf;             // workspace for vcarry_in   (nx*nx + nx, 1, B)
  // stage-major staging (wide kernels, batch 1, see wide.cuh): expansion
  // [t][P R M d Fx Fu] and gains [t][Gamma gamma]; `staged` = the launcher
  // has filled xst for this solve
  R* xst;
  R* gst;
  int staged;
  int prestaged;           // xst already written by the producer (Newton co-state sweep)
  int auto_plan;           // the caller left the scan plan to auto_plan (chunk0 = chunk = 0):
                           // small batches may take the one-CTA solve (k_lqr_cta)
  int gains_in_gst;        // staged: leave the gains in gst (the Newton loop reads no Gamma)
  R* xin_buf;              // workspace for x_in        (nx, 1, B)
  // tree scratch, index l = 1..L, item rows n[l]
  R* vagg[kMaxLevels + 1];
  R* vcar[kMaxLevels + 1];
  R* pagg[kMaxLevels + 1];
  R* pcar[kMaxLevels + 1];
  // wide narrow levels (kw_value_up2 / kw_value_down2): the upper half's
  // aggregate of each unit of level l (rows n[l + 1]); null where unused
  R* vhalf[kMaxLevels + 1];
};

template <typename R>
PTC_D bool lqr_skip(const LqrArgs<R>& a, int b) {
  return a.status != nullptr && a.status[b] != ST_RUNNING;
}

PTC_D int unit_id() { return blockIdx.x * blockDim.x + threadIdx.x; }

// ----------------------------------------------------------------- value up

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) k_value_up0(LqrArgs<R> a) {
  const int P0 = a.plan.units0();
  const int u = unit_id();
  if (u >= P0 * a.B) return;
  const int b = u % a.B, j = u / a.B;
  if (lqr_skip(a, b)) return;
  const int T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const R alpha = R(a.alpha[b]);
  VElem<R, NX> acc;
  Stage<R, NX, NU> st;
  R L[NU][NU];
  bool okr = true, okc = true;
  int start;
  if (j == P0 - 1 && !a.no_terminal) {
    R PT[NX][NX];
    ld_mat(a.PT, 0, 1, B, b, PT);
    velem_terminal(PT, acc);
    start = t1 - 1;
  } else {
    ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, t1 - 1, T, B, b, alpha, st);
    okr &= velem_from_stage(st, acc, L);
    start = t1 - 2;
  }
  int fl = 0;
  for (int t = start; t >= t0; --t) {
    ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, t, T, B, b, alpha, st);
    VElem<R, NX> o;
    fl |= vcombine_stage(st, acc, o);
    acc = o;
  }
  st_velem(a.vagg[1], j, a.plan.n[1], B, b, acc);
  fl |= (okr ? 0 : FLAG_DEF_R) | (okc ? 0 : FLAG_COND);
  if (fl) atomicOr(a.flags + b, fl);
}

template <typename R, int NX>
__global__ void __launch_bounds__(128) k_value_up(LqrArgs<R> a, int l) {
  const int nl = a.plan.n[l], nu = a.plan.n[l + 1];
  const int u = unit_id();
  if (u >= nu * a.B) return;
  const int b = u % a.B, j = u / a.B;
  if (lqr_skip(a, b)) return;
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  VElem<R, NX> acc;
  ld_velem(a.vagg[l], last, nl, a.B, b, acc);
  bool okc = true;
  for (int i = last - 1; i >= first; --i) {
    VElem<R, NX> e, o;
    ld_velem(a.vagg[l], i, nl, a.B, b, e);
    okc &= vcombine(e, acc, o);
    acc = o;
  }
  st_velem(a.vagg[l + 1], j, nu, a.B, b, acc);
  if (!okc) atomicOr(a.flags + b, FLAG_COND);
}

// --------------------------------------------------------------- value down

// top level: one thread per problem, zero carry beyond the terminal
template <typename R, int NX>
__global__ void __launch_bounds__(128) k_value_top(LqrArgs<R> a) {
  const int b = unit_id();
  if (b >= a.B) return;
  if (lqr_skip(a, b)) return;
  const int L = a.plan.L, nL = a.plan.n[L];
  VCarry<R, NX> c;
  if (a.vcarry_in) ld_vcarry(a.vcarry_in, 0, 1, a.B, b, c);
  else vcarry_zero(c);
  bool okc = true;
  for (int i = nL - 1; i >= 0; --i) {
    st_vcarry(a.vcar[L], i, nL, a.B, b, c);
    VElem<R, NX> e;
    ld_velem(a.vagg[L], i, nL, a.B, b, e);
    VCarry<R, NX> o;
    okc &= vstep(e, c, o);
    c = o;
  }
  if (!okc) atomicOr(a.flags + b, FLAG_COND);
}

template <typename R, int NX>
__global__ void __launch_bounds__(128) k_value_down(LqrArgs<R> a, int l) {
  const int nl = a.plan.n[l], nu = a.plan.n[l + 1];
  const int u = unit_id();
  if (u >= nu * a.B) return;
  const int b = u % a.B, j = u / a.B;
  if (lqr_skip(a, b)) return;
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  VCarry<R, NX> c;
  ld_vcarry(a.vcar[l + 1], j, nu, a.B, b, c);
  bool okc = true;
  for (int i = last; i >= first; --i) {
    st_vcarry(a.vcar[l], i, nl, a.B, b, c);
    VElem<R, NX> e;
    ld_velem(a.vagg[l], i, nl, a.B, b, e);
    VCarry<R, NX> o;
    okc &= vstep(e, c, o);
    c = o;
  }
  if (!okc) atomicOr(a.flags + b, FLAG_COND);
}

// level-0 down-sweep: cost-to-go, gains, optional (S, s) output and the
// level-1 aggregates of the forward propagation scan
// kAgg: emit the level-1 aggregates of the propagation scan (tree or block
// mode); the single-sweep schedule instantiates it without, saving registers
template <typename R, int NX, int NU, bool kAgg>
__global__ void __launch_bounds__(128) k_value_down0(LqrArgs<R> a) {
  const int P0 = a.plan.units0();
  const int u = unit_id();
  if (u >= P0 * a.B) return;
  const int b = u % a.B, j = u / a.B;
  if (lqr_skip(a, b)) return;
  const int T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const R alpha = R(a.alpha[b]);
  const bool tree = a.plan.L >= 1;
  constexpr bool emit_pagg = kAgg;
  VCarry<R, NX> c;
  if (tree) ld_vcarry(a.vcar[1], j, a.plan.n[1], B, b, c);
  else if (a.vcarry_in) ld_vcarry(a.vcarry_in, 0, 1, B, b, c);
  else vcarry_zero(c);
  if (j == P0 - 1 && a.no_terminal && a.S) {
    // block end: the cost-to-go handed in by the later blocks
    st_mat(a.S, T, T + 1, B, b, c.Y);
    R sv[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) sv[i] = -c.eta[i];
    st_vec(a.s, T, T + 1, B, b, sv);
  }
  if (j == P0 - 1 && !a.no_terminal) {
    // the terminal element V_{N+1}: Y = P_T, everything else zero
    ld_mat(a.PT, 0, 1, B, b, c.Y);
    set_zero(c.eta);
    if (a.S) {
      st_mat(a.S, T, T + 1, B, b, c.Y);
      R z[NX];
      set_zero(z);
      st_vec(a.s, T, T + 1, B, b, z);
    }
  }
  Aff<R, NX> pa;
  if constexpr (emit_pagg) aff_identity(pa);
  int fl = 0;
  // software pipeline: stage t-1 is loaded while stage t is folded
  Stage<R, NX, NU> st;
  if (t1 - 1 >= t0) ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, t1 - 1, T, B, b, alpha, st);
  for (int t = t1 - 1; t >= t0; --t) {
    Stage<R, NX, NU> nst;
    if (t > t0) ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, t - 1, T, B, b, alpha, nst);
    R Gam[NU][NX], gam[NU];
    VCarry<R, NX> o;
    fl |= riccati_step<R, NX, NU, !kAgg>(st, c, Gam, gam, o);
    st_mat(a.Gam, t, T, B, b, Gam);
    st_vec(a.gam, t, T, B, b, gam);
    if constexpr (emit_pagg) {
      Aff<R, NX> m, ao;
      if (t + a.t_base == 0) {
        set_zero(m.F);
      } else {
        mm<NX, NU, NX>(st.Fu, Gam, m.F);
#pragma unroll
        for (int i = 0; i < NX; ++i)
#pragma unroll
          for (int k = 0; k < NX; ++k) m.F[i][k] += st.Fx[i][k];
      }
      mv<NX, NU>(st.Fu, gam, m.e);
      aff_compose(pa, m, ao);
      pa = ao;
    }
    c = o;
    if (a.S) {
      st_mat(a.S, t, T + 1, B, b, c.Y);
      R sv[NX];
#pragma unroll
      for (int i = 0; i < NX; ++i) sv[i] = -c.eta[i];
      st_vec(a.s, t, T + 1, B, b, sv);
    }
    if (t > t0) st = nst;
  }
  if constexpr (emit_pagg) st_aff(a.pagg[1], j, a.plan.n[1], B, b, pa);
  if (fl) atomicOr(a.flags + b, fl);
}

// ---------------------------------------------------------- propagation scan

template <typename R, int NX>
__global__ void __launch_bounds__(128) k_prop_up(LqrArgs<R> a, int l) {
  const int nl = a.plan.n[l], nu = a.plan.n[l + 1];
  const int u = unit_id();
  if (u >= nu * a.B) return;
  const int b = u % a.B, j = u / a.B;
  if (lqr_skip(a, b)) return;
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  Aff<R, NX> acc;
  ld_aff(a.pagg[l], first, nl, a.B, b, acc);
  for (int i = first + 1; i <= last; ++i) {
    Aff<R, NX> m, o;
    ld_aff(a.pagg[l], i, nl, a.B, b, m);
    aff_compose(m, acc, o);
    acc = o;
  }
  st_aff(a.pagg[l + 1], j, nu, a.B, b, acc);
}

// level-0 up-sweep of the propagation scan for a given feedback law
// (standalone propagation_pass; inside the Newton loop this aggregate is
// produced by k_value_down0 instead)
template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) k_prop_up0(LqrArgs<R> a) {
  const int P0 = a.plan.units0();
  const int u = unit_id();
  if (u >= P0 * a.B) return;
  const int b = u % a.B, j = u / a.B;
  if (lqr_skip(a, b)) return;
  const int T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  Aff<R, NX> acc;
  aff_identity(acc);
  for (int t = t0; t < t1; ++t) {
    R Gam[NU][NX], gam[NU], Fx[NX][NX], Fu[NX][NU];
    ld_mat(a.Gam, t, T, B, b, Gam);
    ld_vec(a.gam, t, T, B, b, gam);
    ld_mat(a.Fx, t, T, B, b, Fx);
    ld_mat(a.Fu, t, T, B, b, Fu);
    Aff<R, NX> m, o;
    mm<NX, NU, NX>(Fu, Gam, m.F);
#pragma unroll
    for (int i = 0; i < NX; ++i)
#pragma unroll
      for (int k = 0; k < NX; ++k) m.F[i][k] = (t + a.t_base == 0) ? R(0) : m.F[i][k] + Fx[i][k];
    mv<NX, NU>(Fu, gam, m.e);
    aff_compose(m, acc, o);
    acc = o;
  }
  st_aff(a.pagg[1], j, a.plan.n[1], B, b, acc);
}

template <typename R, int NX>
__global__ void __launch_bounds__(128) k_prop_top(LqrArgs<R> a) {
  const int b = unit_id();
  if (b >= a.B) return;
  if (lqr_skip(a, b)) return;
  const int L = a.plan.L, nL = a.plan.n[L];
  R x[NX];
  if (a.x_in) ld_vec(a.x_in, 0, 1, a.B, b, x);
  else set_zero(x);
  for (int i = 0; i < nL; ++i) {
    st_vec(a.pcar[L], i, nL, a.B, b, x);
    Aff<R, NX> m;
    ld_aff(a.pagg[L], i, nL, a.B, b, m);
    R y[NX];
    aff_apply(m, x, y);
#pragma unroll
    for (int k = 0; k < NX; ++k) x[k] = y[k];
  }
}

template <typename R, int NX>
__global__ void __launch_bounds__(128) k_prop_down(LqrArgs<R> a, int l) {
  const int nl = a.plan.n[l], nu = a.plan.n[l + 1];
  const int u = unit_id();
  if (u >= nu * a.B) return;
  const int b = u % a.B, j = u / a.B;
  if (lqr_skip(a, b)) return;
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  R x[NX];
  ld_vec(a.pcar[l + 1], j, nu, a.B, b, x);
  for (int i = first; i <= last; ++i) {
    st_vec(a.pcar[l], i, nl, a.B, b, x);
    Aff<R, NX> m;
    ld_aff(a.pagg[l], i, nl, a.B, b, m);
    R y[NX];
    aff_apply(m, x, y);
#pragma unroll
    for (int k = 0; k < NX; ++k) x[k] = y[k];
  }
}

template <typename R, int NX, int NU>
struct PropStage {
  R Gam[NU][NX], gam[NU], Fx[NX][NX], Fu[NX][NU], dd[NU];
};

template <typename R, int NX, int NU>
PTC_D void ld_prop_stage(const LqrArgs<R>& a, int t, int b, PropStage<R, NX, NU>& p) {
  ld_mat(a.Gam, t, a.T, a.B, b, p.Gam);
  ld_vec(a.gam, t, a.T, a.B, b, p.gam);
  ld_mat(a.Fx, t, a.T, a.B, b, p.Fx);
  ld_mat(a.Fu, t, a.T, a.B, b, p.Fu);
  if (a.d && a.red) ld_vec(a.d, t, a.T, a.B, b, p.dd);  // d only feeds the partial sums
  else set_zero(p.dd);
}

// level-0 forward sweep: dx_t, du_t = Gamma_t dx_t + gamma_t and the
// per-chunk partial reductions used by the trust-region test
template <typename R, int NX, int NU, int D = 1>
__global__ void __launch_bounds__(128) k_prop_down0(LqrArgs<R> a) {
  const int P0 = a.plan.units0();
  const int u = unit_id();
  if (u >= P0 * a.B) return;
  const int b = u % a.B, j = u / a.B;
  if (lqr_skip(a, b)) return;
  const int T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  R x[NX];
  if (a.plan.L >= 1) ld_vec(a.pcar[1], j, a.plan.n[1], B, b, x);
  else if (a.x_in) ld_vec(a.x_in, 0, 1, B, b, x);
  else set_zero(x);
  double s2 = 0.0, sd = 0.0, mx = 0.0;
  // software pipeline: a register ring of D stages, stage t + D's law and
  // Jacobians loading while stage t runs
  PropStage<R, NX, NU> ring[D];
#pragma unroll
  for (int k = 0; k < D; ++k)
    if (t0 + k < t1) ld_prop_stage(a, t0 + k, b, ring[k]);
  for (int tb = t0; tb < t1; tb += D) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int t = tb + k;
      if (t >= t1) break;
      const PropStage<R, NX, NU> ps = ring[k];
      if (t + D < t1) ld_prop_stage(a, t + D, b, ring[k]);
      st_vec(a.dX, t, T + 1, B, b, x);
      R du[NU];
      mv<NU, NX>(ps.Gam, x, du);
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        du[i] += ps.gam[i];
        s2 += double(du[i]) * double(du[i]);
        sd += double(du[i]) * double(ps.dd[i]);
        mx = nanmax(mx, double(fabs(du[i])));
      }
      st_vec(a.dU, t, T, B, b, du);
      // closed loop: F = Fx + Fu Gamma (F = 0 on the head stage), e = Fu gamma
      R F[NX][NX], e[NX], y[NX];
      mm<NX, NU, NX>(ps.Fu, ps.Gam, F);
#pragma unroll
      for (int i = 0; i < NX; ++i)
#pragma unroll
        for (int k2 = 0; k2 < NX; ++k2) F[i][k2] = (t + a.t_base == 0) ? R(0) : F[i][k2] + ps.Fx[i][k2];
      mv<NX, NU>(ps.Fu, ps.gam, e);
      mv<NX, NX>(F, x, y);
#pragma unroll
      for (int i = 0; i < NX; ++i) x[i] = y[i] + e[i];
    }
  }
  if (j == P0 - 1) st_vec(a.dX, T, T + 1, B, b, x);
  if (a.red) {
    a.red[((size_t)0 * P0 + j) * B + b] = s2;
    a.red[((size_t)1 * P0 + j) * B + b] = sd;
    a.red[((size_t)2 * P0 + j) * B + b] = mx;
  }
}

// ------------------------------------- one CTA (or cluster) per problem
// Small batches (batch-1 latency, config 1): the whole LQR-scan solve of a
// problem in ONE launch.  One CTA, or a thread-block cluster of nC CTAs on
// nC SMs for longer horizons, per problem: its N = nC * P threads (powers
// of two) own contiguous chunks of the horizon; the level-0 folds are those
// of the multi-launch plan (k_value_up0 / k_value_down0 / k_prop_down0), and
// the two trees between them are Blelloch scans over the N chunk aggregates
// in shared memory -- levels that cross CTAs read and write the partner
// CTA's slots through distributed shared memory (DSMEM) -- with CTA or
// cluster barriers instead of one launch per level:
//   value (suffix): up-sweep with the parent at the left end (vcombine of
//     earlier x later), down-sweep carrying the value function after each
//     node (the right child inherits it, the left child gets
//     vstep(right child's aggregate, carry));
//   propagation (prefix): up-sweep with the parent at the right end
//     (aff_compose later o earlier), down-sweep carrying the entry state.
// Same element functions as the multi-launch plan, so the same math; the
// tree's association order differs (results agree to rounding).
template <typename R, int NX>
struct CtaSmem {
  static constexpr size_t bytes(int P) {
    return (size_t)P * (sizeof(VElem<R, NX>) + sizeof(VCarry<R, NX>));
  }
};

template <typename R, int NX, int NU, bool kCl>
__global__ void __launch_bounds__(256) k_lqr_cta(LqrArgs<R> a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  // kCl: launched as a cluster (the single-CTA instantiation carries no
  // cluster barriers or DSMEM paths: 15-20% of a T = 256 solve)
  const int nC = kCl ? (int)cl.num_blocks() : 1, rank = kCl ? (int)cl.block_rank() : 0;
  // next-stage prefetch where the registers allow a second stage in
  // flight (<= 256 bytes: nx 4 fp64 spills with it, 0.093 -> 0.118 ms at
  // T = 1024)
  constexpr bool kPre = sizeof(Stage<R, NX, NU>) <= 256;
  extern __shared__ __align__(16) unsigned char cta_smem[];
  const int P = blockDim.x;
  VElem<R, NX>* agg = reinterpret_cast<VElem<R, NX>*>(cta_smem);
  VCarry<R, NX>* car = reinterpret_cast<VCarry<R, NX>*>(cta_smem + (size_t)P * sizeof(VElem<R, NX>));
  // the propagation tree reuses the value tree's storage once it is done
  Aff<R, NX>* paf = reinterpret_cast<Aff<R, NX>*>(cta_smem);
  R(*xin)[NX] = reinterpret_cast<R(*)[NX]>(cta_smem + (size_t)P * sizeof(VElem<R, NX>));
  static_assert(sizeof(Aff<R, NX>) <= sizeof(VElem<R, NX>), "propagation aggregates reuse the value slots");
  static_assert(sizeof(R) * NX <= sizeof(VCarry<R, NX>), "entry states reuse the carry slots");
  const int b = blockIdx.x / nC;
  if (lqr_skip(a, b)) return;   // (the whole cluster: same problem)
  const int j = threadIdx.x, N = nC * P, g = rank * P + j;
  const int T = a.T, B = a.B;
  // chunk g = [floor(g T / N), floor((g + 1) T / N)): every chunk non-empty (T >= N)
  const int t0 = (int)((long long)g * T / N), t1 = (int)((long long)(g + 1) * T / N);
  // barrier after a tree level whose partners sit `dist` leaves apart
  auto level_sync = [&](int dist) {
    if (kCl && dist >= P) cl.sync();
    else __syncthreads();
  };
  const R alpha = R(a.alpha[b]);
  int fl = 0;
  bool okc = true;

  // value level 0 up: the chunk's aggregate (the last chunk ends with the terminal)
  {
    VElem<R, NX> acc;
    Stage<R, NX, NU> st;
    R L[NU][NU];
    int start;
    if (g == N - 1) {
      R PT[NX][NX];
      ld_mat(a.PT, 0, 1, B, b, PT);
      velem_terminal(PT, acc);
      start = t1 - 1;
    } else {
      ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, t1 - 1, T, B, b, alpha, st);
      if (!velem_from_stage(st, acc, L)) fl |= FLAG_DEF_R;
      start = t1 - 2;
    }
    // (stage t - 1 loads while stage t is combined)
    if (start >= t0) ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, start, T, B, b, alpha, st);
    for (int t = start; t >= t0; --t) {
      Stage<R, NX, NU> nst;
      if (kPre && t > t0) ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, t - 1, T, B, b, alpha, nst);
      VElem<R, NX> o;
      fl |= vcombine_stage(st, acc, o);
      acc = o;
      if (t > t0) {
        if (kPre) st = nst;
        else ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, t - 1, T, B, b, alpha, st);
      }
    }
    agg[j] = acc;
  }
  __syncthreads();
  // value tree, up: node g covers [g, g + 2d) (stored at its left end); a
  // partner d >= P leaves away is slot 0 of CTA rank + d / P
  for (int d = 1; d < N; d <<= 1) {
    if ((g & (2 * d - 1)) == 0) {
      const VElem<R, NX>* rp = (!kCl || d < P) ? &agg[j + d] : cl.map_shared_rank(agg, rank + d / P);
      VElem<R, NX> o;
      okc &= vcombine(agg[j], *rp, o);
      agg[j] = o;
    }
    level_sync(2 * d);
  }
  // value tree, down: car[g] = value function after the node stored at g
  if (g == 0) vcarry_zero(car[0]);
  __syncthreads();
  for (int d = N >> 1; d >= 1; d >>= 1) {
    if ((g & (2 * d - 1)) == 0) {
      const VCarry<R, NX> cn = car[j];
      VCarry<R, NX>* rc = (!kCl || d < P) ? &car[j + d] : cl.map_shared_rank(car, rank + d / P);
      const VElem<R, NX>* ra = (!kCl || d < P) ? &agg[j + d] : cl.map_shared_rank(agg, rank + d / P);
      VCarry<R, NX> o;
      okc &= vstep(*ra, cn, o);
      *rc = cn;
      car[j] = o;
    }
    level_sync(d);
  }
  // value level 0 down: gains (and S, s), the chunk's closed-loop affine map
  VCarry<R, NX> c = car[j];
  if (g == N - 1) {
    ld_mat(a.PT, 0, 1, B, b, c.Y);
    set_zero(c.eta);
    if (a.S) {
      st_mat(a.S, T, T + 1, B, b, c.Y);
      R z[NX];
      set_zero(z);
      st_vec(a.s, T, T + 1, B, b, z);
    }
  }
  Aff<R, NX> pa;
  aff_identity(pa);
  Stage<R, NX, NU> st;
  ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, t1 - 1, T, B, b, alpha, st);
  for (int t = t1 - 1; t >= t0; --t) {
    Stage<R, NX, NU> nst;
    if (kPre && t > t0) ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, t - 1, T, B, b, alpha, nst);
    R Gam[NU][NX], gam[NU];
    VCarry<R, NX> o;
    fl |= riccati_step<R, NX, NU, false>(st, c, Gam, gam, o);
    st_mat(a.Gam, t, T, B, b, Gam);
    st_vec(a.gam, t, T, B, b, gam);
    Aff<R, NX> m, ao;
    if (t == 0) {
      set_zero(m.F);
    } else {
      mm<NX, NU, NX>(st.Fu, Gam, m.F);
#pragma unroll
      for (int i = 0; i < NX; ++i)
#pragma unroll
        for (int k = 0; k < NX; ++k) m.F[i][k] += st.Fx[i][k];
    }
    mv<NX, NU>(st.Fu, gam, m.e);
    aff_compose(pa, m, ao);
    pa = ao;
    c = o;
    if (a.S) {
      st_mat(a.S, t, T + 1, B, b, c.Y);
      R sv[NX];
#pragma unroll
      for (int i = 0; i < NX; ++i) sv[i] = -c.eta[i];
      st_vec(a.s, t, T + 1, B, b, sv);
    }
    if (t > t0) {
      if (kPre) st = nst;
      else ld_stage(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, t - 1, T, B, b, alpha, st);
    }
  }
  // the value tree's storage is free: remote slots were last touched before
  // a cluster barrier every thread has passed
  __syncthreads();
  paf[j] = pa;
  __syncthreads();
  // propagation tree, up: node g covers (g - 2d, g] (stored at its right
  // end); a partner d >= P leaves back is slot P - 1 of CTA rank - d / P
  for (int d = 1; d < N; d <<= 1) {
    if (((g + 1) & (2 * d - 1)) == 0) {
      const Aff<R, NX>* rp = (!kCl || d < P) ? &paf[j - d] : cl.map_shared_rank(paf, rank - d / P) + (P - 1);
      Aff<R, NX> o;
      aff_compose(paf[j], *rp, o);
      paf[j] = o;
    }
    level_sync(2 * d);
  }
  // propagation tree, down: xin[g] = entry state of the node stored at g
  if (g == N - 1) {
#pragma unroll
    for (int i = 0; i < NX; ++i) xin[j][i] = R(0);
  }
  __syncthreads();
  for (int d = N >> 1; d >= 1; d >>= 1) {
    if (((g + 1) & (2 * d - 1)) == 0) {
      const Aff<R, NX>* rp = (!kCl || d < P) ? &paf[j - d] : cl.map_shared_rank(paf, rank - d / P) + (P - 1);
      R(*rx)[NX] = (!kCl || d < P) ? &xin[j - d] : cl.map_shared_rank(xin, rank - d / P) + (P - 1);
      R e[NX], y[NX];
#pragma unroll
      for (int i = 0; i < NX; ++i) e[i] = xin[j][i];
      aff_apply(*rp, e, y);
#pragma unroll
      for (int i = 0; i < NX; ++i) {
        (*rx)[i] = e[i];
        xin[j][i] = y[i];
      }
    }
    level_sync(d);
  }
  // propagation level 0 down: dx, du over the chunk
  R x[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) x[i] = xin[j][i];
  PropStage<R, NX, NU> ps;
  ld_prop_stage(a, t0, b, ps);
  for (int t = t0; t < t1; ++t) {
    PropStage<R, NX, NU> nps;
    if (t + 1 < t1) ld_prop_stage(a, t + 1, b, nps);
    st_vec(a.dX, t, T + 1, B, b, x);
    R du[NU];
    mv<NU, NX>(ps.Gam, x, du);
#pragma unroll
    for (int i = 0; i < NU; ++i) du[i] += ps.gam[i];
    st_vec(a.dU, t, T, B, b, du);
    R F[NX][NX], e[NX], y[NX];
    mm<NX, NU, NX>(ps.Fu, ps.Gam, F);
#pragma unroll
    for (int i = 0; i < NX; ++i)
#pragma unroll
      for (int k = 0; k < NX; ++k) F[i][k] = (t == 0) ? R(0) : F[i][k] + ps.Fx[i][k];
    mv<NX, NU>(ps.Fu, ps.gam, e);
    mv<NX, NX>(F, x, y);
#pragma unroll
    for (int i = 0; i < NX; ++i) x[i] = y[i] + e[i];
    if (t + 1 < t1) ps = nps;
  }
  if (g == N - 1) st_vec(a.dX, T, T + 1, B, b, x);
  if (!okc) fl |= FLAG_COND;
  if (fl) atomicOr(a.flags + b, fl);
}

// ------------------------------------------------------------ time blocks
// Horizon sharded into contiguous blocks, one per rank (BASELINE config 4).
// Each rank folds its block into one aggregate per scan; the aggregates are
// all-gathered (NCCL) and every rank turns the gathered list into the carry
// entering its block, then finishes its block locally.
// Gathered layout: rank-major, blocks[(r * comps + c) * B + b].

// value aggregate of the whole block: fold of the top-level items
template <typename R, int NX>
__global__ void __launch_bounds__(128) k_value_block(LqrArgs<R> a, R* out) {
  const int b = unit_id();
  if (b >= a.B) return;
  const int L = a.plan.L > 0 ? a.plan.L : 1, nL = a.plan.n[L];
  VElem<R, NX> acc;
  ld_velem(a.vagg[L], nL - 1, nL, a.B, b, acc);
  bool okc = true;
  for (int i = nL - 2; i >= 0; --i) {
    VElem<R, NX> e, o;
    ld_velem(a.vagg[L], i, nL, a.B, b, e);
    okc &= vcombine(e, acc, o);
    acc = o;
  }
  st_velem(out, 0, 1, a.B, b, acc);
  if (!okc) atomicOr(a.flags + b, FLAG_COND);
}

// cost-to-go entering block `rank`: the later blocks' aggregates applied to
// a zero carry (the last block holds the terminal element)
template <typename R, int NX>
__global__ void __launch_bounds__(128) k_value_carry(LqrArgs<R> a, const R* blocks, int rank,
                                                     int world) {
  const int b = unit_id();
  if (b >= a.B) return;
  constexpr int kC = VElem<R, NX>::kComp;
  VCarry<R, NX> c;
  vcarry_zero(c);
  bool okc = true;
  for (int r = world - 1; r > rank; --r) {
    VElem<R, NX> e;
    ld_velem(blocks + (size_t)r * kC * a.B, 0, 1, a.B, b, e);
    VCarry<R, NX> o;
    okc &= vstep(e, c, o);
    c = o;
  }
  st_vcarry(a.vcin_buf, 0, 1, a.B, b, c);
  if (!okc) atomicOr(a.flags + b, FLAG_COND);
}

// propagation aggregate of the whole block (first item applied first)
template <typename R, int NX>
__global__ void __launch_bounds__(128) k_prop_block(LqrArgs<R> a, R* out) {
  const int b = unit_id();
  if (b >= a.B) return;
  const int L = a.plan.L > 0 ? a.plan.L : 1, nL = a.plan.n[L];
  Aff<R, NX> acc;
  ld_aff(a.pagg[L], 0, nL, a.B, b, acc);
  for (int i = 1; i < nL; ++i) {
    Aff<R, NX> m, o;
    ld_aff(a.pagg[L], i, nL, a.B, b, m);
    aff_compose(m, acc, o);
    acc = o;
  }
  st_aff(out, 0, 1, a.B, b, acc);
}

// deviation entering block `rank`: the earlier blocks' maps applied to dx_1 = 0
template <typename R, int NX>
__global__ void __launch_bounds__(128) k_prop_carry(LqrArgs<R> a, const R* blocks, int rank) {
  const int b = unit_id();
  if (b >= a.B) return;
  constexpr int kC = Aff<R, NX>::kComp;
  R x[NX];
  set_zero(x);
  for (int r = 0; r < rank; ++r) {
    Aff<R, NX> m;
    ld_aff(blocks + (size_t)r * kC * a.B, 0, 1, a.B, b, m);
    R y[NX];
    aff_apply(m, x, y);
#pragma unroll
    for (int k = 0; k < NX; ++k) x[k] = y[k];
  }
  st_vec(a.xin_buf, 0, 1, a.B, b, x);
}

}  // namespace ptc
