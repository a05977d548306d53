// Host-side launch sequences (one per pass / per Newton iteration) and the
// registry that maps (dtype, model, nx, nu) to instantiated sequences.
#pragma once

#include <algorithm>
#include <map>
#include <tuple>

#include "bulk_sweeps.cuh"
#include "newton_kernels.cuh"
#include "wide.cuh"
#include "wide_newton.cuh"

namespace ptc {

constexpr int kBlock = 128;
// Single-unit plans cost the candidate inside the forward sweep that rolls
// it out (k_forward_fused; the stage costs fill the recurrences' latency).
// Round 2 measured, per Newton iteration at 32,768 problems, T = 256: the
// pendulum's cost on 8 lanes per problem after a separate rollout 1.14 ms,
// inside the fused forward sweep 0.93 ms.

inline dim3 grid_for(long long n) { return dim3((unsigned)((n + kBlock - 1) / kBlock)); }

// Sequential-sweep kernels (one thread walks a whole unit of stages) launch
// in a single wave when the batch is small: then the step time is that of the
// most loaded SM, and 128-thread CTAs leave it with up to 1.5x the average
// (32,768 problems = 256 CTAs on 148 SMs: 108 SMs hold two, 40 hold one).
// Narrower CTAs even it out (1024 CTAs of 32: 6 or 7 per SM).
struct SeqLaunch {
  dim3 grid;
  int block;
};
inline SeqLaunch seq_launch(long long n) {
  const long long sms = sm_count();
  int best = kBlock;
  if (n <= sms * 512) {
    long long load = ((n + kBlock - 1) / kBlock + sms - 1) / sms * kBlock;
    for (int bs : {64, 32}) {
      const long long l = ((n + bs - 1) / bs + sms - 1) / sms * bs;
      if (l < load) load = l, best = bs;
    }
  }
  return {dim3((unsigned)((n + best - 1) / best)), best};
}
#define PTC_SEQ(n) seq_launch(n).grid, seq_launch(n).block

// Forward (propagation) level-0 sweep: a register ring of kPropRing stages
// in flight per thread for the thread-per-unit sizes (round 2, config 3,
// gpurun pf probe: cart-pole sweep 0.380 -> 0.302 ms, pendulum half 0.506
// -> 0.450 ms; a ring of 4 spills at nx 4 and is slower at nx 2 too).  The
// backward sweep keeps one stage in flight: its 36-word cart-pole stage
// spills at two (0.477 -> 0.937 ms).
template <int NX>
constexpr int kPropRing = NX <= 4 ? 2 : 1;
// One CTA per problem (k_lqr_cta) for the small batches of the latency
// configs: the whole LQR-scan solve in one launch, trees in shared memory.
// One CTA per problem pays off while the level-0 chunks stay short: batch 1,
// fp64 (round 2, gpurun s26/s27, ms per solve, multi-launch -> one CTA):
// nx 2 T = 256 0.040 -> 0.022, T = 1024 0.052 -> 0.028; nx 4 0.087 -> 0.068,
// 0.114 -> 0.093; fp32 nx 4 0.072 -> 0.039, 0.093 -> 0.054.  Longer horizons
// run on a thread-block cluster of up to 16 CTAs (16 SMs, trees crossing
// CTAs through DSMEM) so the chunks stay short (gpurun s31): nx 2 T = 4096
// 0.062 -> 0.037, T = 16384 0.074 -> 0.045; nx 4 0.143 -> 0.100, 0.178 ->
// 0.140; at T = 65536 (16-stage chunks) the whole-GPU tree wins (0.086 vs
// 0.143 ms), hence kCtaMaxT.
constexpr int kCtaThreads = 256;
constexpr int kCtaMaxBatch = 16;
constexpr int kCtaMaxT = 16384;
inline int pow2_floor(int v) {
  int p = 1;
  while (2 * p <= v) p <<= 1;
  return p;
}
template <typename R, int NX, int NU>
bool cta_ok(const LqrArgs<R>& a) {
  if constexpr (NX > 4) {
    return false;
  } else {
    // the pass-level / config-1 solve only: inside the Newton loop (a.red)
    // the tree's association order moved sensitive batch-1 solves (a
    // chaotic fp32 cart-pole, a user cost) past their 1e-9 / count pins
    // and the iteration's other launches kept the latency unchanged
    return a.auto_plan && a.red == nullptr && !a.block_mode && a.vcarry_in == nullptr &&
           a.x_in == nullptr && a.t_base == 0 && !a.staged && a.B <= kCtaMaxBatch && a.T >= 32 &&
           a.T <= kCtaMaxT;
  }
}
// largest cluster (16 non-portable, 8, 4, 2) the device can co-schedule with
// this kernel's shared memory
template <typename R, int NX, int NU>
int cta_max_cluster() {
  static int best = -1;
  if (best >= 0) return best;
  auto k = k_lqr_cta<R, NX, NU, true>;
  const size_t smem = CtaSmem<R, NX>::bytes(kCtaThreads);
  cudaFuncSetAttribute(k_lqr_cta<R, NX, NU, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  best = 1;
  for (int c : {16, 8, 4, 2}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(c);
    cfg.blockDim = dim3(kCtaThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) == cudaSuccess && n >= 1) {
      best = c;
      break;
    }
  }
  cudaGetLastError();
  return best;
}
template <typename R, int NX, int NU>
void launch_lqr_cta(const LqrArgs<R>& a, cudaStream_t s) {
  const int maxc = cta_max_cluster<R, NX, NU>();
  int P, nC;
  if (a.T <= kCtaThreads * 4) {
    P = pow2_floor(std::min(a.T, kCtaThreads));
    nC = 1;
  } else {
    P = kCtaThreads;
    nC = std::min(maxc, pow2_floor(a.T / kCtaThreads));
  }
  if (nC == 1) {   // a plain launch: the implicit one-CTA cluster
    k_lqr_cta<R, NX, NU, false><<<a.B, P, CtaSmem<R, NX>::bytes(P), s>>>(a);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(a.B * nC);
  cfg.blockDim = dim3(P);
  cfg.dynamicSmemBytes = CtaSmem<R, NX>::bytes(P);
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_lqr_cta<R, NX, NU, true>, a);
}

template <typename R, int NX, int NU>
void launch_lqr(const LqrArgs<R>& a, cudaStream_t s) {
  const Plan& pl = a.plan;
  const long long B = a.B, P0 = pl.units0();
  if (bulk_ok<R, NX, NU>(a)) {  // batch-filling single sweep, small stages: TMA-fed rings
    launch_lqr_bulk<R, NX, NU>(a, s);
    return;
  }
  if (cta_ok<R, NX, NU>(a)) {
    launch_lqr_cta<R, NX, NU>(a, s);
    return;
  }
  if (pl.L >= 1) {
    k_value_up0<R, NX, NU><<<PTC_SEQ(P0 * B), 0, s>>>(a);
    for (int l = 1; l < pl.L; ++l) k_value_up<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
    k_value_top<R, NX><<<grid_for(B), kBlock, 0, s>>>(a);
    for (int l = pl.L - 1; l >= 1; --l)
      k_value_down<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
  }
  if (pl.L >= 1 || a.block_mode)
    k_value_down0<R, NX, NU, true><<<PTC_SEQ(P0 * B), 0, s>>>(a);
  else
    k_value_down0<R, NX, NU, false><<<PTC_SEQ(P0 * B), 0, s>>>(a);
  if (pl.L >= 1) {
    for (int l = 1; l < pl.L; ++l) k_prop_up<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
    k_prop_top<R, NX><<<grid_for(B), kBlock, 0, s>>>(a);
    for (int l = pl.L - 1; l >= 1; --l)
      k_prop_down<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
  }
  k_prop_down0<R, NX, NU, kPropRing<NX>><<<PTC_SEQ(P0 * B), 0, s>>>(a);
}

template <typename R, int NX, int NU>
void launch_prop(const LqrArgs<R>& a, cudaStream_t s) {
  const Plan& pl = a.plan;
  const long long B = a.B, P0 = pl.units0();
  if (bulk_ok<R, NX, NU>(a)) {
    launch_prop_bulk<R, NX, NU>(a, s);
    return;
  }
  if (pl.L >= 1) {
    k_prop_up0<R, NX, NU><<<PTC_SEQ(P0 * B), 0, s>>>(a);
    for (int l = 1; l < pl.L; ++l) k_prop_up<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
    k_prop_top<R, NX><<<grid_for(B), kBlock, 0, s>>>(a);
    for (int l = pl.L - 1; l >= 1; --l)
      k_prop_down<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
  }
  k_prop_down0<R, NX, NU, kPropRing<NX>><<<PTC_SEQ(P0 * B), 0, s>>>(a);
}

// Time-block phases (horizon sharded across ranks; sharded.py drives them
// with an all-gather of the block aggregates between phases):
//   0  value up-sweep            -> block value aggregate (VElem) in `out`
//   1  carry from gathered value aggregates, value down-sweep + gains,
//      propagation up-sweep      -> block affine aggregate (Aff) in `out`
//   2  carry from gathered affine aggregates, propagation down-sweep
template <typename R, int NX, int NU>
void launch_lqr_block(const LqrArgs<R>& a0, int phase, const void* blocks, void* out, int rank,
                      int world, cudaStream_t s) {
  LqrArgs<R> a = a0;
  const Plan& pl = a.plan;
  const long long B = a.B, P0 = pl.units0();
  if (phase == 0) {
    k_value_up0<R, NX, NU><<<PTC_SEQ(P0 * B), 0, s>>>(a);
    for (int l = 1; l < pl.L; ++l) k_value_up<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
    k_value_block<R, NX><<<grid_for(B), kBlock, 0, s>>>(a, static_cast<R*>(out));
  } else if (phase == 1) {
    k_value_carry<R, NX><<<grid_for(B), kBlock, 0, s>>>(a, static_cast<const R*>(blocks), rank, world);
    a.vcarry_in = a.vcin_buf;
    if (pl.L >= 1) {
      k_value_top<R, NX><<<grid_for(B), kBlock, 0, s>>>(a);
      for (int l = pl.L - 1; l >= 1; --l)
        k_value_down<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
    }
    k_value_down0<R, NX, NU, true><<<PTC_SEQ(P0 * B), 0, s>>>(a);
    for (int l = 1; l < pl.L; ++l) k_prop_up<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
    k_prop_block<R, NX><<<grid_for(B), kBlock, 0, s>>>(a, static_cast<R*>(out));
  } else {
    k_prop_carry<R, NX><<<grid_for(B), kBlock, 0, s>>>(a, static_cast<const R*>(blocks), rank);
    a.x_in = a.xin_buf;
    if (pl.L >= 1) {
      k_prop_top<R, NX><<<grid_for(B), kBlock, 0, s>>>(a);
      for (int l = pl.L - 1; l >= 1; --l)
        k_prop_down<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
    }
    k_prop_down0<R, NX, NU, kPropRing<NX>><<<PTC_SEQ(P0 * B), 0, s>>>(a);
  }
}

template <typename R, class Dyn>
void launch_costate(const NewtonArgs<R>& a, cudaStream_t s) {
  constexpr int NX = Dyn::NX;
  if constexpr (kWideNewton<Dyn>) {
    WideNewton<R, NX, Dyn::NU>::costate(a, s);
    return;
  }
  const Plan& pl = a.plan;
  const long long B = a.B, P0 = pl.units0();
  if (pl.L >= 1) {
    k_costate_up0<R, Dyn><<<PTC_SEQ(P0 * B), 0, s>>>(a);
    for (int l = 1; l < pl.L; ++l) k_costate_up<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
    k_costate_top<R, NX><<<grid_for(B), kBlock, 0, s>>>(a);
    for (int l = pl.L - 1; l >= 1; --l)
      k_costate_down<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
  }
  k_costate_down0<R, Dyn><<<PTC_SEQ(P0 * B), 0, s>>>(a);
}

// ---------------------------------------------------------------------------
// registry (declared before the Newton sequence, which dispatches its LQR
// solve through it so Newton and LQR kernel sets compile in separate units)
// ---------------------------------------------------------------------------

struct LqrOps {
  void (*solve)(const void* args, cudaStream_t s);
  void (*propagate)(const void* args, cudaStream_t s);
  void (*block)(const void* args, int phase, const void* blocks, void* out, int rank, int world,
                cudaStream_t s);
  // element-level operations (reference passes.py value_element_init,
  // value_combine, costate_combine, rollout_combine), batched over items
  void (*velem_init)(int n, const void* const* stage, const double* alpha, void* out, int* flags,
                     cudaStream_t s);
  void (*vcombine)(int n, const void* l, const void* r, void* o, int* flags, cudaStream_t s);
  void (*affine)(int n, int kind, const void* a, const void* b, void* o, cudaStream_t s);
  void (*diagnose)(int B, int T, const void* const* stage, const double* alpha, int* out,
                   cudaStream_t s);
};

// ------------------------------------------------------- element operations

// dual value elements of stages 0..n-1 (velem_from_stage) and the boundary
// element at n (velem_terminal); out (VC, n + 1, 1), flags[t] |= DEF_R when
// R_t + alpha I fails its Cholesky
template <typename R, int NX, int NU>
__global__ void k_velem_init(int n, const R* P, const R* Rm, const R* M, const R* d, const R* Fx,
                             const R* Fu, const R* PT, const double* alpha, R* out, int* flags) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > n) return;
  VElem<R, NX> e;
  if (t == n) {
    R PTm[NX][NX];
    ld_mat(PT, 0, 1, 1, 0, PTm);
    velem_terminal(PTm, e);
  } else {
    Stage<R, NX, NU> st;
    ld_stage(P, Rm, M, d, Fx, Fu, t, n, 1, 0, R(alpha[0]), st);
    R L[NU][NU];
    if (!velem_from_stage(st, e, L)) flags[t] |= FLAG_DEF_R;
  }
  st_velem(out, t, n + 1, 1, 0, e);
}

// Which stage value_pass's gates name (passes.py:231-241, 310-320): one
// thread per problem sweeps the exact dual-form recursion (vstep over
// velem_from_stage: no factorisation of Q_t on the path, so S_{t+1} stays
// exact past a failing stage) and tests every gate.  out (int32, 3 x B):
// row 0 first t with R_t + alpha I not SPD, row 1 first t with Q_t =
// sym(Rr + Fu^T S_{t+1} Fu) not SPD (-1 = none), row 2 = 1 if some
// I + C Y was singular.  Error path only (after a flagged solve).
template <typename R, int NX, int NU>
__global__ void k_lqr_diagnose(int B, int T, const R* P, const R* Rm, const R* M, const R* d,
                               const R* Fx, const R* Fu, const R* PT, const double* alpha,
                               int* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  VCarry<R, NX> c;
  ld_mat(PT, 0, 1, B, b, c.Y);
  set_zero(c.eta);
  int first_r = -1, first_q = -1, cond = 0;
  for (int t = T - 1; t >= 0; --t) {
    Stage<R, NX, NU> st;
    ld_stage(P, Rm, M, d, Fx, Fu, t, T, B, b, R(alpha[b]), st);
    R FtS[NU][NX], Q[NU][NU];
    mtm<NU, NX, NX>(st.Fu, c.Y, FtS);
    mm<NU, NX, NU>(FtS, st.Fu, Q);
    for (int i = 0; i < NU; ++i)
      for (int j = 0; j < NU; ++j) Q[i][j] += st.Rr[i][j];
    symmetrize<NU>(Q);
    if (!cholesky<NU>(Q)) first_q = t;
    VElem<R, NX> e;
    R L[NU][NU];
    if (!velem_from_stage(st, e, L)) first_r = t;
    VCarry<R, NX> o;
    if (!vstep(e, c, o)) cond = 1;
    c = o;
  }
  out[b] = first_r;
  out[B + b] = first_q;
  out[2 * B + b] = cond;
}

// o_i = l_i (earlier) (x) r_i (later); flags[i] |= COND when I + C_l Y_r is singular
template <typename R, int NX>
__global__ void k_vcombine_n(int n, const R* l, const R* r, R* o, int* flags) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  VElem<R, NX> a, b, c;
  ld_velem(l, i, n, 1, 0, a);
  ld_velem(r, i, n, 1, 0, b);
  if (!vcombine(a, b, c)) flags[i] |= FLAG_COND;
  st_velem(o, i, n, 1, 0, c);
}

// kind 0 (rollout_combine): [F | e] maps, o = b after a;
// kind 1 (costate_combine): [df | dl | dc], a the earlier segment:
//   df = b.df a.df,  dl = a.dl + a.df^T b.dl,  dc = a.dc + a.df^T b.dc
template <typename R, int NX>
__global__ void k_affine_n(int n, int kind, const R* a, const R* b, R* o) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (kind == 0) {
    Aff<R, NX> fa, fb, fo;
    ld_aff(a, i, n, 1, 0, fa);
    ld_aff(b, i, n, 1, 0, fb);
    aff_compose(fb, fa, fo);
    st_aff(o, i, n, 1, 0, fo);
    return;
  }
  R Fa[NX][NX], Fb[NX][NX], Fo[NX][NX], la[NX], lb[NX], ca[NX], cb[NX], tl[NX], tc[NX];
  ld_mat(a, i, n, 1, 0, Fa);
  ld_mat(b, i, n, 1, 0, Fb);
  ld_vec(a, i, n, 1, 0, la, NX * NX);
  ld_vec(b, i, n, 1, 0, lb, NX * NX);
  ld_vec(a, i, n, 1, 0, ca, NX * NX + NX);
  ld_vec(b, i, n, 1, 0, cb, NX * NX + NX);
  mm<NX, NX, NX>(Fb, Fa, Fo);
  mtv<NX, NX>(Fa, lb, tl);
  mtv<NX, NX>(Fa, cb, tc);
#pragma unroll
  for (int k = 0; k < NX; ++k) {
    tl[k] += la[k];
    tc[k] += ca[k];
  }
  st_mat(o, i, n, 1, 0, Fo);
  st_vec(o, i, n, 1, 0, tl, NX * NX);
  st_vec(o, i, n, 1, 0, tc, NX * NX + NX);
}

struct NewtonOps {
  void (*lqr)(const void* la, cudaStream_t s);
  void (*init)(const void* na, cudaStream_t s);
  void (*check)(const void* na, int* bad_t, cudaStream_t s);
  void (*iterate)(const void* na, const void* la, cudaStream_t s);
  void (*expand)(const void* na, cudaStream_t s);
  void (*rollout)(const void* na, cudaStream_t s);
  void (*cost)(const void* na, cudaStream_t s);
  // time-block phase (null: the model has no block mode)
  void (*block)(const void* na, const void* la, int phase, const void* in, void* out, int rank,
                int world, cudaStream_t s);
  int user_cost;   // the model carries its own cost (NewtonArgs::uterm)
};

using LqrKey = std::tuple<int, int, int>;            // dtype, nx, nu
using NewtonKey = std::tuple<int, int, int, int>;    // dtype, dyn, nx, nu

std::map<LqrKey, LqrOps>& lqr_registry();
std::map<NewtonKey, NewtonOps>& newton_registry();

template <typename R>
constexpr int dtype_code() { return sizeof(R) == 8 ? 1 : 0; }

template <typename R, class Dyn>
void launch_newton_iteration(const NewtonArgs<R>& a, const LqrArgs<R>& la, cudaStream_t s) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  const long long B = a.B, P0 = a.plan.units0();
  cudaMemsetAsync(a.n_running, 0, sizeof(int), s);
  if constexpr (kWideNewton<Dyn>) WideNewton<R, NX, NU>::cost_partials(a, 0, s);
  else k_cost_partials<R, NX, NU, Dyn><<<PTC_SEQ(P0 * B), 0, s>>>(a, 0);
  bool fused = false, forward = false;
  if constexpr (NX < 8) {
    if (a.plan.L == 0) {
      // single-sweep schedule: the value sweep re-derives every stage's
      // expansion and its co-state in registers from x, u (no stored
      // expansion or co-states); one forward sweep then runs the
      // propagation (Jacobians re-derived) and the candidate rollout side
      // by side, with the rollout gate applied at its end
      k_value_fused<R, Dyn><<<PTC_SEQ(B), 0, s>>>(a, la);
      k_forward_fused<R, Dyn, true><<<PTC_SEQ(B), 0, s>>>(a, la);
      fused = forward = true;
    }
  }
  if constexpr (kWideNewton<Dyn>) {
    if (la.xst && B == 1) {
      // the co-state sweep writes the expansion straight into the wide LQR's
      // stage-major staging rows (no component-major round trip)
      LqrArgs<R> l2 = la;
      l2.prestaged = 1;
      l2.gains_in_gst = 1;
      WideNewton<R, NX, NU>::costate(a, s, la.xst);
      lqr_registry().at(LqrKey(dtype_code<R>(), NX, NU)).solve(&l2, s);
      fused = true;
    }
  }
  if (!fused) {
    launch_costate<R, Dyn>(a, s);
    lqr_registry().at(LqrKey(dtype_code<R>(), NX, NU)).solve(&la, s);
  }
  const bool fold = partial_rows((int)P0) < (int)P0;
  constexpr int kOpsRed = RED_SUM | (RED_SUM << 2) | (RED_MAX << 4);     // sum du^2, sum du.d, max |du|
  constexpr int kOpsCost = RED_SUM | (RED_SUM << 2) | (RED_FIRST << 4);  // sum l, sum c, first infeasible
  if (fold) k_reduce_partials<<<(unsigned)B, 256, 0, s>>>(a.red, 3, kOpsRed, (int)P0, (int)B);
  if (!forward) k_roll_gate<R><<<grid_for(B), kBlock, 0, s>>>(a);
  bool rolled = forward;
  if constexpr (kWideNewton<Dyn>) {
    // affine: the candidate is one exact forward scan (tree plans) or the
    // warp-per-problem recurrence
    if (a.pr_iters > 0 && a.plan.L >= 1) {
      WideNewton<R, NX, NU>::rollout_scan(a, la.dU, s);
      rolled = true;
    } else if (B <= kWarpRolloutMaxB) {
      WideNewton<R, NX, NU>::rollout_seq(a, la.dU, s);
      rolled = true;
    }
    if (rolled) WideNewton<R, NX, NU>::cost_partials(a, 1, s);
  }
  if (rolled) {
  } else if (a.pr_iters > 0 && a.plan.L >= 1) {
    // log-depth Newton rollout, sequential fallback for what did not converge
    const Plan& pl = a.plan;
    const long long nT = (long long)(a.T + 1) * B;
    k_pr_init<R, NX, NU><<<grid_for(nT), kBlock, 0, s>>>(a, la.dX, la.dU);
    // affine dynamics: the first guess x + dx already satisfies the
    // recurrence up to the LQR scan's rounding and one sweep is exact, so two
    // checks and one sweep replace the nonlinear budget (each unneeded sweep
    // is ~2(L + 1) early-exit launches in the captured iteration)
    const int iters = (IsAffine<Dyn>::value && a.pr_iters > 1) ? 1 : a.pr_iters;
    for (int k = 0; k <= iters; ++k) {
      k_pr_up0<R, Dyn><<<PTC_SEQ(P0 * B), 0, s>>>(a, k);
      if (fold) k_reduce_partials<<<(unsigned)B, 256, 0, s>>>(a.rres, 1, RED_MAX, (int)P0, (int)B);
      k_pr_check<R><<<grid_for(B), kBlock, 0, s>>>(a, k);
      if (k == iters) break;
      for (int l = 1; l < pl.L; ++l) k_pr_up<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
      k_pr_top<R, NX><<<grid_for(B), kBlock, 0, s>>>(a, k);
      for (int l = pl.L - 1; l >= 1; --l)
        k_pr_down<R, NX><<<grid_for(pl.n[l + 1] * B), kBlock, 0, s>>>(a, l);
      k_pr_down0<R, Dyn><<<PTC_SEQ(P0 * B), 0, s>>>(a, k);
    }
    k_pr_finish<R, NX><<<grid_for(nT), kBlock, 0, s>>>(a);
    k_rollout<R, Dyn, true><<<PTC_SEQ(B), 0, s>>>(a, la.dU);
    k_cost_partials<R, NX, NU, Dyn><<<PTC_SEQ(P0 * B), 0, s>>>(a, 1);
  } else if (P0 == 1) {
    // one unit per problem: the rollout also accumulates the candidate cost
    k_rollout<R, Dyn, false, true><<<PTC_SEQ(B), 0, s>>>(a, la.dU);
  } else {
    k_rollout<R, Dyn, false><<<PTC_SEQ(B), 0, s>>>(a, la.dU);
    k_cost_partials<R, NX, NU, Dyn><<<PTC_SEQ(P0 * B), 0, s>>>(a, 1);
  }
  if (fold) {
    k_reduce_partials<<<(unsigned)B, 256, 0, s>>>(a.cpart[0], 3, kOpsCost, (int)P0, (int)B);
    k_reduce_partials<<<(unsigned)B, 256, 0, s>>>(a.cpart[1], 3, kOpsCost, (int)P0, (int)B);
  }
  k_control<R, NX, NU><<<grid_for(B), kBlock, 0, s>>>(a);
  if constexpr (kUserCon<Dyn>) k_user_bad_value<R, Dyn><<<grid_for(B), kBlock, 0, s>>>(a);
  k_round_end<R, NX, NU, Dyn><<<PTC_SEQ(P0 * B), 0, s>>>(a);
  if (fold && a.apart && a.opt.method == METHOD_ADMM)
    k_reduce_partials<<<(unsigned)B, 256, 0, s>>>(a.apart, 2, RED_MAX | (RED_MAX << 2), (int)P0, (int)B);
  k_outer<R><<<grid_for(B), kBlock, 0, s>>>(a);
}

// in-place rollout of buffer 0 from its x_0 (problem.py:449 `rollout`)
template <typename R, class Dyn>
__global__ void k_rollout_inplace(NewtonArgs<R> a) {
  constexpr int NX = Dyn::NX, NU = Dyn::NU;
  const int b = unit_id();
  if (b >= a.B) return;
  R x[NX];
  ld_x(a, 0, 0, b, x);
  bool finite = true;
  for (int t = 0; t < a.T; ++t) {
    R u[NU], xn[NX];
    ld_u(a, 0, t, b, u);
    Dyn::step(*a.pp, t, b, x, u, xn);
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      if (finite && !isfinite(xn[i])) { finite = false; a.bad_index[b] = t + 1; }
      x[i] = xn[i];
    }
    st_vec(a.X, t + 1, a.T + 1, a.B, b, x);
  }
}

// total_cost of buffer parity[b] (problem.py:476), result in cur_cost[b],
// first infeasible (stage * W + row) in bad_index[b]
template <typename R, int NX, int NU>
__global__ void k_cost_finalize(NewtonArgs<R> a) {
  const int b = unit_id();
  if (b >= a.B) return;
  int bad;
  a.cur_cost[b] = finalize_cost<R, NX>(a, 0, a.parity[b], b, bad);
  a.bad_index[b] = bad;
  a.bad_value[b] = bad >= 0 ? infeasible_value<R, NX, NU>(a, a.parity[b], b, bad) : NAN;
}

template <typename R>
__global__ void k_force_phase(NewtonArgs<R> a, int ph) {
  const int b = unit_id();
  if (b >= a.B) return;
  a.status[b] = ST_RUNNING;
  a.phase[b] = ph;
}

// ---------------------------------------------------------------------------
// registry
// ---------------------------------------------------------------------------

template <typename R, int NX, int NU>
struct RegisterLqr {
  // nx >= 8: warp-cooperative kernels (wide.cuh); smaller states keep one
  // thread per scan unit with every operand in registers
  static constexpr bool kWide = NX >= 8;
  static void solve(const void* a, cudaStream_t s) {
    if constexpr (kWide) launch_lqr_wide<R, NX, NU>(*static_cast<const LqrArgs<R>*>(a), s);
    else launch_lqr<R, NX, NU>(*static_cast<const LqrArgs<R>*>(a), s);
  }
  static void propagate(const void* a, cudaStream_t s) {
    if constexpr (kWide) launch_prop_wide<R, NX, NU>(*static_cast<const LqrArgs<R>*>(a), s);
    else launch_prop<R, NX, NU>(*static_cast<const LqrArgs<R>*>(a), s);
  }
  static void block(const void* a, int phase, const void* blocks, void* out, int rank, int world,
                    cudaStream_t s) {
    if constexpr (kWide)
      launch_lqr_block_wide<R, NX, NU>(*static_cast<const LqrArgs<R>*>(a), phase, blocks, out,
                                       rank, world, s);
    else
      launch_lqr_block<R, NX, NU>(*static_cast<const LqrArgs<R>*>(a), phase, blocks, out, rank,
                                  world, s);
  }
  static void velem_init(int n, const void* const* st, const double* alpha, void* out, int* flags,
                         cudaStream_t s) {
    k_velem_init<R, NX, NU><<<grid_for(n + 1), kBlock, 0, s>>>(
        n, static_cast<const R*>(st[0]), static_cast<const R*>(st[1]),
        static_cast<const R*>(st[2]), static_cast<const R*>(st[3]), static_cast<const R*>(st[4]),
        static_cast<const R*>(st[5]), static_cast<const R*>(st[6]), alpha, static_cast<R*>(out),
        flags);
  }
  static void vcombine(int n, const void* l, const void* r, void* o, int* flags, cudaStream_t s) {
    k_vcombine_n<R, NX><<<grid_for(n), kBlock, 0, s>>>(n, static_cast<const R*>(l),
                                                         static_cast<const R*>(r),
                                                         static_cast<R*>(o), flags);
  }
  static void affine(int n, int kind, const void* a, const void* b, void* o, cudaStream_t s) {
    k_affine_n<R, NX><<<grid_for(n), kBlock, 0, s>>>(n, kind, static_cast<const R*>(a),
                                                       static_cast<const R*>(b),
                                                       static_cast<R*>(o));
  }
  static void diagnose(int B, int T, const void* const* st, const double* alpha, int* out,
                       cudaStream_t s) {
    k_lqr_diagnose<R, NX, NU><<<grid_for(B), kBlock, 0, s>>>(
        B, T, static_cast<const R*>(st[0]), static_cast<const R*>(st[1]),
        static_cast<const R*>(st[2]), static_cast<const R*>(st[3]), static_cast<const R*>(st[4]),
        static_cast<const R*>(st[5]), static_cast<const R*>(st[6]), alpha, out);
  }
  RegisterLqr() {
    lqr_registry()[LqrKey(dtype_code<R>(), NX, NU)] =
        LqrOps{&solve, &propagate, &block, &velem_init, &vcombine, &affine, &diagnose};
  }
};

template <typename R, class Dyn, int DYN>
struct RegisterNewton {
  static constexpr int NX = Dyn::NX, NU = Dyn::NU;
  static const NewtonArgs<R>& A(const void* p) { return *static_cast<const NewtonArgs<R>*>(p); }
  static void lqr(const void* la, cudaStream_t s) {
    lqr_registry().at(LqrKey(dtype_code<R>(), NX, NU)).solve(la, s);
  }
  static void init(const void* p, cudaStream_t s) {
    const NewtonArgs<R>& a = A(p);
    k_init_state<R><<<grid_for(a.B), kBlock, 0, s>>>(a);
    if (a.opt.method == METHOD_ADMM)
      k_admm_init<R, NX, NU, Dyn><<<grid_for((long long)a.T * a.B), kBlock, 0, s>>>(a);
  }
  static void check(const void* p, int* bad_t, cudaStream_t s) {
    const NewtonArgs<R>& a = A(p);
    k_check_consistent<R, Dyn><<<grid_for((long long)a.T * a.B), kBlock, 0, s>>>(a, bad_t);
  }
  static void iterate(const void* p, const void* la, cudaStream_t s) {
    launch_newton_iteration<R, Dyn>(A(p), *static_cast<const LqrArgs<R>*>(la), s);
  }
  static void expand(const void* p, cudaStream_t s) {
    const NewtonArgs<R>& a = A(p);
    k_force_phase<R><<<grid_for(a.B), kBlock, 0, s>>>(a, PH_NEED_EXP);
    launch_costate<R, Dyn>(a, s);
  }
  static void rollout(const void* p, cudaStream_t s) {
    const NewtonArgs<R>& a = A(p);
    if constexpr (kWideNewton<Dyn>) {
      if (a.B <= kWarpRolloutMaxB) {
        WideNewton<R, NX, NU>::rollout_inplace(a, s);
        return;
      }
    }
    k_rollout_inplace<R, Dyn><<<PTC_SEQ(a.B), 0, s>>>(a);
  }
  static void cost(const void* p, cudaStream_t s) {
    const NewtonArgs<R>& a = A(p);
    k_force_phase<R><<<grid_for(a.B), kBlock, 0, s>>>(a, PH_NEED_COST);
    const int P0 = a.plan.units0();
    k_cost_partials<R, NX, NU, Dyn><<<PTC_SEQ((long long)P0 * a.B), 0, s>>>(a, 0);
    if (partial_rows(P0) < P0)
      k_reduce_partials<<<(unsigned)a.B, 256, 0, s>>>(a.cpart[0], 3,
                                                      RED_SUM | (RED_SUM << 2) | (RED_FIRST << 4),
                                                      P0, a.B);
    k_cost_finalize<R, NX, NU><<<grid_for(a.B), kBlock, 0, s>>>(a);
    if constexpr (kUserCon<Dyn>) k_user_bad_value<R, Dyn><<<grid_for(a.B), kBlock, 0, s>>>(a);
  }
  static void block(const void* p, const void* la, int phase, const void* in, void* out,
                    int rank, int world, cudaStream_t s) {
    if constexpr (kWideNewton<Dyn>)
      WideNewton<R, NX, NU>::block_phase(A(p), *static_cast<const LqrArgs<R>*>(la),
                                         lqr_registry().at(LqrKey(dtype_code<R>(), NX, NU)).block,
                                         phase, in, out, rank, world, s);
  }
  RegisterNewton() {
    newton_registry()[NewtonKey(dtype_code<R>(), DYN, NX, NU)] =
        NewtonOps{&lqr, &init, &check, &iterate, &expand, &rollout, &cost,
                  kWideNewton<Dyn> ? &block : nullptr, kUserCost<Dyn> ? 1 : 0};
  }
};

}  // namespace ptc
