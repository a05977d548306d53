// Single-sweep LQR kernels fed by the TMA engine (one-dimensional bulk
// copies, cp.async.bulk) for the batch-filling schedule (no scan tree:
// K0 = T, B >= 16384 -- BASELINE config 3's headline solve).
//
// One CTA owns 128 problems (a thread each).  Each stage of those problems
// is, per scalar component of the expansion, one contiguous 1 KB row of the
// SoA batch-minor layout (field[(c * T + t) * B + b0 .. b0 + 127]); a stage slot
// in shared memory holds all the component rows the sweep reads, and a ring
// of D slots is refilled by bulk copies that complete on one mbarrier per
// slot.  The loads thus run D - 1 stages ahead of the FP64 recursion without
// holding a stage's ~40 operands in registers per prefetched stage, and the
// per-component address arithmetic of the register path collapses to one
// pointer per copy.  The arithmetic is the register path's (riccati_step,
// the closed-loop forward step), so results are identical to k_value_down0
// / k_prop_down0 bit for bit.
#pragma once

#include <cstdint>
#include <cstdlib>

#include "lqr_kernels.cuh"

namespace ptc {

PTC_D uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

PTC_D void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

PTC_D void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

PTC_D void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

PTC_D void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred done;\n"
      " WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      " @!done bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy (TMA engine), completing `bytes` on `bar`
PTC_D void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// generic-proxy reads of a slot are ordered before the async-proxy refill
PTC_D void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int kBulkTile = 128;  // problems per CTA (one thread each, TILE / 32 warps)

// Component rows a sweep stages per stage, in slot order.
template <int NX, int NU>
struct ValueRows {   // backward sweep: P, R upper triangles, M, d, Fx, Fu
  static constexpr int kP = NX * (NX + 1) / 2, kR = NU * (NU + 1) / 2, kM = NX * NU, kD = NU,
                       kFx = NX * NX, kFu = NX * NU;
  static constexpr int kN = kP + kR + kM + kD + kFx + kFu;
};

template <int NX, int NU>
struct PropRows {    // forward sweep: Fx, Fu, Gamma, gamma (+ d for the partial sums)
  static constexpr int kFx = NX * NX, kFu = NX * NU, kG = NU * NX, kg = NU, kD = NU;
  static constexpr int kN = kFx + kFu + kG + kg + kD;
};

// upper-triangle row r of an n x n matrix -> component index i * n + j
PTC_HD int upper_comp(int r, int n) {
  int i = 0;
  while (r >= n - i) {
    r -= n - i;
    ++i;
  }
  return i * n + i + r;
}

template <typename R, int NX, int NU>
PTC_D const R* value_row(const LqrArgs<R>& a, int r) {
  using V = ValueRows<NX, NU>;
  const size_t TB = (size_t)a.T * a.B;
  if (r < V::kP) return a.P + upper_comp(r, NX) * TB;
  r -= V::kP;
  if (r < V::kR) return a.Rm + upper_comp(r, NU) * TB;
  r -= V::kR;
  if (r < V::kM) return a.M + r * TB;
  r -= V::kM;
  if (r < V::kD) return a.d + r * TB;
  r -= V::kD;
  if (r < V::kFx) return a.Fx + r * TB;
  r -= V::kFx;
  return a.Fu + r * TB;
}

template <typename R, int NX, int NU>
PTC_D const R* prop_row(const LqrArgs<R>& a, int r) {
  using Pr = PropRows<NX, NU>;
  const size_t TB = (size_t)a.T * a.B;
  if (r < Pr::kFx) return a.Fx + r * TB;
  r -= Pr::kFx;
  if (r < Pr::kFu) return a.Fu + r * TB;
  r -= Pr::kFu;
  if (r < Pr::kG) return a.Gam + r * TB;
  r -= Pr::kG;
  if (r < Pr::kg) return a.gam + r * TB;
  r -= Pr::kg;
  return a.d + r * TB;
}

// Stage from a slot (mirrors ld_stage: mirrored triangles, R + alpha I)
template <typename R, int NX, int NU, int TILE>
PTC_D void slot_stage(const R* s, int lane, R alpha, Stage<R, NX, NU>& st) {
  using V = ValueRows<NX, NU>;
  int r = 0;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = i; j < NX; ++j, ++r) st.P[i][j] = st.P[j][i] = s[r * TILE + lane];
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = i; j < NU; ++j, ++r) st.Rr[i][j] = st.Rr[j][i] = s[r * TILE + lane];
#pragma unroll
  for (int i = 0; i < NU; ++i) st.Rr[i][i] += alpha;
  r = V::kP + V::kR;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NU; ++j) st.M[i][j] = s[(r + i * NU + j) * TILE + lane];
  r += V::kM;
#pragma unroll
  for (int i = 0; i < NU; ++i) st.d[i] = s[(r + i) * TILE + lane];
  r += V::kD;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) st.Fx[i][j] = s[(r + i * NX + j) * TILE + lane];
  r += V::kFx;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NU; ++j) st.Fu[i][j] = s[(r + i * NU + j) * TILE + lane];
}

// Ring refill by warp 0: lane 0 arms the slot's barrier with the stage's
// byte count, then lanes issue one bulk copy per component row (row r by
// lane r % 32), each row TILE problems long.
template <typename R, int TILE, class RowFn>
PTC_D void bulk_issue(R* ring, uint64_t* bars, int nc, int stride, int slot, int t, int b0,
                      int nb, int B, RowFn row) {
  const int lane = threadIdx.x;
  const uint32_t bytes = nb * sizeof(R);
  if (lane == 0) mbar_expect_tx(bars + slot, nc * bytes);
  __syncwarp();
  for (int r = lane; r < nc; r += 32)
    bulk_g2s(ring + ((size_t)slot * stride + r) * TILE, row(r) + (size_t)t * B + b0, bytes,
             bars + slot);
}

// Backward (value) sweep: Riccati-form steps from the terminal element,
// gains out (and the cost-to-go if S is requested).
template <typename R, int NX, int NU, int D, int TILE>
__global__ void __launch_bounds__(TILE) k_value_sweep_bulk(LqrArgs<R> a) {
  using V = ValueRows<NX, NU>;
  constexpr int NC = V::kN;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  R* ring = reinterpret_cast<R*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + (size_t)D * NC * TILE);
  const int tid = threadIdx.x, b0 = blockIdx.x * TILE, b = b0 + tid;
  const int T = a.T, B = a.B, nb = min(TILE, B - b0);
  const bool producer = tid < 32;
  if (tid == 0) {
    for (int k = 0; k < D; ++k) mbar_init(bars + k, 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto row = [&](int r) { return value_row<R, NX, NU>(a, r); };
  if (producer)
    for (int k = 0; k < D && k < T; ++k)
      bulk_issue<R, TILE>(ring, bars, NC, NC, k, T - 1 - k, b0, nb, B, row);
  const bool live = b < B && !lqr_skip(a, b);
  VCarry<R, NX> c;
  R alpha = R(0);
  if (live) {
    alpha = R(a.alpha[b]);
    ld_mat(a.PT, 0, 1, B, b, c.Y);
    set_zero(c.eta);
    if (a.S) {
      st_mat(a.S, T, T + 1, B, b, c.Y);
      R z[NX];
      set_zero(z);
      st_vec(a.s, T, T + 1, B, b, z);
    }
  }
  int fl = 0;
  for (int i = 0; i < T; ++i) {
    const int t = T - 1 - i, slot = i % D;
    mbar_wait(bars + slot, (i / D) & 1);
    if (live) {
      Stage<R, NX, NU> st;
      slot_stage<R, NX, NU, TILE>(ring + (size_t)slot * NC * TILE, tid, alpha, st);
      R Gam[NU][NX], gam[NU];
      VCarry<R, NX> o;
      fl |= riccati_step<R, NX, NU, true>(st, c, Gam, gam, o);
      st_mat(a.Gam, t, T, B, b, Gam);
      st_vec(a.gam, t, T, B, b, gam);
      c = o;
      if (a.S) {
        st_mat(a.S, t, T + 1, B, b, c.Y);
        R sv[NX];
#pragma unroll
        for (int k = 0; k < NX; ++k) sv[k] = -c.eta[k];
        st_vec(a.s, t, T + 1, B, b, sv);
      }
    }
    if (i + D < T) {
      __syncthreads();                 // every warp has read the slot
      if (producer) {
        fence_proxy_async();
        bulk_issue<R, TILE>(ring, bars, NC, NC, slot, t - D, b0, nb, B, row);
      }
    }
  }
  if (live && fl) atomicOr(a.flags + b, fl);
}

// Forward (propagation) sweep: dx_t, du_t = Gamma_t dx_t + gamma_t and the
// trust-region partial sums, from dx_0 = 0.
template <typename R, int NX, int NU, int D, int TILE>
__global__ void __launch_bounds__(TILE) k_prop_sweep_bulk(LqrArgs<R> a) {
  using Pr = PropRows<NX, NU>;
  const bool with_d = a.d && a.red;
  const int NC = with_d ? Pr::kN : Pr::kN - Pr::kD;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  R* ring = reinterpret_cast<R*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + (size_t)D * Pr::kN * TILE);
  const int tid = threadIdx.x, b0 = blockIdx.x * TILE, b = b0 + tid;
  const int T = a.T, B = a.B, nb = min(TILE, B - b0);
  const bool producer = tid < 32;
  if (tid == 0) {
    for (int k = 0; k < D; ++k) mbar_init(bars + k, 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto row = [&](int r) { return prop_row<R, NX, NU>(a, r); };
  if (producer)
    for (int k = 0; k < D && k < T; ++k)
      bulk_issue<R, TILE>(ring, bars, NC, Pr::kN, k, k, b0, nb, B, row);
  const bool live = b < B && !lqr_skip(a, b);
  R x[NX];
  set_zero(x);
  double s2 = 0.0, sd = 0.0, mx = 0.0;
  for (int t = 0; t < T; ++t) {
    const int slot = t % D;
    mbar_wait(bars + slot, (t / D) & 1);
    if (live) {
      const R* s = ring + (size_t)slot * Pr::kN * TILE;
      R Fx[NX][NX], Fu[NX][NU], Gam[NU][NX], gam[NU], dd[NU];
#pragma unroll
      for (int i = 0; i < NX; ++i)
#pragma unroll
        for (int k = 0; k < NX; ++k) Fx[i][k] = s[(i * NX + k) * TILE + tid];
#pragma unroll
      for (int i = 0; i < NX; ++i)
#pragma unroll
        for (int k = 0; k < NU; ++k) Fu[i][k] = s[(Pr::kFx + i * NU + k) * TILE + tid];
#pragma unroll
      for (int i = 0; i < NU; ++i)
#pragma unroll
        for (int k = 0; k < NX; ++k) Gam[i][k] = s[(Pr::kFx + Pr::kFu + i * NX + k) * TILE + tid];
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        gam[i] = s[(Pr::kFx + Pr::kFu + Pr::kG + i) * TILE + tid];
        dd[i] = with_d ? s[(Pr::kFx + Pr::kFu + Pr::kG + Pr::kg + i) * TILE + tid] : R(0);
      }
      st_vec(a.dX, t, T + 1, B, b, x);
      R du[NU];
      mv<NU, NX>(Gam, x, du);
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        du[i] += gam[i];
        s2 += double(du[i]) * double(du[i]);
        sd += double(du[i]) * double(dd[i]);
        mx = nanmax(mx, double(fabs(du[i])));
      }
      st_vec(a.dU, t, T, B, b, du);
      // closed loop: F = Fx + Fu Gamma (F = 0 on the head stage), e = Fu gamma
      R F[NX][NX], e[NX], y[NX];
      mm<NX, NU, NX>(Fu, Gam, F);
#pragma unroll
      for (int i = 0; i < NX; ++i)
#pragma unroll
        for (int k = 0; k < NX; ++k) F[i][k] = (t == 0) ? R(0) : F[i][k] + Fx[i][k];
      mv<NX, NU>(Fu, gam, e);
      mv<NX, NX>(F, x, y);
#pragma unroll
      for (int i = 0; i < NX; ++i) x[i] = y[i] + e[i];
    }
    if (t + D < T) {
      __syncthreads();
      if (producer) {
        fence_proxy_async();
        bulk_issue<R, TILE>(ring, bars, NC, Pr::kN, slot, t + D, b0, nb, B, row);
      }
    }
  }
  if (live) {
    st_vec(a.dX, T, T + 1, B, b, x);
    if (a.red) {
      a.red[(size_t)0 * B + b] = s2;
      a.red[(size_t)1 * B + b] = sd;
      a.red[(size_t)2 * B + b] = mx;
    }
  }
}

// Ring depth for a sweep: all CTAs of the launch resident in one wave when
// the shared memory allows it, D in [2, 8].
inline int bulk_depth(int B, size_t slot_bytes, int sms) {
  const int ctas = (B + kBulkTile - 1) / kBulkTile;   // one CTA per kBulkTile problems
  const int per_sm = std::max(1, (ctas + sms - 1) / sms);
  const size_t budget = 224u * 1024u / per_sm;   // 228 KB per SM, 1 KB reserved per CTA
  int d = (int)(budget / (slot_bytes + 8));
  return std::min(8, std::max(2, d));
}

// Whether the bulk path applies: single-sweep plan, no block mode, every
// component row 16-byte aligned (B * sizeof(R) a multiple of 16 and the
// fields 16-byte aligned).
inline int bulk_mode() {   // PTC_BULK=1 selects the ring path (read per launch)
  const char* e = std::getenv("PTC_BULK");
  return e ? std::atoi(e) : -1;
}

// Measured (scratch/bulk_probe.py and bench.py, config-3 halves, 32,768
// problems each): alone, the ring wins for small stages (pendulum, 13
// component rows: fp64 0.547 -> 0.472 ms, fp32 0.495 -> 0.456 ms) and loses
// for wide ones (cart-pole, 36 rows: fp64 0.902 -> 0.958, fp32 0.748 -> 0.932
// ms), where the register path's per-thread loads already keep the stage
// stream at 0.8-0.9 of the copy bandwidth.  In the headline step the two
// halves run concurrently and the ring's shared memory (106 KB per CTA for
// the pendulum) displaces co-resident cart-pole blocks: the step slows from
// 1.143 to 1.182 ms with the pendulum on the ring (1.246 ms with both).  The
// register path is therefore the default; PTC_BULK=1 selects the ring.
constexpr int kBulkMaxRows = 0;

template <typename R, int NX, int NU>
inline bool bulk_ok(const LqrArgs<R>& a) {
  if (bulk_mode() == 0) return false;
  if (bulk_mode() < 0 && ValueRows<NX, NU>::kN > kBulkMaxRows) return false;
  if (a.plan.L != 0 || a.block_mode || a.vcarry_in || a.x_in || a.B < 2048) return false;
  if ((a.B * sizeof(R)) % 16 != 0) return false;
  const void* ptrs[] = {a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, a.Gam, a.gam};
  for (const void* p : ptrs)
    if (!p || (reinterpret_cast<uintptr_t>(p) & 15)) return false;
  return true;
}

template <typename R, int NX, int NU, int D>
void launch_value_bulk_d(const LqrArgs<R>& a, cudaStream_t s) {
  constexpr int NC = ValueRows<NX, NU>::kN;
  const size_t smem = (size_t)D * NC * kBulkTile * sizeof(R) + D * sizeof(uint64_t);
  auto k = k_value_sweep_bulk<R, NX, NU, D, kBulkTile>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<(a.B + kBulkTile - 1) / kBulkTile, kBulkTile, smem, s>>>(a);
}

template <typename R, int NX, int NU, int D>
void launch_prop_bulk_d(const LqrArgs<R>& a, cudaStream_t s) {
  constexpr int NC = PropRows<NX, NU>::kN;
  const size_t smem = (size_t)D * NC * kBulkTile * sizeof(R) + D * sizeof(uint64_t);
  auto k = k_prop_sweep_bulk<R, NX, NU, D, kBulkTile>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<(a.B + kBulkTile - 1) / kBulkTile, kBulkTile, smem, s>>>(a);
}

inline int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// the instantiated ring depths: the largest not above bulk_depth's choice
inline int bulk_depth_rounded(int d) { return d >= 8 ? 8 : d >= 6 ? 6 : d >= 4 ? 4 : d >= 3 ? 3 : 2; }

template <typename R, int NX, int NU>
void launch_prop_bulk(const LqrArgs<R>& a, cudaStream_t s) {
  const int d = bulk_depth_rounded(
      bulk_depth(a.B, PropRows<NX, NU>::kN * kBulkTile * sizeof(R), sm_count()));
  switch (d) {
    case 2: launch_prop_bulk_d<R, NX, NU, 2>(a, s); break;
    case 3: launch_prop_bulk_d<R, NX, NU, 3>(a, s); break;
    case 4: launch_prop_bulk_d<R, NX, NU, 4>(a, s); break;
    case 6: launch_prop_bulk_d<R, NX, NU, 6>(a, s); break;
    default: launch_prop_bulk_d<R, NX, NU, 8>(a, s); break;
  }
}

template <typename R, int NX, int NU>
void launch_lqr_bulk(const LqrArgs<R>& a, cudaStream_t s) {
  const int d = bulk_depth_rounded(
      bulk_depth(a.B, ValueRows<NX, NU>::kN * kBulkTile * sizeof(R), sm_count()));
  switch (d) {
    case 2: launch_value_bulk_d<R, NX, NU, 2>(a, s); break;
    case 3: launch_value_bulk_d<R, NX, NU, 3>(a, s); break;
    case 4: launch_value_bulk_d<R, NX, NU, 4>(a, s); break;
    case 6: launch_value_bulk_d<R, NX, NU, 6>(a, s); break;
    default: launch_value_bulk_d<R, NX, NU, 8>(a, s); break;
  }
  launch_prop_bulk<R, NX, NU>(a, s);
}

}  // namespace ptc
