// Warp-cooperative LQR-scan kernels for wide states (nx >= 8).
//
// The thread-per-unit kernels of lqr_kernels.cuh keep every matrix of a
// combine in registers; at nx = 12 a value element alone is 456 words and
// the combines spill to local memory and run as one long serial chain per
// thread.  Here one WARP owns one scan unit: its operands live in a
// per-warp shared-memory slab and the 32 lanes split every product over
// output entries, every LU step over rows, every triangular solve over
// right-hand-side columns.  Same plan, same tree, same block phases, same
// arithmetic as the thread kernels (dual combine, Riccati-form level-0 step,
// affine compositions) -- only the execution mapping differs.
#pragma once

#include "lqr_kernels.cuh"

namespace ptc {

constexpr int kWarpsPerBlock = 2;

PTC_D int lane_id() { return threadIdx.x & 31; }
PTC_D int warp_unit() { return blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); }

// ------------------------------------------------------------ primitives

// Register blocking of a warp product: each lane owns a BI x BJ block of the
// output, so one k-step costs BI + BJ shared loads for BI*BJ FMAs.  The plan
// minimises per-lane work ceil(blocks / 32) * (BI*BJ + 2 (BI + BJ)) over
// divisors BI | M, BJ | N up to 6.
struct MMPlan {
  int bi, bj;
};

constexpr MMPlan mm_plan(int M, int N) {
  MMPlan best{1, 1};
  int best_cost = 1 << 30;
  for (int bi = 1; bi <= 6; ++bi) {
    if (M % bi) continue;
    for (int bj = 1; bj <= 6; ++bj) {
      if (N % bj) continue;
      const int blocks = (M / bi) * (N / bj);
      const int cost = ((blocks + 31) / 32) * (bi * bj + 2 * (bi + bj));
      if (cost < best_cost) {
        best_cost = cost;
        best = MMPlan{bi, bj};
      }
    }
  }
  return best;
}

// FP64 tensor-core product on 8x8x4 DMMA tiles (mma.sync m8n8k4 .f64):
// the warp's operands are gathered from the slab straight into fragments
// (zero padding to multiples of 8 / 4), accumulated in registers, and
// scattered back -- for nx = 12 a 12x12x12 product is 12 DMMA instructions
// and 24 shared loads per lane instead of ~72 DFMA + ~60 loads.  FP64 MMA
// peak equals the FP64 vector peak on B200; the win is issue and
// shared-memory traffic, which bound these latency-limited kernels.
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64): a: A[l/4][l%4], b: B[l%4][l/4],
// c/d: C[l/4][2 (l%4) + {0, 1}].
PTC_D void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Accumulator fragments to / from a dense M x N row-major matrix.  A 64-bit
// shared access serves a half-warp (fragment rows fr = 0..3 or 4..7) per
// wavefront; rows sit 2N words apart, and for N = 12 the c/d layout (lane
// column group fc holds columns 2fc, 2fc + 1) puts rows fr and fr + 1 on the
// same banks (2-way conflict, in the merged 128-bit form too).  The fix is
// to permute the product's columns inside each 8-column tile: MMA column n
// holds matrix column pi(n) = n ^ 1 for n >= 4 (the b fragment is gathered
// from column pi(fr) instead of fr; pi is an involution).  A lane's register
// e then holds column 2fc + (e ^ (fc >> 1)): for every store / load
// instruction the lane-to-address map changes but the register does not, and
// the half-warp covers all 32 banks.  The b-operand gathers keep their bank
// pattern (pi only permutes the columns within each half-warp).  Picked at
// compile time per N by counting bank multiplicity over a half-warp.
__host__ __device__ constexpr int frag_pi(int n, bool perm) { return perm ? (n ^ ((n >> 2) & 1)) : n; }
constexpr int frag_bank_ways(int N, bool perm) {
  int worst = 1;
  for (int half = 0; half < 2; ++half)
    for (int e = 0; e < 2; ++e) {
      int cnt[32] = {};
      for (int fr = 4 * half; fr < 4 * half + 4; ++fr)
        for (int fc = 0; fc < 4; ++fc) {
          const int j = frag_pi(2 * fc + e, perm);
          if (fr >= N || j >= N) continue;
          cnt[(2 * (fr * N + j)) & 31]++;
        }
      for (int b = 0; b < 32; ++b) worst = cnt[b] > worst ? cnt[b] : worst;
    }
  return worst;
}
template <int N>
struct FragOrder {
  static constexpr bool perm = frag_bank_ways(N, true) < frag_bank_ways(N, false);
};

// acc = D (zero outside M x N)
template <int M, int N, int MB, int NB>
PTC_D void frag_ld(double (&acc)[MB][NB][2], const double* D) {
  const int ln = lane_id();
  const int fr = ln >> 2, fc = ln & 3;
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = mb * 8 + fr, j = nb * 8 + frag_pi(2 * fc + e, FragOrder<N>::perm);
        acc[mb][nb][e] = (i < M && j < N) ? D[i * N + j] : 0.0;
      }
}

// C = acc (MODE 0), C += acc (MODE 1), C -= acc (MODE -1), inside M x N
template <int M, int N, int MODE, int MB, int NB>
PTC_D void frag_st(const double (&acc)[MB][NB][2], double* C) {
  const int ln = lane_id();
  const int fr = ln >> 2, fc = ln & 3;
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = mb * 8 + fr, j = nb * 8 + frag_pi(2 * fc + e, FragOrder<N>::perm);
        if (i < M && j < N) {
          double& c = C[i * N + j];
          if (MODE == 0) c = acc[mb][nb][e];
          else if (MODE > 0) c += acc[mb][nb][e];
          else c -= acc[mb][nb][e];
        }
      }
}

// acc (fragments of an M x N product, the c/d layout above) += sign op(A) op(B);
// LDA / LDB: row strides of the stored A / B (0: dense)
template <int M, int K, int N, bool TA, bool TB, bool NEG, int MB, int NB, int LDA = 0,
          int LDB = 0>
PTC_D void dmma_accumulate(double (&acc)[MB][NB][2], const double* A, const double* B) {
  constexpr int la = LDA ? LDA : (TA ? M : K), lb = LDB ? LDB : (TB ? K : N);
  constexpr int KB = (K + 3) / 4;
  const int ln = lane_id();
  const int fr = ln >> 2, fc = ln & 3;
#pragma unroll
  for (int kb = 0; kb < KB; ++kb) {
    const int k = kb * 4 + fc;
    double af[MB], bf[NB];
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
      const int i = mb * 8 + fr;
      af[mb] = (i < M && k < K) ? (TA ? A[k * la + i] : A[i * la + k]) : 0.0;
      if (NEG) af[mb] = -af[mb];
    }
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int j = nb * 8 + frag_pi(fr, FragOrder<N>::perm);
      bf[nb] = (j < N && k < K) ? (TB ? B[j * lb + k] : B[k * lb + j]) : 0.0;
    }
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) dmma_8x8x4(acc[mb][nb], af[mb], bf[nb]);
  }
}

// C = sym(D + op(A1) op(B1) + op(A2) op(B2)) for N x N (N <= 16): both
// products accumulate in the same fragments and the symmetrisation is done
// there with shuffles (the transposed entry of (i, j) sits in tile (nb, mb)
// of lane ((j % 8) << 2) | (pi(i % 8) >> 1), register pi(i % 8) & 1, pi the
// column order of frag_ld), so the result is stored once,
// already symmetric -- no separate w_sym pass.  D may be C.
template <int N, int K1, int K2, bool TA1, bool TB1, bool TA2, bool TB2, int LDB1 = 0>
PTC_D void w_mm2_sym_dmma(const double* A1, const double* B1, const double* A2,
                          const double* B2, const double* D, double* C) {
  constexpr int NB = (N + 7) / 8;
  const int ln = lane_id();
  const int fr = ln >> 2, fc = ln & 3;
  double acc[NB][NB][2];
  frag_ld<N, N>(acc, D);
  dmma_accumulate<N, K1, N, TA1, TB1, false, NB, NB, 0, LDB1>(acc, A1, B1);
  dmma_accumulate<N, K2, N, TA2, TB2, false>(acc, A2, B2);
  double out[NB][NB][2];
#pragma unroll
  for (int mb = 0; mb < NB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        constexpr bool kP = FragOrder<N>::perm;
        const int pr = frag_pi(fr, kP);
        const int src = (frag_pi(2 * fc + e, kP) << 2) | (pr >> 1);
        const double v0 = __shfl_sync(0xffffffffu, acc[nb][mb][0], src);
        const double v1 = __shfl_sync(0xffffffffu, acc[nb][mb][1], src);
        out[mb][nb][e] = 0.5 * (acc[mb][nb][e] + ((pr & 1) ? v1 : v0));
      }
  __syncwarp();  // every lane has read its operands (and D) before C is written
  frag_st<N, N, 0>(out, C);
  __syncwarp();
}

// C (M x N, dense) = op(A) B with B read at row stride LDB (a column block
// of a wider matrix), on DMMA
template <int M, int K, int N, bool TA, int LDB>
PTC_D void w_mm_ldb_dmma(const double* A, const double* B, double* C) {
  constexpr int MB = (M + 7) / 8, NB = (N + 7) / 8;
  double acc[MB][NB][2];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
  dmma_accumulate<M, K, N, TA, false, false, MB, NB, 0, LDB>(acc, A, B);
  __syncwarp();
  frag_st<M, N, 0>(acc, C);
  __syncwarp();
}

template <int M, int K, int N, bool TA, bool TB, int MODE>
PTC_D void w_mm_dmma(const double* A, const double* B, double* C, const double* D = nullptr) {
  constexpr int MB = (M + 7) / 8, NB = (N + 7) / 8, KB = (K + 3) / 4;
  const int ln = lane_id();
  const int fr = ln >> 2, fc = ln & 3;
  double acc[MB][NB][2];
  if constexpr (MODE == 2 || MODE == -2) {   // the accumulator starts from D (C = D +- AB)
    frag_ld<M, N>(acc, D);
  } else {
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
  }
#pragma unroll
  for (int kb = 0; kb < KB; ++kb) {
    const int k = kb * 4 + fc;
    double af[MB], bf[NB];
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
      const int i = mb * 8 + fr;
      af[mb] = (i < M && k < K) ? (TA ? A[k * M + i] : A[i * K + k]) : 0.0;
      if (MODE == -2) af[mb] = -af[mb];
    }
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int j = nb * 8 + frag_pi(fr, FragOrder<N>::perm);
      bf[nb] = (j < N && k < K) ? (TB ? B[j * K + k] : B[k * N + j]) : 0.0;
    }
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) dmma_8x8x4(acc[mb][nb], af[mb], bf[nb]);
  }
  __syncwarp();  // every lane has read its operands before C is written
  frag_st<M, N, (MODE == 1 || MODE == -1) ? MODE : 0>(acc, C);
  __syncwarp();
}

// C (MxN) = op(A) op(B); A stored row-major as (TA ? KxM : MxK), B as
// (TB ? NxK : KxN).  MODE 0: C = AB, 1: C += AB, -1: C -= AB, 2: C = D + AB,
// -2: C = D - AB (D MxN, may be C).  C must not alias A or B.  FP64 products
// with at least 48 outputs go to the tensor cores (w_mm_dmma); the rest are
// register-blocked lane products.
template <int M, int K, int N, bool TA, bool TB, int MODE, typename R>
PTC_D void w_mm(const R* A, const R* B, R* C, const R* D = nullptr) {
  if constexpr (sizeof(R) == 8 && M * N >= 48 && M >= 4 && N >= 4) {
    w_mm_dmma<M, K, N, TA, TB, MODE>(reinterpret_cast<const double*>(A),
                                     reinterpret_cast<const double*>(B),
                                     reinterpret_cast<double*>(C),
                                     reinterpret_cast<const double*>(D));
    return;
  }
  constexpr MMPlan pl = mm_plan(M, N);
  constexpr int BI = pl.bi, BJ = pl.bj, NBJ = N / BJ, NB = (M / BI) * NBJ;
  for (int blk = lane_id(); blk < NB; blk += 32) {
    const int i0 = (blk / NBJ) * BI, j0 = (blk - (blk / NBJ) * NBJ) * BJ;
    R acc[BI][BJ];
    constexpr bool kD = MODE == 2 || MODE == -2;
    if constexpr (kD) {
#pragma unroll
      for (int ii = 0; ii < BI; ++ii)
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) acc[ii][jj] = D[(i0 + ii) * N + j0 + jj];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      R av[BI], bv[BJ];
#pragma unroll
      for (int ii = 0; ii < BI; ++ii) {
        av[ii] = TA ? A[k * M + i0 + ii] : A[(i0 + ii) * K + k];
        if (MODE == -2) av[ii] = -av[ii];
      }
#pragma unroll
      for (int jj = 0; jj < BJ; ++jj) bv[jj] = TB ? B[(j0 + jj) * K + k] : B[k * N + j0 + jj];
#pragma unroll
      for (int ii = 0; ii < BI; ++ii)
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj)
          acc[ii][jj] = (k == 0 && !kD) ? av[ii] * bv[jj] : fma(av[ii], bv[jj], acc[ii][jj]);
    }
    // (D may be C: each output position is read and written by its own lane)
#pragma unroll
    for (int ii = 0; ii < BI; ++ii)
#pragma unroll
      for (int jj = 0; jj < BJ; ++jj) {
        R& c = C[(i0 + ii) * N + j0 + jj];
        if (MODE == 0 || kD) c = acc[ii][jj];
        else if (MODE > 0) c += acc[ii][jj];
        else c -= acc[ii][jj];
      }
  }
  __syncwarp();
}

// y (M) = op(A) x; A stored as (TA ? KxM : MxK).  MODE as w_mm.
template <int M, int K, bool TA, int MODE, typename R>
PTC_D void w_mv(const R* A, const R* x, R* y) {
  for (int i = lane_id(); i < M; i += 32) {
    R s = R(0);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const R av = TA ? A[k * M + i] : A[i * K + k];
      s = (k == 0) ? av * x[k] : fma(av, x[k], s);
    }
    if (MODE == 0) y[i] = s;
    else if (MODE > 0) y[i] += s;
    else y[i] -= s;
  }
  __syncwarp();
}

// A = (A + A^T) / 2 in place: lanes walk the N (N - 1) / 2 strictly-upper
// pairs (row-major), the pair's row from the quadratic offset formula
// i (2N - 1 - i) / 2 <= p (float root, corrected by one step either way)
template <int N, typename R>
PTC_D void w_sym(R* A) {
  constexpr int NP = N * (N - 1) / 2;
  constexpr float kB = float(2 * N - 1);
  for (int p = lane_id(); p < NP; p += 32) {
    int i = int((kB - sqrtf(kB * kB - 8.0f * float(p))) * 0.5f);
    int off = i * (2 * N - 1 - i) / 2;
    if (off > p) {
      --i;
      off = i * (2 * N - 1 - i) / 2;
    } else if (p >= off + (N - 1 - i)) {
      off += N - 1 - i;
      ++i;
    }
    const int j = i + 1 + (p - off);
    const R v = R(0.5) * (A[i * N + j] + A[j * N + i]);
    A[i * N + j] = v;
    A[j * N + i] = v;
  }
  __syncwarp();
}

template <int N, typename R>
PTC_D void w_copy(const R* src, R* dst) {
  for (int e = lane_id(); e < N; e += 32) dst[e] = src[e];
  __syncwarp();
}

template <int N, typename R>
PTC_D void w_fill(R* dst, R v) {
  for (int e = lane_id(); e < N; e += 32) dst[e] = v;
  __syncwarp();
}

template <int N, typename R>
PTC_D void w_identity(R* A) {
  for (int e = lane_id(); e < N * N; e += 32) A[e] = (e / N == e - (e / N) * N) ? R(1) : R(0);
  __syncwarp();
}

// LU with partial pivoting of G (NxN, in place), reciprocal pivots on the
// diagonal, the same pivot rule as lu_factor (first row of maximal |.|).
template <int N, typename R>
PTC_D bool w_lu(R* G, int* piv) {
  const int ln = lane_id();
  bool ok = true;
  // unrolled: the trailing-block extents (N - k - 1) are compile-time
  // constants, so the rank-1 update's row / column split is shifts and
  // multiplies instead of integer divisions on the dependent chain
#pragma unroll
  for (int k = 0; k < N; ++k) {
    R v = (ln >= k && ln < N) ? fabs(G[ln * N + k]) : R(-1);
    int p = (ln >= k && ln < N) ? ln : N;
    // arg-max over the candidate lanes: N <= 16 fits one half-warp (four
    // butterfly rounds), then lane 0's answer is broadcast
    constexpr int kTop = N <= 16 ? 8 : 16;
#pragma unroll
    for (int off = kTop; off > 0; off >>= 1) {
      const R ov = __shfl_xor_sync(0xffffffffu, v, off);
      const int op = __shfl_xor_sync(0xffffffffu, p, off);
      if (ov > v || (ov == v && op < p)) {
        v = ov;
        p = op;
      }
    }
    if constexpr (N <= 16) {
      v = __shfl_sync(0xffffffffu, v, 0);
      p = __shfl_sync(0xffffffffu, p, 0);
    }
    // NaN column: keep the diagonal, as lu_factor does (with NaN candidates
    // the butterfly can also end on lane 0's sentinel p = N: never a row)
    if (!(v == v) || p >= N) p = k;
    if (ln == 0) piv[k] = p;
    if (p != k)
      for (int j = ln; j < N; j += 32) {
        const R t = G[k * N + j];
        G[k * N + j] = G[p * N + j];
        G[p * N + j] = t;
      }
    __syncwarp();
    const R pv = G[k * N + k];
    ok = ok && (pv != R(0));
    const R inv = rcp_rn(pv);
    __syncwarp();
    if (ln == 0) G[k * N + k] = inv;
    for (int i = k + 1 + ln; i < N; i += 32) G[i * N + k] *= inv;
    __syncwarp();
    for (int e = ln; e < (N - k - 1) * (N - k - 1); e += 32) {
      const int i = k + 1 + e / (N - k - 1), j = k + 1 + e % (N - k - 1);
      G[i * N + j] = fma(-G[i * N + k], G[k * N + j], G[i * N + j]);
    }
    __syncwarp();
  }
  return ok;
}

// Solve G X = B (B: N x M row-major, in place); lanes own columns.
template <int N, int M, typename R>
PTC_D void w_lu_solve(const R* LU, const int* piv, R* B) {
  for (int c = lane_id(); c < M; c += 32) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int p = piv[k];
      if (p != k) {
        const R t = B[k * M + c];
        B[k * M + c] = B[p * M + c];
        B[p * M + c] = t;
      }
    }
    // the lane's column in registers: the triangular solves' dependent
    // chains run without a shared-memory round trip per row
    R x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = B[i * M + c];
#pragma unroll
    for (int i = 1; i < N; ++i)
#pragma unroll
      for (int k = 0; k < i; ++k) x[i] = fma(-LU[i * N + k], x[k], x[i]);
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
#pragma unroll
      for (int k = i + 1; k < N; ++k) x[i] = fma(-LU[i * N + k], x[k], x[i]);
      x[i] *= LU[i * N + i];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) B[i * M + c] = x[i];
  }
  __syncwarp();
}

// Solve G^T X = B (B: N x M row-major, in place) with the factors of
// w_lu(G): G^T = U^T L^T P (as lu_solve_t); lanes own columns.
template <int N, int M, typename R>
PTC_D void w_lu_solve_t(const R* LU, const int* piv, R* B) {
  for (int c = lane_id(); c < M; c += 32) {
    R x[N];  // the lane's column in registers (as w_lu_solve)
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = B[i * M + c];
#pragma unroll
    for (int i = 0; i < N; ++i) {  // U^T y = b (lower, reciprocal diagonal)
#pragma unroll
      for (int k = 0; k < i; ++k) x[i] = fma(-LU[k * N + i], x[k], x[i]);
      x[i] *= LU[i * N + i];
    }
#pragma unroll
    for (int i = N - 2; i >= 0; --i)  // L^T z = y (upper, unit diagonal)
#pragma unroll
      for (int k = i + 1; k < N; ++k) x[i] = fma(-LU[k * N + i], x[k], x[i]);
#pragma unroll
    for (int i = 0; i < N; ++i) B[i * M + c] = x[i];
#pragma unroll
    for (int k = N - 1; k >= 0; --k) {  // undo the row interchanges
      const int p = piv[k];
      if (p != k) {
        const R t = B[k * M + c];
        B[k * M + c] = B[p * M + c];
        B[p * M + c] = t;
      }
    }
  }
  __syncwarp();
}

// Small general matrices (nu <= 6): every lane factors its own register copy
// with the arithmetic of w_lu (same pivot rule, reciprocal pivots), fully
// unrolled so rows are swapped by static selects instead of local memory.
template <int N, typename R>
PTC_D bool lu_regs(R (&G)[N][N], int (&perm)[N]) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    R v = fabs(G[k][k]);
    int p = k;
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      const R vi = fabs(G[i][k]);
      if (vi > v) {
        v = vi;
        p = i;
      }
    }
    if (!(v == v)) p = k;
    perm[k] = p;
#pragma unroll
    for (int i = k + 1; i < N; ++i)
      if (i == p)
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const R t = G[k][j];
          G[k][j] = G[i][j];
          G[i][j] = t;
        }
    const R pv = G[k][k];
    ok = ok && (pv != R(0));
    const R inv = rcp_rn(pv);
    G[k][k] = inv;
#pragma unroll
    for (int i = k + 1; i < N; ++i) G[i][k] *= inv;
#pragma unroll
    for (int i = k + 1; i < N; ++i)
#pragma unroll
      for (int j = k + 1; j < N; ++j) G[i][j] = fma(-G[i][k], G[k][j], G[i][j]);
  }
  return ok;
}

// one right-hand side through the factors of lu_regs (as w_lu_solve)
template <int N, typename R>
PTC_D void lu_solve_regs(const R (&LU)[N][N], const int (&perm)[N], R (&b)[N]) {
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int i = k + 1; i < N; ++i)
      if (i == perm[k]) {
        const R t = b[k];
        b[k] = b[i];
        b[i] = t;
      }
#pragma unroll
  for (int i = 1; i < N; ++i) {
    R v = b[i];
#pragma unroll
    for (int k = 0; k < i; ++k) v = fma(-LU[i][k], b[k], v);
    b[i] = v;
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    R v = b[i];
#pragma unroll
    for (int k = i + 1; k < N; ++k) v = fma(-LU[i][k], b[k], v);
    b[i] = v * LU[i][i];
  }
}

// Small SPD matrices (nu <= 6): every lane factors its own register copy.
template <int N, typename R>
PTC_D bool w_chol_regs(const R* Q, R (&L)[N][N]) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) L[i][j] = Q[i * N + j];
  return cholesky_rsqrt<N>(L);
}

// ------------------------------------------------------------ slab layout

template <typename R, int NX, int NU>
struct WSlab {
  static constexpr int VC = 3 * NX * NX + 2 * NX;   // value element
  static constexpr int CC = NX * NX + NX;           // carry / affine map
  static constexpr int SC = NX * NX + NU * NU + NX * NU + NU + NX * NX + NX * NU;  // stage
  // stage sub-offsets
  static constexpr int sP = 0, sR = NX * NX, sM = sR + NU * NU, sd = sM + NX * NU,
                       sFx = sd + NU, sFu = sFx + NX * NX;
  // value element sub-offsets (global component order)
  static constexpr int eA = 0, eY = NX * NX, eC = 2 * NX * NX, eEta = 3 * NX * NX,
                       eB = 3 * NX * NX + NX;
  // scratch needs of the element algebra
  static constexpr int SCR_COMB = NX * NX + NX * (2 * NX + 1) + NX * (NX + 1) + NX * NX;
  static constexpr int SCR_STEP = NX * NX + NX * (NX + 1);
  static constexpr int SCR_RIC = 2 * NU * NX + NU * NU + NX * NX + NU;
  static constexpr int BASE = 5 * NU * NX + 2 * NU + 4 * NX + NU * NU;
  static constexpr int SCR_STAGE = BASE + 2 * NX * NX;
  static constexpr int SCR_VELEM = NU * (2 * NX + 1);
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  // per-kernel slab sizes (elements of R per warp; 16 pivot ints follow)
  static constexpr int kUp0 = 2 * VC + SC + mx(SCR_STAGE, mx(SCR_VELEM, NX * NX));
  static constexpr int kUp = 3 * VC + SCR_COMB;
  static constexpr int kStep = 2 * CC + VC + SCR_STEP;
  static constexpr int kDown0 = 5 * CC + SC + NU * NX + NU + SCR_RIC;
  static constexpr int kProp = 3 * CC;
  static constexpr int kPropUp0 = 3 * CC + NX * NX + NX * NU + NU * NX + NU;
  static constexpr int kPropDown0 = 2 * NX + NU + NX * NX + NX * NU + NU * NX + 2 * NU;
  static constexpr int bytes_of(int elems) { return elems * (int)sizeof(R) + 16 * (int)sizeof(int); }
};

// this warp's slab of `elems` elements (+16 pivot ints) in dynamic shared memory
template <typename R>
PTC_D R* warp_slab(int elems) {
  extern __shared__ __align__(16) unsigned char w_smem[];
  const int stride = elems * (int)sizeof(R) + 16 * (int)sizeof(int);
  return reinterpret_cast<R*>(w_smem + (threadIdx.x >> 5) * stride);
}

template <typename R>
PTC_D int* warp_piv(R* slab, int elems) {
  return reinterpret_cast<int*>(slab + elems);
}

// global <-> slab (component c of item t at f[(c * rows + t) * B + b])
template <int C, typename R>
PTC_D void w_ld(const R* f, int t, int rows, int B, int b, R* dst, int c0 = 0) {
  for (int c = lane_id(); c < C; c += 32) dst[c] = __ldg(f + ((size_t)(c0 + c) * rows + t) * B + b);
  __syncwarp();
}

// register prefetch of one component-major item (C components of item t,
// the w_ld layout): issued before the current combine, stored after it
template <typename R, int C>
struct WPrefetchItem {
  static constexpr int PER = (C + 31) / 32;
  R v[PER];
  PTC_D void load(const R* f, int t, int rows, int B, int b) {
    const int ln = lane_id();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int c = ln + 32 * k;
      v[k] = c < C ? __ldg(f + ((size_t)c * rows + t) * B + b) : R(0);
    }
  }
  PTC_D void store(R* dst) const {
    const int ln = lane_id();
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (ln + 32 * k < C) dst[ln + 32 * k] = v[k];
    __syncwarp();
  }
};

template <int C, typename R>
PTC_D void w_st(R* f, int t, int rows, int B, int b, const R* src, int c0 = 0) {
  for (int c = lane_id(); c < C; c += 32) f[((size_t)(c0 + c) * rows + t) * B + b] = src[c];
  __syncwarp();
}

template <typename R, int NX, int NU>
PTC_D void w_ld_stage(const LqrArgs<R>& a, int t, int b, R alpha, R* st) {
  using S = WSlab<R, NX, NU>;
  const int T = a.T, B = a.B;
  if (a.staged) {
    // the staging rows are authoritative (a producer may have written only them)
    const R* row = a.xst + (size_t)t * S::SC;
    for (int c = lane_id(); c < S::SC; c += 32) st[c] = row[c];
  } else {
    w_ld<NX * NX>(a.P, t, T, B, b, st + S::sP);
    w_ld<NU * NU>(a.Rm, t, T, B, b, st + S::sR);
    w_ld<NX * NU>(a.M, t, T, B, b, st + S::sM);
    w_ld<NU>(a.d, t, T, B, b, st + S::sd);
    w_ld<NX * NX>(a.Fx, t, T, B, b, st + S::sFx);
    w_ld<NX * NU>(a.Fu, t, T, B, b, st + S::sFu);
  }
  __syncwarp();
  for (int i = lane_id(); i < NU; i += 32) st[S::sR + i * NU + i] += alpha;
  __syncwarp();
}

// Register prefetch of one stage's fields: lane l holds components
// l, l+32, ... of the concatenation of up to 6 fields (each a SoA field of
// NC_f components over `rows` items).  load(t) issues the global loads for
// item t, store(dst) writes them to the slab in concatenated order -- so the
// loads of stage t-1 are in flight while stage t is being combined.
template <typename R, int N0, int N1 = 0, int N2 = 0, int N3 = 0, int N4 = 0, int N5 = 0>
struct WPrefetch {
  static constexpr int TOTAL = N0 + N1 + N2 + N3 + N4 + N5;
  static constexpr int PER = (TOTAL + 31) / 32;
  const R* p[PER];
  R v[PER];
  size_t step;
  PTC_D void init(const R* f0, const R* f1, const R* f2, const R* f3, const R* f4, const R* f5,
                  int rows, int B, int b) {
    step = (size_t)B;
    const int ln = lane_id();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      int c = ln + 32 * k;
      const R* base = nullptr;
      int comp = 0;
      if (c < N0) { base = f0; comp = c; }
      else if ((c -= N0) < N1) { base = f1; comp = c; }
      else if ((c -= N1) < N2) { base = f2; comp = c; }
      else if ((c -= N2) < N3) { base = f3; comp = c; }
      else if ((c -= N3) < N4) { base = f4; comp = c; }
      else if ((c -= N4) < N5) { base = f5; comp = c; }
      p[k] = base ? base + (size_t)comp * rows * B + b : nullptr;
    }
  }
  PTC_D void load(int t) {
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = p[k] ? __ldg(p[k] + (size_t)t * step) : R(0);
  }
  PTC_D void store(R* dst) const {
    const int ln = lane_id();
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (ln + 32 * k < TOTAL) dst[ln + 32 * k] = v[k];
    __syncwarp();
  }
};

template <typename R, int NX, int NU>
using StagePrefetch = WPrefetch<R, NX * NX, NU * NU, NX * NU, NU, NX * NX, NX * NU>;

template <typename R, int NX, int NU>
PTC_D void w_stage_prefetch_init(StagePrefetch<R, NX, NU>& pf, const LqrArgs<R>& a, int b) {
  pf.init(a.P, a.Rm, a.M, a.d, a.Fx, a.Fu, a.T, a.B, b);
}

// prefetched stage -> slab, with Rr = R + alpha I
template <typename R, int NX, int NU>
PTC_D void w_stage_store(const StagePrefetch<R, NX, NU>& pf, R alpha, R* st) {
  using S = WSlab<R, NX, NU>;
  pf.store(st);
  for (int i = lane_id(); i < NU; i += 32) st[S::sR + i * NU + i] += alpha;
  __syncwarp();
}

// Contiguous-row prefetch (staged mode): row t of a stage-major array is N
// consecutive words, so the warp's loads are fully coalesced.
template <typename R, int N>
struct WPrefetchRow {
  static constexpr int PER = (N + 31) / 32;
  const R* base;
  size_t stride;
  R v[PER];
  PTC_D void init(const R* b, size_t st) {
    base = b;
    stride = st;
  }
  PTC_D void load(int t) {
    const R* p = base + (size_t)t * stride;
    const int ln = lane_id();
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = (ln + 32 * k < N) ? p[ln + 32 * k] : R(0);
  }
  PTC_D void store(R* dst) const {
    const int ln = lane_id();
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (ln + 32 * k < N) dst[ln + 32 * k] = v[k];
    __syncwarp();
  }
};

// component c of the stage tuple [P R M d Fx Fu] at stage t (batch 1)
template <typename R, int NX, int NU>
PTC_D R stage_comp(const LqrArgs<R>& a, int c, int t) {
  using S = WSlab<R, NX, NU>;
  const size_t T = a.T;
  if (c < S::sR) return a.P[c * T + t];
  if (c < S::sM) return a.Rm[(c - S::sR) * T + t];
  if (c < S::sd) return a.M[(c - S::sM) * T + t];
  if (c < S::sFx) return a.d[(c - S::sd) * T + t];
  if (c < S::sFu) return a.Fx[(c - S::sFx) * T + t];
  return a.Fu[(c - S::sFu) * T + t];
}

// expansion (component-major, batch 1) -> xst (stage-major): 32 x 32 tiles
template <typename R, int NX, int NU>
__global__ void __launch_bounds__(256) kw_stage_in(LqrArgs<R> a) {
  constexpr int SC = WSlab<R, NX, NU>::SC;
  __shared__ R tile[32][33];
  const int c0 = blockIdx.x * 32, t0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, t = t0 + threadIdx.x;
    tile[i][threadIdx.x] = (c < SC && t < a.T) ? stage_comp<R, NX, NU>(a, c, t) : R(0);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int t = t0 + i, c = c0 + threadIdx.x;
    if (c < SC && t < a.T) a.xst[(size_t)t * SC + c] = tile[threadIdx.x][i];
  }
}

// gst (stage-major [Gamma | gamma]) -> Gamma, gamma (component-major, batch 1)
template <typename R, int NX, int NU>
__global__ void __launch_bounds__(256) kw_gains_out(LqrArgs<R> a) {
  constexpr int GC = NU * NX + NU;
  __shared__ R tile[32][33];
  const int c0 = blockIdx.x * 32, t0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int t = t0 + i, c = c0 + threadIdx.x;
    tile[threadIdx.x][i] = (c < GC && t < a.T) ? a.gst[(size_t)t * GC + c] : R(0);
  }
  __syncthreads();
  const size_t T = a.T;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, t = t0 + threadIdx.x;
    if (c < GC && t < a.T) {
      if (c < NU * NX) a.Gam[c * T + t] = tile[i][threadIdx.x];
      else a.gam[(c - NU * NX) * T + t] = tile[i][threadIdx.x];
    }
  }
}

// --------------------------------------------------------- element algebra

// dual element of a stage (velem_from_stage); returns false when Rr fails
// its Cholesky.  Uses X as scratch for Rr^-1 [M^T | Fu^T | d].
template <typename R, int NX, int NU>
PTC_D bool w_velem(const R* st, R* e, R* X) {
  using S = WSlab<R, NX, NU>;
  constexpr int W = 2 * NX + 1;  // columns of X (NU rows used)
  R L[NU][NU];
  const bool ok = w_chol_regs<NU>(st + S::sR, L);
  const int ln = lane_id();
  if (ln < W) {
    R v[NU];
#pragma unroll
    for (int i = 0; i < NU; ++i)
      v[i] = ln < NX ? st[S::sM + ln * NU + i]
                     : (ln < 2 * NX ? st[S::sFu + (ln - NX) * NU + i] : st[S::sd + i]);
    chol_solve_vec<NU>(L, v);
#pragma unroll
    for (int i = 0; i < NU; ++i) X[i * W + ln] = v[i];
  }
  __syncwarp();
  // A = Fx - Fu RiMt, Y = sym(P - M RiMt), C = sym(Fu RiFt), eta = M Rid, b = -Fu Rid
  for (int q = ln; q < NX * NX; q += 32) {
    const int i = q / NX, j = q - (q / NX) * NX;
    R fa = R(0), my = R(0), fc = R(0);
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      const R fu = st[S::sFu + i * NU + k], m = st[S::sM + i * NU + k];
      fa = (k == 0) ? fu * X[k * W + j] : fma(fu, X[k * W + j], fa);
      my = (k == 0) ? m * X[k * W + j] : fma(m, X[k * W + j], my);
      fc = (k == 0) ? fu * X[k * W + NX + j] : fma(fu, X[k * W + NX + j], fc);
    }
    e[S::eA + q] = st[S::sFx + q] - fa;
    e[S::eY + q] = st[S::sP + q] - my;
    e[S::eC + q] = fc;
  }
  for (int i = ln; i < NX; i += 32) {
    R me = R(0), fb = R(0);
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      me = (k == 0) ? st[S::sM + i * NU + k] * X[k * W + 2 * NX]
                    : fma(st[S::sM + i * NU + k], X[k * W + 2 * NX], me);
      fb = (k == 0) ? st[S::sFu + i * NU + k] * X[k * W + 2 * NX]
                    : fma(st[S::sFu + i * NU + k], X[k * W + 2 * NX], fb);
    }
    e[S::eEta + i] = me;
    e[S::eB + i] = -fb;
  }
  __syncwarp();
  w_sym<NX>(e + S::eY);
  w_sym<NX>(e + S::eC);
  return ok;
}

template <typename R, int NX, int NU>
PTC_D void w_velem_terminal(const R* PT, R* e) {
  using S = WSlab<R, NX, NU>;
  for (int q = lane_id(); q < S::VC; q += 32)
    e[q] = (q >= S::eY && q < S::eY + NX * NX) ? PT[q - S::eY] : R(0);
  __syncwarp();
}

// general combine o = l (x) r (vcombine); slab scratch G, X, Z, T1
template <typename R, int NX, int NU>
PTC_D bool w_vcombine(const R* l, const R* r, R* o, R* scr, int* piv) {
  using S = WSlab<R, NX, NU>;
  R* G = scr;
  R* X = G + NX * NX;
  R* Z = X + NX * (2 * NX + 1);
  R* T1 = Z + NX * (NX + 1);
  constexpr int WX = 2 * NX + 1, WZ = NX + 1;
  // G = I + C_l Y_r, factored once; Z uses G^T through the same factors
  // Z = G^-T [Y_r A_l | eta_r - Y_r b_l]   X = G^-1 [A_l | C_l | b_l + C_l eta_r]
  w_mm<NX, NX, NX, false, false, 0>(l + S::eC, r + S::eY, G);
  // X rhs, Z rhs (independent of the factorisation)
  for (int q = lane_id(); q < NX * WX; q += 32) {
    const int i = q / WX, j = q - (q / WX) * WX;
    if (j < NX) X[q] = l[S::eA + i * NX + j];
    else if (j < 2 * NX) X[q] = l[S::eC + i * NX + (j - NX)];
    else {
      R s = l[S::eB + i];
#pragma unroll
      for (int k = 0; k < NX; ++k) s = fma(l[S::eC + i * NX + k], r[S::eEta + k], s);
      X[q] = s;
    }
  }
  for (int q = lane_id(); q < NX * WZ; q += 32) {
    const int i = q / WZ, j = q - (q / WZ) * WZ;
    R s = R(0);
    if (j < NX) {
#pragma unroll
      for (int k = 0; k < NX; ++k)
        s = (k == 0) ? r[S::eY + i * NX] * l[S::eA + j] : fma(r[S::eY + i * NX + k], l[S::eA + k * NX + j], s);
    } else {
      R yb = R(0);
#pragma unroll
      for (int k = 0; k < NX; ++k) yb = (k == 0) ? r[S::eY + i * NX] * l[S::eB] : fma(r[S::eY + i * NX + k], l[S::eB + k], yb);
      s = r[S::eEta + i] - yb;
    }
    Z[q] = s;
  }
  for (int i = lane_id(); i < NX; i += 32) G[i * NX + i] += R(1);
  __syncwarp();
  // one factorisation serves both orientations (G^T = U^T L^T P)
  const bool ok = w_lu<NX>(G, piv);
  w_lu_solve<NX, WX>(G, piv, X);
  w_lu_solve_t<NX, WZ>(G, piv, Z);
  // Y = sym(A_l^T Z1 + Y_l), eta = A_l^T z + eta_l
  constexpr bool kFragSym = sizeof(R) == 8 && NX >= 8 && NX <= 16;
  if constexpr (kFragSym) {
    w_mm2_sym_dmma<NX, NX, 0, true, false, false, false, WZ>(
        reinterpret_cast<const double*>(l + S::eA), reinterpret_cast<const double*>(Z), nullptr,
        nullptr, reinterpret_cast<const double*>(l + S::eY), reinterpret_cast<double*>(o + S::eY));
  } else {
    for (int q = lane_id(); q < NX * NX; q += 32) {
      const int i = q / NX, j = q - (q / NX) * NX;
      R s = R(0);
#pragma unroll
      for (int k = 0; k < NX; ++k) s = (k == 0) ? l[S::eA + i] * Z[j] : fma(l[S::eA + k * NX + i], Z[k * WZ + j], s);
      o[S::eY + q] = s + l[S::eY + q];
    }
  }
  for (int i = lane_id(); i < NX; i += 32) {
    R s = R(0);
#pragma unroll
    for (int k = 0; k < NX; ++k) s = (k == 0) ? l[S::eA + i] * Z[NX] : fma(l[S::eA + k * NX + i], Z[k * WZ + NX], s);
    o[S::eEta + i] = s + l[S::eEta + i];
  }
  // A = A_r X1, T1 = A_r X2, b = A_r x + b_r
  if constexpr (kFragSym) {
    w_mm_ldb_dmma<NX, NX, NX, false, WX>(reinterpret_cast<const double*>(r + S::eA),
                                         reinterpret_cast<const double*>(X),
                                         reinterpret_cast<double*>(o + S::eA));
    w_mm_ldb_dmma<NX, NX, NX, false, WX>(reinterpret_cast<const double*>(r + S::eA),
                                         reinterpret_cast<const double*>(X + NX),
                                         reinterpret_cast<double*>(T1));
  } else {
    for (int q = lane_id(); q < NX * NX; q += 32) {
      const int i = q / NX, j = q - (q / NX) * NX;
      R s1 = R(0), s2 = R(0);
#pragma unroll
      for (int k = 0; k < NX; ++k) {
        const R ar = r[S::eA + i * NX + k];
        s1 = (k == 0) ? ar * X[j] : fma(ar, X[k * WX + j], s1);
        s2 = (k == 0) ? ar * X[NX + j] : fma(ar, X[k * WX + NX + j], s2);
      }
      o[S::eA + q] = s1;
      T1[q] = s2;
    }
  }
  for (int i = lane_id(); i < NX; i += 32) {
    R s = R(0);
#pragma unroll
    for (int k = 0; k < NX; ++k) s = (k == 0) ? r[S::eA + i * NX] * X[2 * NX] : fma(r[S::eA + i * NX + k], X[k * WX + 2 * NX], s);
    o[S::eB + i] = s + r[S::eB + i];
  }
  __syncwarp();
  // C = sym(T1 A_r^T + C_r)
  if constexpr (kFragSym) {
    w_mm2_sym_dmma<NX, NX, 0, false, true, false, false>(
        reinterpret_cast<const double*>(T1), reinterpret_cast<const double*>(r + S::eA), nullptr,
        nullptr, reinterpret_cast<const double*>(r + S::eC), reinterpret_cast<double*>(o + S::eC));
  } else {
    for (int q = lane_id(); q < NX * NX; q += 32) {
      const int i = q / NX, j = q - (q / NX) * NX;
      R s = R(0);
#pragma unroll
      for (int k = 0; k < NX; ++k) s = (k == 0) ? T1[i * NX] * r[S::eA + j * NX] : fma(T1[i * NX + k], r[S::eA + j * NX + k], s);
      o[S::eC + q] = s + r[S::eC + q];
    }
    __syncwarp();
    w_sym<NX>(o + S::eY);
    w_sym<NX>(o + S::eC);
  }
  return ok;
}

// stage (x) aggregate in Woodbury form (vcombine_stage of elements.cuh):
// st is a loaded stage, r the aggregate, o the result (o != r).  Scratch:
// the contiguous G | X | Z region and T1, T2.
template <typename R, int NX, int NU>
PTC_D int w_vcombine_stage(const R* st, const R* r, R* o, R* scr, int* piv) {
  using S = WSlab<R, NX, NU>;
  R* base = scr;
  R* RiMt = base;                 // NU x NX
  R* Rid = RiMt + NU * NX;        // NU
  R* YF = Rid + NU;               // NX x NU
  R* W = YF + NX * NU;            // NU x NX
  R* v = W + NU * NX;             // NX
  R* x = v + NX;                  // NX
  R* z = x + NX;                  // NX
  R* bl = z + NX;                 // NX
  R* AF = bl + NX;                // NX x NU
  R* Y2 = AF + NX * NU;           // NU x NX
  R* q = Y2 + NU * NX;            // NU
  R* Al = scr + S::BASE;          // NX x NX
  R* Z1 = Al + NX * NX;           // NX x NX
  const R* Fu = st + S::sFu;
  const int ln = lane_id();
  int fl = 0;
  R L[NU][NU];
  if (!w_chol_regs<NU>(st + S::sR, L)) fl |= FLAG_DEF_R;
  if (ln <= NX) {  // columns of Rr^-1 [M^T | d]
    R c[NU];
#pragma unroll
    for (int i = 0; i < NU; ++i) c[i] = ln < NX ? st[S::sM + ln * NU + i] : st[S::sd + i];
    chol_solve_vec<NU>(L, c);
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      if (ln < NX) RiMt[i * NX + ln] = c[i];
      else Rid[i] = c[i];
    }
  }
  __syncwarp();
  // A_l = Fx - Fu RiMt ;  Y_l = sym(P - M RiMt) (into o.Y) ;  YF = Y_r Fu
  w_mm<NX, NU, NX, false, false, -2>(Fu, RiMt, Al, st + S::sFx);
  // (Y_l is only accumulated into o.Y, symmetrised once at the end:
  // sym(sym(P - M RiMt) + A_l^T Z1) == sym(P - M RiMt + A_l^T Z1))
  w_mm<NX, NU, NX, false, false, -2>(st + S::sM, RiMt, o + S::eY, st + S::sP);
  w_mm<NX, NX, NU, false, false, 0>(r + S::eY, Fu, YF);
  for (int i = ln; i < NX; i += 32) {  // eta_l (into o.eta), b_l
    R me = R(0), fb = R(0);
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      me = fma(st[S::sM + i * NU + k], Rid[k], me);
      fb = fma(Fu[i * NU + k], Rid[k], fb);
    }
    o[S::eEta + i] = me;
    bl[i] = -fb;
  }
  __syncwarp();
  // Y_r A_l, and v = eta_r - Y_r b_l
  w_mm<NX, NX, NX, false, false, 0>(r + S::eY, Al, Z1);
  for (int i = ln; i < NX; i += 32) {
    R yb = R(0);
#pragma unroll
    for (int k = 0; k < NX; ++k) yb = fma(r[S::eY + i * NX + k], bl[k], yb);
    v[i] = r[S::eEta + i] - yb;
  }
  __syncwarp();
  // Q = sym(Rr + Fu^T YF) (NU x NU), warp LU in shared memory
  R* Q = q + NU;                  // NU x NU
  for (int e = ln; e < NU * NU; e += 32) {
    const int i = e / NU, j = e - (e / NU) * NU;
    R s1 = R(0), s2 = R(0);
#pragma unroll
    for (int k = 0; k < NX; ++k) {
      s1 = fma(Fu[k * NU + i], YF[k * NU + j], s1);
      s2 = fma(Fu[k * NU + j], YF[k * NU + i], s2);
    }
    Q[e] = R(0.5) * ((s1 + st[S::sR + i * NU + j]) + (s2 + st[S::sR + j * NU + i]));
  }
  // W = YF^T A_l (NU x NX), q = Fu^T v, AF = A_r Fu; then Y2 = AF^T
  w_mm<NU, NX, NX, true, false, 0>(YF, Al, W);
  w_mv<NU, NX, true, 0>(Fu, v, q);
  w_mm<NX, NX, NU, false, false, 0>(r + S::eA, Fu, AF);
  for (int e = ln; e < NU * NX; e += 32) {
    const int i = e / NX, j = e - (e / NX) * NX;
    Y2[e] = AF[j * NU + i];
  }
  __syncwarp();
  {
    // Q^-1 [W | Y2 | q]: each lane factors Q in registers and solves one of
    // the 2 NX + 1 columns (no shuffles or warp barriers inside)
    R G[NU][NU];
    int perm[NU];
#pragma unroll
    for (int i = 0; i < NU; ++i)
#pragma unroll
      for (int j = 0; j < NU; ++j) G[i][j] = Q[i * NU + j];
    if (!lu_regs<NU>(G, perm)) fl |= FLAG_COND;
    static_assert(2 * NX + 1 <= 32, "one lane per right-hand side");
    if (ln < 2 * NX + 1) {
      R* col = ln < NX ? W + ln : (ln < 2 * NX ? Y2 + (ln - NX) : q);
      const int stride = ln < 2 * NX ? NX : 1;
      R bv[NU];
#pragma unroll
      for (int i = 0; i < NU; ++i) bv[i] = col[i * stride];
      lu_solve_regs<NU>(G, perm, bv);
#pragma unroll
      for (int i = 0; i < NU; ++i) col[i * stride] = bv[i];
    }
    __syncwarp();
  }
  // Z1 = Y_r A_l - YF W ;  o.Y += A_l^T Z1 ; z = v - YF q ; x = b_l + Fu q
  w_mm<NX, NU, NX, false, false, -1>(YF, W, Z1);
  for (int i = ln; i < NX; i += 32) {
    R yq = R(0), fq = R(0);
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      yq = fma(YF[i * NU + k], q[k], yq);
      fq = fma(Fu[i * NU + k], q[k], fq);
    }
    z[i] = v[i] - yq;
    x[i] = bl[i] + fq;
  }
  __syncwarp();
  constexpr bool kFragSym = sizeof(R) == 8 && NX >= 8 && NX <= 16;
  if constexpr (kFragSym) {   // Y = sym(Y_l + A_l^T Z1), symmetrised in the fragments
    w_mm2_sym_dmma<NX, NX, 0, true, false, false, false>(
        reinterpret_cast<const double*>(Al), reinterpret_cast<const double*>(Z1), nullptr,
        nullptr, reinterpret_cast<const double*>(o + S::eY), reinterpret_cast<double*>(o + S::eY));
  } else {
    w_mm<NX, NX, NX, true, false, 1>(Al, Z1, o + S::eY);
  }
  w_mv<NX, NX, true, 1>(Al, z, o + S::eEta);
  // A = A_r (A_l - Fu W)   (A_l no longer needed as such)
  w_mm<NX, NU, NX, false, false, -1>(Fu, W, Al);
  w_mm<NX, NX, NX, false, false, 0>(r + S::eA, Al, o + S::eA);
  // C = sym(AF Y2 + C_r) ;  b = A_r x + b_r
  if constexpr (kFragSym) {   // C = sym(C_r + AF Y2)
    w_mm2_sym_dmma<NX, NU, 0, false, false, false, false>(
        reinterpret_cast<const double*>(AF), reinterpret_cast<const double*>(Y2), nullptr,
        nullptr, reinterpret_cast<const double*>(r + S::eC), reinterpret_cast<double*>(o + S::eC));
  } else {
    w_mm<NX, NU, NX, false, false, 2>(AF, Y2, o + S::eC, r + S::eC);
  }
  w_copy<NX>(r + S::eB, o + S::eB);
  w_mv<NX, NX, false, 1>(r + S::eA, x, o + S::eB);
  if constexpr (!kFragSym) {
    w_sym<NX>(o + S::eY);
    w_sym<NX>(o + S::eC);
  }
  return fl;
}

// carry step o = e (x) c for a carry (Y, eta) (vstep); c and o are carries
// stored as [Y (NX*NX) | eta (NX)]
template <typename R, int NX, int NU>
PTC_D bool w_vstep(const R* e, const R* c, R* o, R* scr, int* piv) {
  using S = WSlab<R, NX, NU>;
  R* G = scr;
  R* Z = scr + NX * NX;
  constexpr int WZ = NX + 1;
  // G = I + Y_c C_e ; Z = [Y_c A_e | eta_c - Y_c b_e] ; Z <- G^-1 Z
  w_mm<NX, NX, NX, false, false, 0>(c, e + S::eC, G);
  for (int q = lane_id(); q < NX * WZ; q += 32) {
    const int i = q / WZ, j = q - (q / WZ) * WZ;
    R s = R(0);
    if (j < NX) {
#pragma unroll
      for (int k = 0; k < NX; ++k) s = (k == 0) ? c[i * NX] * e[S::eA + j] : fma(c[i * NX + k], e[S::eA + k * NX + j], s);
    } else {
      R yb = R(0);
#pragma unroll
      for (int k = 0; k < NX; ++k) yb = (k == 0) ? c[i * NX] * e[S::eB] : fma(c[i * NX + k], e[S::eB + k], yb);
      s = c[NX * NX + i] - yb;
    }
    Z[q] = s;
  }
  for (int i = lane_id(); i < NX; i += 32) G[i * NX + i] += R(1);
  __syncwarp();
  const bool ok = w_lu<NX>(G, piv);
  w_lu_solve<NX, WZ>(G, piv, Z);
  constexpr bool kFragSym = sizeof(R) == 8 && NX >= 8 && NX <= 16;
  if constexpr (kFragSym) {   // Y' = sym(A_e^T Z1 + Y_e) in the DMMA fragments
    w_mm2_sym_dmma<NX, NX, 0, true, false, false, false, WZ>(
        reinterpret_cast<const double*>(e + S::eA), reinterpret_cast<const double*>(Z), nullptr,
        nullptr, reinterpret_cast<const double*>(e + S::eY), reinterpret_cast<double*>(o));
  } else {
    for (int q = lane_id(); q < NX * NX; q += 32) {
      const int i = q / NX, j = q - (q / NX) * NX;
      R s = R(0);
#pragma unroll
      for (int k = 0; k < NX; ++k) s = (k == 0) ? e[S::eA + i] * Z[j] : fma(e[S::eA + k * NX + i], Z[k * WZ + j], s);
      o[q] = s + e[S::eY + q];
    }
  }
  for (int i = lane_id(); i < NX; i += 32) {
    R s = R(0);
#pragma unroll
    for (int k = 0; k < NX; ++k) s = (k == 0) ? e[S::eA + i] * Z[NX] : fma(e[S::eA + k * NX + i], Z[k * WZ + NX], s);
    o[NX * NX + i] = s + e[S::eEta + i];
  }
  __syncwarp();
  if constexpr (!kFragSym) w_sym<NX>(o);
  return ok;
}

// Riccati-form level-0 step (riccati_step): stage st, carry c -> gains
// (written to Gam (NU*NX) and gam (NU) in the slab) and carry o.
// kCheckR as riccati_step (elements.cuh)
template <typename R, int NX, int NU, bool kCheckR = true>
PTC_D int w_riccati(const R* st, const R* c, R* o, R* Gam, R* gam, R* scr) {
  using S = WSlab<R, NX, NU>;
  R* FtS = scr;                          // NU x NX
  R* Qux = FtS + NU * NX;                // NU x NX
  R* Qm = Qux + NU * NX;                 // NU x NU
  R* SF = Qm + NU * NU;                  // NX x NX
  R* fe = SF + NX * NX;                  // NU: Fu^T eta
  int fl = 0;
  if constexpr (kCheckR) {
    R L[NU][NU];
    if (!w_chol_regs<NU>(st + S::sR, L)) fl |= FLAG_DEF_R;
  }
  w_mm<NU, NX, NX, true, false, 0>(st + S::sFu, c, FtS);
  w_mm<NX, NX, NX, false, false, 0>(c, st + S::sFx, SF);
  w_mm<NU, NX, NU, false, false, 0>(FtS, st + S::sFu, Qm);
  w_mm<NU, NX, NX, false, false, 0>(FtS, st + S::sFx, Qux);
  for (int q = lane_id(); q < NU * NX; q += 32) {
    const int i = q / NX, j = q - (q / NX) * NX;
    Qux[q] += st[S::sM + j * NU + i];
  }
  for (int i = lane_id(); i < NU; i += 32) {   // Fu^T eta, one lane per control
    R f = R(0);
#pragma unroll
    for (int k = 0; k < NX; ++k) f = (k == 0) ? st[S::sFu + i] * c[NX * NX] : fma(st[S::sFu + k * NU + i], c[NX * NX + k], f);
    fe[i] = f;
  }
  __syncwarp();
  R L[NU][NU];
#pragma unroll
  for (int i = 0; i < NU; ++i)
#pragma unroll
    for (int j = 0; j < NU; ++j)
      L[i][j] = R(0.5) * ((Qm[i * NU + j] + st[S::sR + i * NU + j]) +
                          (Qm[j * NU + i] + st[S::sR + j * NU + i]));
  if (!cholesky_rsqrt<NU>(L)) fl |= FLAG_DEF_Q;
  const int ln = lane_id();
  if (ln <= NX) {  // lanes 0..NX-1: columns of Gamma, lane NX: gamma
    R v[NU];
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      v[i] = ln < NX ? Qux[i * NX + ln] : st[S::sd + i] - fe[i];
    }
    chol_solve_vec<NU>(L, v);
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      if (ln < NX) Gam[i * NX + ln] = -v[i];
      else gam[i] = -v[i];
    }
  }
  __syncwarp();
  // S' = sym(P + Fx^T SF + Qux^T Gam), eta' = Fx^T eta - Qux^T gam
  const bool fused_sym = sizeof(R) == 8 && NX >= 8 && NX <= 16;
  if constexpr (sizeof(R) == 8 && NX >= 8 && NX <= 16) {
    // S' = sym(P + Fx^T SF + Qux^T Gam), symmetrised in the product fragments
    w_mm2_sym_dmma<NX, NX, NU, true, false, true, false>(
        reinterpret_cast<const double*>(st + S::sFx), reinterpret_cast<const double*>(SF),
        reinterpret_cast<const double*>(Qux), reinterpret_cast<const double*>(Gam),
        reinterpret_cast<const double*>(st + S::sP), reinterpret_cast<double*>(o));
  } else {
    w_mm<NX, NX, NX, true, false, 2>(st + S::sFx, SF, o, st + S::sP);
    w_mm<NX, NU, NX, true, false, 1>(Qux, Gam, o);
  }
  for (int i = ln; i < NX; i += 32) {
    R s = R(0);
#pragma unroll
    for (int k = 0; k < NX; ++k) s = (k == 0) ? st[S::sFx + i] * c[NX * NX] : fma(st[S::sFx + k * NX + i], c[NX * NX + k], s);
    R g = R(0);
#pragma unroll
    for (int k = 0; k < NU; ++k) g = (k == 0) ? Qux[i] * gam[0] : fma(Qux[k * NX + i], gam[k], g);
    o[NX * NX + i] = s - g;
  }
  __syncwarp();
  if (!fused_sym) w_sym<NX>(o);
  return fl;
}

// affine maps [F (NX*NX) | e (NX)]: o = outer o inner
template <typename R, int NX>
PTC_D void w_aff_compose(const R* outer, const R* inner, R* o) {
  w_mm<NX, NX, NX, false, false, 0>(outer, inner, o);
  w_mv<NX, NX, false, 0>(outer, inner + NX * NX, o + NX * NX);
  for (int i = lane_id(); i < NX; i += 32) o[NX * NX + i] += outer[NX * NX + i];
  __syncwarp();
}

// closed-loop map of stage t: F = Fx + Fu Gamma (0 at global stage 0), e = Fu gamma
template <typename R, int NX, int NU>
PTC_D void w_closed_loop(const R* Fx, const R* Fu, const R* Gam, const R* gam, bool head, R* m) {
  if (head) w_fill<NX * NX>(m, R(0));
  else w_mm<NX, NU, NX, false, false, 2>(Fu, Gam, m, Fx);   // Fx + Fu Gamma
  for (int i = lane_id(); i < NX; i += 32) {
    R s = R(0);
#pragma unroll
    for (int k = 0; k < NU; ++k) s = (k == 0) ? Fu[i * NU] * gam[0] : fma(Fu[i * NU + k], gam[k], s);
    m[NX * NX + i] = s;
  }
  __syncwarp();
}

// Every kernel below carves its own compact per-warp slab (WSlab::k*), so
// the light kernels (carries, propagation) run at high occupancy and only the
// combine-heavy ones pay for large slabs.
#define PTC_WIDE_PROLOGUE(count, ...)                \
  const int u = warp_unit();                         \
  if (u >= (count) * a.B) return;                    \
  const int b = u % a.B, j = u / a.B;                \
  (void)j;                                           \
  if (lqr_skip(a, b)) return;                        \
  using S = WSlab<R, NX, NU>;                        \
  constexpr int kElems = (__VA_ARGS__);              \
  R* slab = warp_slab<R>(kElems);                    \
  int* piv = warp_piv<R>(slab, kElems);              \
  (void)piv;

// ------------------------------------------------------------ value scan

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_value_up0(LqrArgs<R> a) {
  PTC_WIDE_PROLOGUE(a.plan.units0(), WSlab<R, NX, NU>::kUp0)
  const int P0 = a.plan.units0(), T = a.T;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const R alpha = R(a.alpha[b]);
  R* acc = slab;
  R* o = acc + S::VC;
  R* st = o + S::VC;
  R* scr = st + S::SC;
  int fl = 0;
  int start;
  if (j == P0 - 1 && !a.no_terminal) {
    w_ld<NX * NX>(a.PT, 0, 1, a.B, b, scr);
    w_velem_terminal<R, NX, NU>(scr, acc);
    start = t1 - 1;
  } else {
    w_ld_stage<R, NX, NU>(a, t1 - 1, b, alpha, st);
    if (!w_velem<R, NX, NU>(st, acc, scr)) fl |= FLAG_DEF_R;
    start = t1 - 2;
  }
  if (a.staged) {
    WPrefetchRow<R, S::SC> pf;
    pf.init(a.xst, S::SC);
    if (start >= t0) pf.load(start);
    for (int t = start; t >= t0; --t) {
      pf.store(st);
      for (int i = lane_id(); i < NU; i += 32) st[S::sR + i * NU + i] += alpha;
      __syncwarp();
      if (t > t0) pf.load(t - 1);
      fl |= w_vcombine_stage<R, NX, NU>(st, acc, o, scr, piv);
      R* tmp = acc;  // ping-pong instead of copying the aggregate back
      acc = o;
      o = tmp;
    }
  } else {
    StagePrefetch<R, NX, NU> pf;
    w_stage_prefetch_init<R, NX, NU>(pf, a, b);
    if (start >= t0) pf.load(start);
    for (int t = start; t >= t0; --t) {
      w_stage_store<R, NX, NU>(pf, alpha, st);
      if (t > t0) pf.load(t - 1);
      fl |= w_vcombine_stage<R, NX, NU>(st, acc, o, scr, piv);
      R* tmp = acc;
      acc = o;
      o = tmp;
    }
  }
  w_st<S::VC>(a.vagg[1], j, a.plan.n[1], a.B, b, acc);
  if (fl && lane_id() == 0) atomicOr(a.flags + b, fl);
}

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_value_up(LqrArgs<R> a, int l) {
  PTC_WIDE_PROLOGUE(a.plan.n[l + 1], WSlab<R, NX, NU>::kUp)
  const int nl = a.plan.n[l], nn = a.plan.n[l + 1];
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  R* acc = slab;
  R* e = acc + S::VC;
  R* o = e + S::VC;
  R* scr = o + S::VC;
  w_ld<S::VC>(a.vagg[l], last, nl, a.B, b, acc);
  bool okc = true;
  // the next item loads while the current combine runs; acc / o ping-pong
  WPrefetchItem<R, S::VC> pf;
  if (last - 1 >= first) pf.load(a.vagg[l], last - 1, nl, a.B, b);
  for (int i = last - 1; i >= first; --i) {
    pf.store(e);
    if (i - 1 >= first) pf.load(a.vagg[l], i - 1, nl, a.B, b);
    okc &= w_vcombine<R, NX, NU>(e, acc, o, scr, piv);
    R* tmp = acc;
    acc = o;
    o = tmp;
  }
  w_st<S::VC>(a.vagg[l + 1], j, nn, a.B, b, acc);
  if (!okc && lane_id() == 0) atomicOr(a.flags + b, FLAG_COND);
}

// narrow tree levels (few units, latency-bound): one unit per block, its
// items split between the block's two warps -- each folds its half (the
// same right-to-left fold as kw_value_up), then warp 0 combines the halves
// (lower (x) upper).  Depth ceil(K/2) combines instead of K - 1; the
// association differs from the sequential fold only in rounding.
static_assert(kWarpsPerBlock == 2, "kw_value_up2 splits a unit over two warps");
template <typename R, int NX, int NU>
__global__ void __launch_bounds__(64) kw_value_up2(LqrArgs<R> a, int l) {
  using S = WSlab<R, NX, NU>;
  const int u = blockIdx.x;
  if (u >= a.plan.n[l + 1] * a.B) return;  // block-uniform exits only
  const int b = u % a.B, j = u / a.B;
  if (lqr_skip(a, b)) return;
  const int w = threadIdx.x >> 5;
  R* slab = warp_slab<R>(S::kUp);
  int* piv = warp_piv<R>(slab, S::kUp);
  const int nl = a.plan.n[l], nn = a.plan.n[l + 1];
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  const int mid = first + (last - first + 2) / 2;  // warp 0: [first, mid), warp 1: [mid, last]
  const int lo = w == 0 ? first : mid, hi = w == 0 ? mid - 1 : last;
  R* acc = slab;
  R* e = acc + S::VC;
  R* o = e + S::VC;
  R* scr = o + S::VC;
  bool okc = true;
  if (lo <= hi) {
    w_ld<S::VC>(a.vagg[l], hi, nl, a.B, b, acc);
    WPrefetchItem<R, S::VC> pf;
    if (hi - 1 >= lo) pf.load(a.vagg[l], hi - 1, nl, a.B, b);
    for (int i = hi - 1; i >= lo; --i) {
      pf.store(e);
      if (i - 1 >= lo) pf.load(a.vagg[l], i - 1, nl, a.B, b);
      okc &= w_vcombine<R, NX, NU>(e, acc, o, scr, piv);
      R* tmp = acc;
      acc = o;
      o = tmp;
    }
    if (acc != slab) {  // the half's aggregate at the slab base for the other warp
      w_copy<S::VC>(acc, slab);
      o = acc;
      acc = slab;
    }
    // ... and, for the down-sweep's split (kw_value_down2), in global memory
    if (w == 1 && a.vhalf[l]) w_st<S::VC>(a.vhalf[l], j, nn, a.B, b, acc);
  }
  __syncthreads();
  if (w == 0) {
    if (mid <= last) {
      const R* upper = reinterpret_cast<const R*>(reinterpret_cast<const unsigned char*>(slab) +
                                                  S::bytes_of(S::kUp));
      okc &= w_vcombine<R, NX, NU>(acc, upper, o, scr, piv);
      acc = o;
    }
    w_st<S::VC>(a.vagg[l + 1], j, nn, a.B, b, acc);
  }
  if (!okc && lane_id() == 0) atomicOr(a.flags + b, FLAG_COND);
}

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_value_top(LqrArgs<R> a) {
  PTC_WIDE_PROLOGUE(1, WSlab<R, NX, NU>::kStep)
  const int L = a.plan.L, nL = a.plan.n[L];
  R* c = slab;
  R* o = c + S::CC;
  R* e = o + S::CC;
  R* scr = e + S::VC;
  if (a.vcarry_in) w_ld<S::CC>(a.vcarry_in, 0, 1, a.B, b, c);
  else w_fill<S::CC>(c, R(0));
  bool okc = true;
  WPrefetchItem<R, S::VC> pf;
  pf.load(a.vagg[L], nL - 1, nL, a.B, b);
  for (int i = nL - 1; i >= 0; --i) {
    w_st<S::CC>(a.vcar[L], i, nL, a.B, b, c);
    pf.store(e);
    if (i > 0) pf.load(a.vagg[L], i - 1, nL, a.B, b);
    okc &= w_vstep<R, NX, NU>(e, c, o, scr, piv);
    R* tmp = c;
    c = o;
    o = tmp;
  }
  if (!okc && lane_id() == 0) atomicOr(a.flags + b, FLAG_COND);
}

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_value_down(LqrArgs<R> a, int l) {
  PTC_WIDE_PROLOGUE(a.plan.n[l + 1], WSlab<R, NX, NU>::kStep)
  const int nl = a.plan.n[l], nn = a.plan.n[l + 1];
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  R* c = slab;
  R* o = c + S::CC;
  R* e = o + S::CC;
  R* scr = e + S::VC;
  w_ld<S::CC>(a.vcar[l + 1], j, nn, a.B, b, c);
  bool okc = true;
  WPrefetchItem<R, S::VC> pf;
  pf.load(a.vagg[l], last, nl, a.B, b);
  for (int i = last; i >= first; --i) {
    w_st<S::CC>(a.vcar[l], i, nl, a.B, b, c);
    pf.store(e);
    if (i > first) pf.load(a.vagg[l], i - 1, nl, a.B, b);
    okc &= w_vstep<R, NX, NU>(e, c, o, scr, piv);
    R* tmp = c;
    c = o;
    o = tmp;
  }
  if (!okc && lane_id() == 0) atomicOr(a.flags + b, FLAG_COND);
}

// the down-sweep of a split-fold level: warp 1 walks the upper half from
// the unit's carry; warp 0 first applies the upper half's aggregate (stored
// by kw_value_up2) to the carry -- vstep(e_mid (x) .. (x) e_last, c) is the
// carry entering item mid - 1 -- and walks the lower half.  No exchange
// between the warps; depth ceil(K/2) + 1 steps instead of K.
template <typename R, int NX, int NU>
__global__ void __launch_bounds__(64) kw_value_down2(LqrArgs<R> a, int l) {
  using S = WSlab<R, NX, NU>;
  const int u = blockIdx.x;
  if (u >= a.plan.n[l + 1] * a.B) return;
  const int b = u % a.B, j = u / a.B;
  if (lqr_skip(a, b)) return;
  const int w = threadIdx.x >> 5;
  R* slab = warp_slab<R>(S::kStep);
  int* piv = warp_piv<R>(slab, S::kStep);
  const int nl = a.plan.n[l], nn = a.plan.n[l + 1];
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  const int mid = first + (last - first + 2) / 2;
  const int lo = w == 0 ? first : mid, hi = w == 0 ? mid - 1 : last;
  if (lo > hi) return;  // warp-level exit: no block barrier below
  R* c = slab;
  R* o = c + S::CC;
  R* e = o + S::CC;
  R* scr = e + S::VC;
  w_ld<S::CC>(a.vcar[l + 1], j, nn, a.B, b, c);
  bool okc = true;
  WPrefetchItem<R, S::VC> pf;
  pf.load(a.vagg[l], hi, nl, a.B, b);
  if (w == 0 && mid <= last) {
    w_ld<S::VC>(a.vhalf[l], j, nn, a.B, b, e);
    okc &= w_vstep<R, NX, NU>(e, c, o, scr, piv);
    R* tmp = c;
    c = o;
    o = tmp;
  }
  for (int i = hi; i >= lo; --i) {
    w_st<S::CC>(a.vcar[l], i, nl, a.B, b, c);
    pf.store(e);
    if (i > lo) pf.load(a.vagg[l], i - 1, nl, a.B, b);
    okc &= w_vstep<R, NX, NU>(e, c, o, scr, piv);
    R* tmp = c;
    c = o;
    o = tmp;
  }
  if (!okc && lane_id() == 0) atomicOr(a.flags + b, FLAG_COND);
}

template <typename R, int NX, int NU, bool kAgg>
__global__ void __launch_bounds__(128) kw_value_down0(LqrArgs<R> a) {
  PTC_WIDE_PROLOGUE(a.plan.units0(), WSlab<R, NX, NU>::kDown0)
  const int P0 = a.plan.units0(), T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  const R alpha = R(a.alpha[b]);
  const bool tree = a.plan.L >= 1;
  R* c = slab;                       // carry [Y | eta]
  R* o = c + S::CC;                  // next carry
  R* pa = o + S::CC;                 // propagation aggregate [F | e]
  R* m = pa + S::CC;                 // stage closed-loop map
  R* pt = m + S::CC;                 // composition scratch
  R* st = pt + S::CC;
  R* Gam = st + S::SC;               // NU x NX
  R* gam = Gam + NU * NX;            // NU
  R* scr = gam + NU;
  if (tree) w_ld<S::CC>(a.vcar[1], j, a.plan.n[1], B, b, c);
  else if (a.vcarry_in) w_ld<S::CC>(a.vcarry_in, 0, 1, B, b, c);
  else w_fill<S::CC>(c, R(0));
  if (j == P0 - 1 && a.no_terminal && a.S) {
    w_st<NX * NX>(a.S, T, T + 1, B, b, c);
    for (int i = lane_id(); i < NX; i += 32) o[i] = -c[NX * NX + i];
    __syncwarp();
    w_st<NX>(a.s, T, T + 1, B, b, o);
  }
  if (j == P0 - 1 && !a.no_terminal) {
    w_ld<NX * NX>(a.PT, 0, 1, B, b, c);
    w_fill<NX>(c + NX * NX, R(0));
    if (a.S) {
      w_st<NX * NX>(a.S, T, T + 1, B, b, c);
      w_st<NX>(a.s, T, T + 1, B, b, c + NX * NX);
    }
  }
  if constexpr (kAgg) {
    w_identity<NX>(pa);
    w_fill<NX>(pa + NX * NX, R(0));
  }
  int fl = 0;
  constexpr int GC = NU * NX + NU;
  StagePrefetch<R, NX, NU> pf;
  WPrefetchRow<R, S::SC> pfr;
  if (a.staged) {
    pfr.init(a.xst, S::SC);
    if (t1 - 1 >= t0) pfr.load(t1 - 1);
  } else {
    w_stage_prefetch_init<R, NX, NU>(pf, a, b);
    if (t1 - 1 >= t0) pf.load(t1 - 1);
  }
  for (int t = t1 - 1; t >= t0; --t) {
    if (a.staged) {
      pfr.store(st);
      for (int i = lane_id(); i < NU; i += 32) st[S::sR + i * NU + i] += alpha;
      __syncwarp();
      if (t > t0) pfr.load(t - 1);
    } else {
      w_stage_store<R, NX, NU>(pf, alpha, st);
      if (t > t0) pf.load(t - 1);
    }
    fl |= w_riccati<R, NX, NU, !kAgg>(st, c, o, Gam, gam, scr);
    if (a.staged) {  // [Gamma | gamma] contiguous in the slab and in gst
      for (int i = lane_id(); i < GC; i += 32) a.gst[(size_t)t * GC + i] = Gam[i];
    } else {
      w_st<NU * NX>(a.Gam, t, T, B, b, Gam);
      w_st<NU>(a.gam, t, T, B, b, gam);
    }
    if constexpr (kAgg) {
      w_closed_loop<R, NX, NU>(st + S::sFx, st + S::sFu, Gam, gam, t + a.t_base == 0, m);
      w_aff_compose<R, NX>(pa, m, pt);
      R* tp = pa;  // ping-pong
      pa = pt;
      pt = tp;
    }
    {
      R* tc = c;
      c = o;
      o = tc;
    }
    if (a.S) {
      w_st<NX * NX>(a.S, t, T + 1, B, b, c);
      for (int i = lane_id(); i < NX; i += 32) o[i] = -c[NX * NX + i];
      __syncwarp();
      w_st<NX>(a.s, t, T + 1, B, b, o);
    }
  }
  if constexpr (kAgg) w_st<S::CC>(a.pagg[1], j, a.plan.n[1], B, b, pa);
  if (fl && lane_id() == 0) atomicOr(a.flags + b, fl);
}

// ------------------------------------------------------ propagation scan

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_prop_up(LqrArgs<R> a, int l) {
  PTC_WIDE_PROLOGUE(a.plan.n[l + 1], WSlab<R, NX, NU>::kProp)
  const int nl = a.plan.n[l], nn = a.plan.n[l + 1];
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  R* acc = slab;
  R* m = acc + S::CC;
  R* o = m + S::CC;
  w_ld<S::CC>(a.pagg[l], first, nl, a.B, b, acc);
  for (int i = first + 1; i <= last; ++i) {
    w_ld<S::CC>(a.pagg[l], i, nl, a.B, b, m);
    w_aff_compose<R, NX>(m, acc, o);
    w_copy<S::CC>(o, acc);
  }
  w_st<S::CC>(a.pagg[l + 1], j, nn, a.B, b, acc);
}

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_prop_up0(LqrArgs<R> a) {
  PTC_WIDE_PROLOGUE(a.plan.units0(), WSlab<R, NX, NU>::kPropUp0)
  const int T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  R* acc = slab;
  R* m = acc + S::CC;
  R* o = m + S::CC;
  R* Fx = o + S::CC;
  R* Fu = Fx + NX * NX;
  R* Gam = Fu + NX * NU;
  R* gam = Gam + NU * NX;
  w_identity<NX>(acc);
  w_fill<NX>(acc + NX * NX, R(0));
  WPrefetch<R, NX * NX, NX * NU, NU * NX, NU> pf;
  pf.init(a.Fx, a.Fu, a.Gam, a.gam, nullptr, nullptr, T, B, b);
  if (t0 < t1) pf.load(t0);
  for (int t = t0; t < t1; ++t) {
    pf.store(Fx);
    if (t + 1 < t1) pf.load(t + 1);
    w_closed_loop<R, NX, NU>(Fx, Fu, Gam, gam, t + a.t_base == 0, m);
    w_aff_compose<R, NX>(m, acc, o);
    w_copy<S::CC>(o, acc);
  }
  w_st<S::CC>(a.pagg[1], j, a.plan.n[1], B, b, acc);
}

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_prop_top(LqrArgs<R> a) {
  PTC_WIDE_PROLOGUE(1, WSlab<R, NX, NU>::kProp)
  const int L = a.plan.L, nL = a.plan.n[L];
  R* x = slab;
  R* m = x + S::CC;
  R* y = m + S::CC;
  if (a.x_in) w_ld<NX>(a.x_in, 0, 1, a.B, b, x);
  else w_fill<NX>(x, R(0));
  for (int i = 0; i < nL; ++i) {
    w_st<NX>(a.pcar[L], i, nL, a.B, b, x);
    w_ld<S::CC>(a.pagg[L], i, nL, a.B, b, m);
    w_mv<NX, NX, false, 0>(m, x, y);
    for (int k = lane_id(); k < NX; k += 32) x[k] = y[k] + m[NX * NX + k];
    __syncwarp();
  }
}

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_prop_down(LqrArgs<R> a, int l) {
  PTC_WIDE_PROLOGUE(a.plan.n[l + 1], WSlab<R, NX, NU>::kProp)
  const int nl = a.plan.n[l], nn = a.plan.n[l + 1];
  const int first = j * a.plan.K, last = min(nl, first + a.plan.K) - 1;
  R* x = slab;
  R* m = x + S::CC;
  R* y = m + S::CC;
  w_ld<NX>(a.pcar[l + 1], j, nn, a.B, b, x);
  for (int i = first; i <= last; ++i) {
    w_st<NX>(a.pcar[l], i, nl, a.B, b, x);
    w_ld<S::CC>(a.pagg[l], i, nl, a.B, b, m);
    w_mv<NX, NX, false, 0>(m, x, y);
    for (int k = lane_id(); k < NX; k += 32) x[k] = y[k] + m[NX * NX + k];
    __syncwarp();
  }
}

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_prop_down0(LqrArgs<R> a) {
  PTC_WIDE_PROLOGUE(a.plan.units0(), WSlab<R, NX, NU>::kPropDown0)
  const int P0 = a.plan.units0(), T = a.T, B = a.B;
  const int t0 = j * a.plan.K0, t1 = min(T, t0 + a.plan.K0);
  R* x = slab;
  R* y = x + NX;
  R* du = y + NX;
  R* Fx = du + NU;                   // prefetched [Fx | Fu | Gamma | gamma | d]
  R* Fu = Fx + NX * NX;
  R* Gam = Fu + NX * NU;
  R* gam = Gam + NU * NX;
  R* dd = gam + NU;
  if (a.plan.L >= 1) w_ld<NX>(a.pcar[1], j, a.plan.n[1], B, b, x);
  else if (a.x_in) w_ld<NX>(a.x_in, 0, 1, B, b, x);
  else w_fill<NX>(x, R(0));
  double s2 = 0.0, sd = 0.0, mx = 0.0;  // accumulated by lane 0
  const int ln = lane_id();
  WPrefetch<R, NX * NX, NX * NU, NU * NX, NU, NU> pf;
  WPrefetchRow<R, NX * NX + NX * NU> pfa;   // staged: [Fx | Fu] of xst
  WPrefetchRow<R, NU * NX + NU> pfb;        //         [Gamma | gamma] of gst
  WPrefetchRow<R, NU> pfc;                  //         d of xst
  if (a.staged) {
    pfa.init(a.xst + S::sFx, S::SC);
    pfb.init(a.gst, NU * NX + NU);
    pfc.init(a.xst + S::sd, S::SC);
    if (t0 < t1) {
      pfa.load(t0);
      pfb.load(t0);
      pfc.load(t0);
    }
  } else {
    pf.init(a.Fx, a.Fu, a.Gam, a.gam, a.d, nullptr, T, B, b);
    if (t0 < t1) pf.load(t0);
  }
  for (int t = t0; t < t1; ++t) {
    w_st<NX>(a.dX, t, T + 1, B, b, x);
    if (a.staged) {
      pfa.store(Fx);
      pfb.store(Gam);
      pfc.store(dd);
      if (t + 1 < t1) {
        pfa.load(t + 1);
        pfb.load(t + 1);
        pfc.load(t + 1);
      }
    } else {
      pf.store(Fx);
      if (t + 1 < t1) pf.load(t + 1);
    }
    w_mv<NU, NX, false, 0>(Gam, x, du);
    for (int i = ln; i < NU; i += 32) du[i] += gam[i];
    __syncwarp();
    if (ln == 0) {
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        s2 += double(du[i]) * double(du[i]);
        sd += double(du[i]) * double(dd[i]);
        mx = nanmax(mx, double(fabs(du[i])));
      }
    }
    w_st<NU>(a.dU, t, T, B, b, du);
    // x <- Fx x + Fu du  (= (Fx + Fu Gamma) x + Fu gamma; at global stage 0
    // the closed-loop map is 0 and x <- Fu gamma)
    const bool head = t + a.t_base == 0;
    for (int i = ln; i < NX; i += 32) {
      R fu = R(0);
#pragma unroll
      for (int k = 0; k < NU; ++k)
        fu = (k == 0) ? Fu[i * NU] * (head ? gam[0] : du[0]) : fma(Fu[i * NU + k], head ? gam[k] : du[k], fu);
      R fx = R(0);
#pragma unroll
      for (int q = 0; q < NX; ++q) fx = (q == 0) ? Fx[i * NX] * x[0] : fma(Fx[i * NX + q], x[q], fx);
      y[i] = head ? fu : fx + fu;
    }
    __syncwarp();
    w_copy<NX>(y, x);
  }
  if (j == P0 - 1) w_st<NX>(a.dX, T, T + 1, B, b, x);
  if (a.red && ln == 0) {
    a.red[((size_t)0 * P0 + j) * B + b] = s2;
    a.red[((size_t)1 * P0 + j) * B + b] = sd;
    a.red[((size_t)2 * P0 + j) * B + b] = mx;
  }
}

// ------------------------------------------------------------ time blocks

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_value_block(LqrArgs<R> a, R* out) {
  PTC_WIDE_PROLOGUE(1, WSlab<R, NX, NU>::kUp)
  const int L = a.plan.L > 0 ? a.plan.L : 1, nL = a.plan.n[L];
  R* acc = slab;
  R* e = acc + S::VC;
  R* o = e + S::VC;
  R* scr = o + S::VC;
  w_ld<S::VC>(a.vagg[L], nL - 1, nL, a.B, b, acc);
  bool okc = true;
  for (int i = nL - 2; i >= 0; --i) {
    w_ld<S::VC>(a.vagg[L], i, nL, a.B, b, e);
    okc &= w_vcombine<R, NX, NU>(e, acc, o, scr, piv);
    w_copy<S::VC>(o, acc);
  }
  w_st<S::VC>(out, 0, 1, a.B, b, acc);
  if (!okc && lane_id() == 0) atomicOr(a.flags + b, FLAG_COND);
}

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_value_carry(LqrArgs<R> a, const R* blocks, int rank,
                                                      int world) {
  PTC_WIDE_PROLOGUE(1, WSlab<R, NX, NU>::kStep)
  R* c = slab;
  R* o = c + S::CC;
  R* e = o + S::CC;
  R* scr = e + S::VC;
  w_fill<S::CC>(c, R(0));
  bool okc = true;
  for (int r = world - 1; r > rank; --r) {
    w_ld<S::VC>(blocks + (size_t)r * S::VC * a.B, 0, 1, a.B, b, e);
    okc &= w_vstep<R, NX, NU>(e, c, o, scr, piv);
    w_copy<S::CC>(o, c);
  }
  w_st<S::CC>(a.vcin_buf, 0, 1, a.B, b, c);
  if (!okc && lane_id() == 0) atomicOr(a.flags + b, FLAG_COND);
}

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_prop_block(LqrArgs<R> a, R* out) {
  PTC_WIDE_PROLOGUE(1, WSlab<R, NX, NU>::kProp)
  const int L = a.plan.L > 0 ? a.plan.L : 1, nL = a.plan.n[L];
  R* acc = slab;
  R* m = acc + S::CC;
  R* o = m + S::CC;
  w_ld<S::CC>(a.pagg[L], 0, nL, a.B, b, acc);
  for (int i = 1; i < nL; ++i) {
    w_ld<S::CC>(a.pagg[L], i, nL, a.B, b, m);
    w_aff_compose<R, NX>(m, acc, o);
    w_copy<S::CC>(o, acc);
  }
  w_st<S::CC>(out, 0, 1, a.B, b, acc);
}

template <typename R, int NX, int NU>
__global__ void __launch_bounds__(128) kw_prop_carry(LqrArgs<R> a, const R* blocks, int rank) {
  PTC_WIDE_PROLOGUE(1, WSlab<R, NX, NU>::kProp)
  R* x = slab;
  R* m = x + S::CC;
  R* y = m + S::CC;
  w_fill<NX>(x, R(0));
  for (int r = 0; r < rank; ++r) {
    w_ld<S::CC>(blocks + (size_t)r * S::CC * a.B, 0, 1, a.B, b, m);
    w_mv<NX, NX, false, 0>(m, x, y);
    for (int k = lane_id(); k < NX; k += 32) x[k] = y[k] + m[NX * NX + k];
    __syncwarp();
  }
  w_st<NX>(a.xin_buf, 0, 1, a.B, b, x);
}

#undef PTC_WIDE_PROLOGUE

// ------------------------------------------------------------ launchers

template <typename R, int NX, int NU>
struct Wide {
  using S = WSlab<R, NX, NU>;
  static constexpr int smem(int elems) { return kWarpsPerBlock * S::bytes_of(elems); }
  static dim3 grid(long long units) {
    return dim3((unsigned)((units + kWarpsPerBlock - 1) / kWarpsPerBlock));
  }
  template <class K>
  static void allow(K kernel, int elems) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem(elems));
  }
  static void setup() {
    static bool done = false;
    if (done) return;
    allow(kw_value_up0<R, NX, NU>, S::kUp0);
    allow(kw_value_up<R, NX, NU>, S::kUp);
    allow(kw_value_up2<R, NX, NU>, S::kUp);
    allow(kw_value_down2<R, NX, NU>, S::kStep);
    allow(kw_value_top<R, NX, NU>, S::kStep);
    allow(kw_value_down<R, NX, NU>, S::kStep);
    allow(kw_value_down0<R, NX, NU, true>, S::kDown0);
    allow(kw_value_down0<R, NX, NU, false>, S::kDown0);
    allow(kw_prop_up<R, NX, NU>, S::kProp);
    allow(kw_prop_up0<R, NX, NU>, S::kPropUp0);
    allow(kw_prop_top<R, NX, NU>, S::kProp);
    allow(kw_prop_down<R, NX, NU>, S::kProp);
    allow(kw_prop_down0<R, NX, NU>, S::kPropDown0);
    allow(kw_value_block<R, NX, NU>, S::kUp);
    allow(kw_value_carry<R, NX, NU>, S::kStep);
    allow(kw_prop_block<R, NX, NU>, S::kProp);
    allow(kw_prop_carry<R, NX, NU>, S::kProp);
    done = true;
  }
};

#define PTC_WL(kernel, units, elems) kernel<<<W::grid(units), 32 * kWarpsPerBlock, W::smem(elems), s>>>

// one up-sweep level: the sequential fold while the level is wide enough to
// fill the GPU, the two-warp split fold on the narrow (latency-bound) levels
constexpr long long kUp2MaxUnits = 1024;
template <typename R, int NX, int NU>
void kw_value_up_level(const LqrArgs<R>& a, int l, cudaStream_t s) {
  using W = Wide<R, NX, NU>;
  using S = WSlab<R, NX, NU>;
  const long long units = (long long)a.plan.n[l + 1] * a.B;
  if (units <= kUp2MaxUnits)
    kw_value_up2<R, NX, NU><<<(unsigned)units, 32 * kWarpsPerBlock, W::smem(S::kUp), s>>>(a, l);
  else
    PTC_WL((kw_value_up<R, NX, NU>), units, S::kUp)(a, l);
}

template <typename R, int NX, int NU>
void launch_prop_tree_wide(const LqrArgs<R>& a, cudaStream_t s) {
  using W = Wide<R, NX, NU>;
  using S = WSlab<R, NX, NU>;
  const Plan& pl = a.plan;
  const long long B = a.B;
  for (int l = 1; l < pl.L; ++l) PTC_WL((kw_prop_up<R, NX, NU>), pl.n[l + 1] * B, S::kProp)(a, l);
  PTC_WL((kw_prop_top<R, NX, NU>), B, S::kProp)(a);
  for (int l = pl.L - 1; l >= 1; --l) PTC_WL((kw_prop_down<R, NX, NU>), pl.n[l + 1] * B, S::kProp)(a, l);
}

template <typename R, int NX, int NU>
void launch_value_tree_wide(const LqrArgs<R>& a, cudaStream_t s) {
  using W = Wide<R, NX, NU>;
  using S = WSlab<R, NX, NU>;
  const Plan& pl = a.plan;
  const long long B = a.B;
  PTC_WL((kw_value_top<R, NX, NU>), B, S::kStep)(a);
  for (int l = pl.L - 1; l >= 1; --l) {
    const long long units = (long long)pl.n[l + 1] * B;
    if (a.vhalf[l] && units <= kUp2MaxUnits)
      kw_value_down2<R, NX, NU><<<(unsigned)units, 32 * kWarpsPerBlock, W::smem(S::kStep), s>>>(a, l);
    else
      PTC_WL((kw_value_down<R, NX, NU>), units, S::kStep)(a, l);
  }
}

template <typename R, int NX, int NU>
void launch_stage_in(const LqrArgs<R>& a, cudaStream_t s) {
  constexpr int SC = WSlab<R, NX, NU>::SC;
  kw_stage_in<R, NX, NU><<<dim3((SC + 31) / 32, (a.T + 31) / 32), dim3(32, 8), 0, s>>>(a);
}

template <typename R, int NX, int NU>
void launch_gains_out(const LqrArgs<R>& a, cudaStream_t s) {
  constexpr int GC = NU * NX + NU;
  kw_gains_out<R, NX, NU><<<dim3((GC + 31) / 32, (a.T + 31) / 32), dim3(32, 8), 0, s>>>(a);
}

template <typename R, int NX, int NU>
void launch_lqr_wide(const LqrArgs<R>& a0, cudaStream_t s) {
  using W = Wide<R, NX, NU>;
  using S = WSlab<R, NX, NU>;
  W::setup();
  LqrArgs<R> a = a0;
  a.staged = (a.xst != nullptr && a.B == 1) ? 1 : 0;
  if (a.staged && !a.prestaged) launch_stage_in<R, NX, NU>(a, s);
  const Plan& pl = a.plan;
  const long long B = a.B, P0 = pl.units0();
  if (pl.L >= 1) {
    PTC_WL((kw_value_up0<R, NX, NU>), P0 * B, S::kUp0)(a);
    for (int l = 1; l < pl.L; ++l) kw_value_up_level<R, NX, NU>(a, l, s);
    launch_value_tree_wide<R, NX, NU>(a, s);
    PTC_WL((kw_value_down0<R, NX, NU, true>), P0 * B, S::kDown0)(a);
    launch_prop_tree_wide<R, NX, NU>(a, s);
  } else {
    PTC_WL((kw_value_down0<R, NX, NU, false>), P0 * B, S::kDown0)(a);
  }
  PTC_WL((kw_prop_down0<R, NX, NU>), P0 * B, S::kPropDown0)(a);
  if (a.staged && !a.gains_in_gst) launch_gains_out<R, NX, NU>(a, s);
}

template <typename R, int NX, int NU>
void launch_prop_wide(const LqrArgs<R>& a, cudaStream_t s) {
  using W = Wide<R, NX, NU>;
  using S = WSlab<R, NX, NU>;
  W::setup();
  const Plan& pl = a.plan;
  const long long B = a.B, P0 = pl.units0();
  if (pl.L >= 1) {
    PTC_WL((kw_prop_up0<R, NX, NU>), P0 * B, S::kPropUp0)(a);
    launch_prop_tree_wide<R, NX, NU>(a, s);
  }
  PTC_WL((kw_prop_down0<R, NX, NU>), P0 * B, S::kPropDown0)(a);
}

template <typename R, int NX, int NU>
void launch_lqr_block_wide(const LqrArgs<R>& a0, int phase, const void* blocks, void* out,
                           int rank, int world, cudaStream_t s) {
  using W = Wide<R, NX, NU>;
  using S = WSlab<R, NX, NU>;
  W::setup();
  LqrArgs<R> a = a0;
  a.staged = (a.xst != nullptr && a.B == 1) ? 1 : 0;
  const Plan& pl = a.plan;
  const long long B = a.B, P0 = pl.units0();
  if (phase == 0) {
    if (a.staged && !a.prestaged) launch_stage_in<R, NX, NU>(a, s);
    PTC_WL((kw_value_up0<R, NX, NU>), P0 * B, S::kUp0)(a);
    for (int l = 1; l < pl.L; ++l) kw_value_up_level<R, NX, NU>(a, l, s);
    PTC_WL((kw_value_block<R, NX, NU>), B, S::kUp)(a, static_cast<R*>(out));
  } else if (phase == 1) {
    PTC_WL((kw_value_carry<R, NX, NU>), B, S::kStep)(a, static_cast<const R*>(blocks), rank, world);
    a.vcarry_in = a.vcin_buf;
    if (pl.L >= 1) launch_value_tree_wide<R, NX, NU>(a, s);
    PTC_WL((kw_value_down0<R, NX, NU, true>), P0 * B, S::kDown0)(a);
    for (int l = 1; l < pl.L; ++l) PTC_WL((kw_prop_up<R, NX, NU>), pl.n[l + 1] * B, S::kProp)(a, l);
    PTC_WL((kw_prop_block<R, NX, NU>), B, S::kProp)(a, static_cast<R*>(out));
  } else {
    PTC_WL((kw_prop_carry<R, NX, NU>), B, S::kProp)(a, static_cast<const R*>(blocks), rank);
    a.x_in = a.xin_buf;
    if (pl.L >= 1) {
      PTC_WL((kw_prop_top<R, NX, NU>), B, S::kProp)(a);
      for (int l = pl.L - 1; l >= 1; --l) PTC_WL((kw_prop_down<R, NX, NU>), pl.n[l + 1] * B, S::kProp)(a, l);
    }
    PTC_WL((kw_prop_down0<R, NX, NU>), P0 * B, S::kPropDown0)(a);
    if (a.staged && !a.gains_in_gst) launch_gains_out<R, NX, NU>(a, s);
  }
}

#undef PTC_WL

}  // namespace ptc
