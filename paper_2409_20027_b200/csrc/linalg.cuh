// Fixed-size dense linear algebra in registers (compile-time shapes, fully
// unrolled).  Everything a value-function combine needs: products,
// Cholesky (with the LAPACK potrf failure rule), LU with partial pivoting
// applied by predicated row swaps so no register array is ever indexed
// dynamically, and solves with the matrix or its transpose.
#pragma once

#include "common.cuh"

namespace ptc {

// Structural sparsity: a mask bit (row * cols + col) set = the entry may be
// nonzero.  A model whose Jacobian has known zeros (the Euler steps' identity
// blocks) passes its mask, and the products skip those terms: a skipped term
// fma(a, 0, acc) = acc for finite a, so the result is the dense one up to
// the sign of an exact zero.  kDense (every entry) is the default.
constexpr uint64_t kDense = ~0ull;
PTC_HD constexpr bool may_nz(uint64_t mask, int idx) { return idx >= 64 || ((mask >> idx) & 1ull); }
// structure of A + B G for A: R x C (mask MA), B: R x K (mask MB), G dense:
// every row of B with a nonzero fills its whole row
template <int R_, int C_, int K_>
PTC_HD constexpr uint64_t plus_rows_mask(uint64_t MA, uint64_t MB) {
  if (R_ * C_ > 64 || R_ * K_ > 64) return kDense;
  uint64_t m = MA;
  for (int i = 0; i < R_; ++i) {
    bool row = false;
    for (int k = 0; k < K_; ++k) row = row || may_nz(MB, i * K_ + k);
    if (row)
      for (int j = 0; j < C_; ++j) m |= 1ull << (i * C_ + j);
  }
  return m;
}

// C = A * B  (A: MxK, B: KxN; MB, MA = structures of B and A)
template <int M, int K, int N, typename R, uint64_t MB = kDense, uint64_t MA = kDense>
PTC_D void mm(const R (&A)[M][K], const R (&B)[K][N], R (&C)[M][N]) {
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R acc = R(0);
      bool any = false;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!may_nz(MB, k * N + j) || !may_nz(MA, i * K + k)) continue;
        acc = any ? fma(A[i][k], B[k][j], acc) : A[i][k] * B[k][j];
        any = true;
      }
      C[i][j] = acc;
    }
}

// C = A^T * B  (A: KxM, B: KxN; MA = structure of A)
template <int M, int K, int N, typename R, uint64_t MA = kDense>
PTC_D void mtm(const R (&A)[K][M], const R (&B)[K][N], R (&C)[M][N]) {
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R acc = R(0);
      bool any = false;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!may_nz(MA, k * M + i)) continue;
        acc = any ? fma(A[k][i], B[k][j], acc) : A[k][i] * B[k][j];
        any = true;
      }
      C[i][j] = acc;
    }
}

// C = A * B^T  (A: MxK, B: NxK)
template <int M, int K, int N, typename R>
PTC_D void mmt(const R (&A)[M][K], const R (&B)[N][K], R (&C)[M][N]) {
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R acc = A[i][0] * B[j][0];
#pragma unroll
      for (int k = 1; k < K; ++k) acc = fma(A[i][k], B[j][k], acc);
      C[i][j] = acc;
    }
}

// y = A x  (MA = structure of A)
template <int M, int K, typename R, uint64_t MA = kDense>
PTC_D void mv(const R (&A)[M][K], const R (&x)[K], R (&y)[M]) {
#pragma unroll
  for (int i = 0; i < M; ++i) {
    R acc = R(0);
    bool any = false;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!may_nz(MA, i * K + k)) continue;
      acc = any ? fma(A[i][k], x[k], acc) : A[i][k] * x[k];
      any = true;
    }
    y[i] = acc;
  }
}

// y = A^T x  (A: KxM; MA = structure of A)
template <int M, int K, typename R, uint64_t MA = kDense>
PTC_D void mtv(const R (&A)[K][M], const R (&x)[K], R (&y)[M]) {
#pragma unroll
  for (int i = 0; i < M; ++i) {
    R acc = R(0);
    bool any = false;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!may_nz(MA, k * M + i)) continue;
      acc = any ? fma(A[k][i], x[k], acc) : A[k][i] * x[k];
      any = true;
    }
    y[i] = acc;
  }
}

template <int N, typename R>
PTC_D void symmetrize(R (&A)[N][N]) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i + 1; j < N; ++j) {
      R v = R(0.5) * (A[i][j] + A[j][i]);
      A[i][j] = v;
      A[j][i] = v;
    }
}

template <int N, typename R>
PTC_D void set_identity(R (&A)[N][N]) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) A[i][j] = (i == j) ? R(1) : R(0);
}

template <int M, int N, typename R>
PTC_D void set_zero(R (&A)[M][N]) {
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) A[i][j] = R(0);
}

template <int N, typename R>
PTC_D void set_zero(R (&a)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = R(0);
}

// In-place lower Cholesky factor L (A = L L^T) with the RECIPROCAL of the
// diagonal stored on the diagonal, so the solves below multiply instead of
// divide (one division per row instead of one per right-hand side).  Fails
// (returns false) exactly when LAPACK potrf would: a non-positive or NaN pivot.
template <int N, typename R>
PTC_D bool cholesky(R (&A)[N][N]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    R s = A[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) s = fma(-A[j][k], A[j][k], s);
    ok = ok && (s > R(0));
    const R inv = R(1) / sqrt(s);
    A[j][j] = inv;
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      R v = A[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) v = fma(-A[i][k], A[j][k], v);
      A[i][j] = v * inv;
    }
  }
  return ok;
}

// The same factorisation with the reciprocal diagonal from one rsqrt
// (<= 1 ulp, like 1/sqrt) instead of a square root and a division: the
// warp-per-unit kernels' Cholesky factors sit on their latency-critical path.
template <int N, typename R>
PTC_D bool cholesky_rsqrt(R (&A)[N][N]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    R s = A[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) s = fma(-A[j][k], A[j][k], s);
    ok = ok && (s > R(0));
    const R inv = rsqrt(s);
    A[j][j] = inv;
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      R v = A[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) v = fma(-A[i][k], A[j][k], v);
      A[i][j] = v * inv;
    }
  }
  return ok;
}

// Solve (L L^T) X = B in place, L from cholesky() (reciprocal diagonal).
template <int N, int M, typename R>
PTC_D void chol_solve(const R (&L)[N][N], R (&B)[N][M]) {
#pragma unroll
  for (int c = 0; c < M; ++c) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R v = B[i][c];
#pragma unroll
      for (int k = 0; k < i; ++k) v = fma(-L[i][k], B[k][c], v);
      B[i][c] = v * L[i][i];
    }
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
      R v = B[i][c];
#pragma unroll
      for (int k = i + 1; k < N; ++k) v = fma(-L[k][i], B[k][c], v);
      B[i][c] = v * L[i][i];
    }
  }
}

template <int N, typename R>
PTC_D void chol_solve_vec(const R (&L)[N][N], R (&b)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R v = b[i];
#pragma unroll
    for (int k = 0; k < i; ++k) v = fma(-L[i][k], b[k], v);
    b[i] = v * L[i][i];
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    R v = b[i];
#pragma unroll
    for (int k = i + 1; k < N; ++k) v = fma(-L[k][i], b[k], v);
    b[i] = v * L[i][i];
  }
}

// Row swap i <-> k of an N x M array, applied only when `cond` holds.  All
// indices are compile-time after unrolling, so the arrays stay in registers.
template <int N, int M, typename R>
PTC_D void cswap_rows(R (&A)[N][M], int i, int k, bool cond) {
#pragma unroll
  for (int j = 0; j < M; ++j) {
    R a = A[i][j], b = A[k][j];
    A[i][j] = cond ? b : a;
    A[k][j] = cond ? a : b;
  }
}

// LU factorisation with partial pivoting (P A = L U, unit L), LAPACK getrf
// pivot rule (first maximal |a_ik|).  Returns false on an exactly zero pivot
// (numpy raises LinAlgError "Singular matrix" in that case).
template <int N, typename R>
PTC_D bool lu_factor(R (&A)[N][N], int (&piv)[N]) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int p = k;
    R best = fabs(A[k][k]);
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      R v = fabs(A[i][k]);
      bool take = v > best;
      best = take ? v : best;
      p = take ? i : p;
    }
    piv[k] = p;
#pragma unroll
    for (int i = k + 1; i < N; ++i) cswap_rows<N, N>(A, i, k, p == i);
    R pv = A[k][k];
    ok = ok && (pv != R(0));
    R inv = rcp_rn(pv);
    A[k][k] = inv;  // U's diagonal is kept as reciprocals (solves multiply)
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      R l = A[i][k] * inv;
      A[i][k] = l;
#pragma unroll
      for (int j = k + 1; j < N; ++j) A[i][j] = fma(-l, A[k][j], A[i][j]);
    }
  }
  return ok;
}

// Solve A X = B in place given lu_factor(A).
template <int N, int M, typename R>
PTC_D void lu_solve(const R (&LU)[N][N], const int (&piv)[N], R (&B)[N][M]) {
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int i = k + 1; i < N; ++i) cswap_rows<N, M>(B, i, k, piv[k] == i);
#pragma unroll
  for (int c = 0; c < M; ++c) {
#pragma unroll
    for (int i = 1; i < N; ++i) {
      R v = B[i][c];
#pragma unroll
      for (int k = 0; k < i; ++k) v = fma(-LU[i][k], B[k][c], v);
      B[i][c] = v;
    }
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
      R v = B[i][c];
#pragma unroll
      for (int k = i + 1; k < N; ++k) v = fma(-LU[i][k], B[k][c], v);
      B[i][c] = v * LU[i][i];
    }
  }
}

// Solve A^T X = B in place given lu_factor(A):  A^T = U^T L^T P.
template <int N, int M, typename R>
PTC_D void lu_solve_t(const R (&LU)[N][N], const int (&piv)[N], R (&B)[N][M]) {
#pragma unroll
  for (int c = 0; c < M; ++c) {
#pragma unroll
    for (int i = 0; i < N; ++i) {  // U^T y = b (lower, non-unit)
      R v = B[i][c];
#pragma unroll
      for (int k = 0; k < i; ++k) v = fma(-LU[k][i], B[k][c], v);
      B[i][c] = v * LU[i][i];
    }
#pragma unroll
    for (int i = N - 2; i >= 0; --i) {  // L^T z = y (upper, unit)
      R v = B[i][c];
#pragma unroll
      for (int k = i + 1; k < N; ++k) v = fma(-LU[k][i], B[k][c], v);
      B[i][c] = v;
    }
  }
#pragma unroll
  for (int k = N - 1; k >= 0; --k)
#pragma unroll
    for (int i = k + 1; i < N; ++i) cswap_rows<N, M>(B, i, k, piv[k] == i);
}

}  // namespace ptc
