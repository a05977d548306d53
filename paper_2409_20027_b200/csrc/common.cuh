// Common definitions for the pintoc-b200 CUDA library (sm_100a).
//
// HBM layout convention ("SoA, batch-minor"): every per-stage quantity is a
// field of C scalar components over (rows, batch) stored as
//     field[(c * rows + t) * B + b]
// so consecutive problems b are adjacent (coalesced when a warp walks a
// batch) and, for batch 1, consecutive stages t are adjacent (coalesced when
// a warp walks time).  Matrices are stored row-major inside the component
// index (c = i * ncols + j).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <math.h>

#define PTC_HD __host__ __device__ __forceinline__
#define PTC_D __device__ __forceinline__

namespace ptc {

// a rounded product the compiler may not contract into a following add
// (keeps the bits of code that formed the product as a separate value)
PTC_D double mul_rn(double a, double b) { return __dmul_rn(a, b); }
PTC_D float mul_rn(float a, float b) { return __fmul_rn(a, b); }
// correctly rounded reciprocal (bit-identical to R(1) / x under IEEE
// division, without the general division's numerator path)
__device__ __forceinline__ double rcp_rn(double x) { return __drcp_rn(x); }
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }
}  // namespace ptc

namespace ptc {

constexpr int kMaxLevels = 12;

// per-problem flag bits raised by the kernels of one Newton iteration
enum : int {
  FLAG_DEF_R = 1,       // R + alpha I not positive definite (DefinitenessError)
  FLAG_DEF_Q = 2,       // Q_t not positive definite (DefinitenessError)
  FLAG_COND = 4,        // singular I + C Y inside a combine (ConditioningError)
  FLAG_DIVERGED = 8,    // candidate rollout produced a non-finite state
};

// solver phase bits (what the next iteration has to do for a problem)
enum : int {
  PH_NEED_COST = 1,     // evaluate the augmented cost of the current trajectory
  PH_NEED_EXP = 2,      // recompute co-states and the expansion
  PH_ROUND_DONE = 4,    // the Newton solve of this outer round just finished
};

enum : int {
  ST_RUNNING = 0,
  ST_DONE = 1,
  ST_ERR_STALLED = -1,     // SolverStalledError
  ST_ERR_INFEASIBLE = -2,  // InfeasibleError at the start of a Newton solve
};

enum : int { TERM_NONE = 0, TERM_COST = 1, TERM_STEP = 2, TERM_MAX_ITERS = 3, TERM_STALLED = 4 };

enum : int { AUG_ZERO = 0, AUG_BARRIER = 1, AUG_ADMM = 2 };

// NaN-propagating max (numpy semantics: a NaN on either side wins), unlike fmax
template <typename T>
PTC_HD T nanmax(T a, T b) { return (a != a) ? a : ((b != b || b > a) ? b : a); }

// Plan of the blocked scan tree over one horizon.
//   level 0 items: the T stages; one level-0 unit folds K0 consecutive stages
//   level l >= 1 items: aggregates of level l-1 units; a unit folds K items
//   L = number of tree levels above 0 (0 means one unit spans the horizon)
struct Plan {
  int K0, K, L;
  int n[kMaxLevels + 1];  // n[0] = T, n[l] = item count at level l
  PTC_HD int units0() const { return n[0] <= 0 ? 0 : (n[0] + K0 - 1) / K0; }
};

inline Plan make_plan(int T, int K0, int K) {
  Plan p{};
  if (K < 2) K = 2;
  if (K0 < 1) K0 = 1;
  if (K0 > T) K0 = T;
  p.K0 = K0;
  p.K = K;
  p.n[0] = T;
  int n1 = (T + K0 - 1) / K0;
  p.n[1] = n1;  // level-1 rows also serve the block aggregates when L == 0
  if (n1 <= 1) { p.L = 0; return p; }
  int l = 1;
  while (p.n[l] > K && l < kMaxLevels) {
    p.n[l + 1] = (p.n[l] + K - 1) / K;
    ++l;
  }
  p.L = l;
  return p;
}

template <typename R>
PTC_HD R rzero() { return R(0); }

}  // namespace ptc
