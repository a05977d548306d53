// C ABI implementation (include/pintoc_b200.h): workspace carving, the
// batched solver object and dispatch into the instantiated kernel sets.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pintoc_b200.h"
#include "launch.cuh"

namespace ptc {

std::map<LqrKey, LqrOps>& lqr_registry() {
  static std::map<LqrKey, LqrOps> r;
  return r;
}
std::map<NewtonKey, NewtonOps>& newton_registry() {
  static std::map<NewtonKey, NewtonOps> r;
  return r;
}

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define PTC_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess)                                                    \
      return fail(PTC_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(_e)); \
  } while (0)

// ------------------------------------------------------------------ planning

// Automatic scan plan.  Large batches fill the GPU on their own: one thread
// per problem sweeps its horizon (no tree, work optimal).  Small batches
// split the horizon into chunks of K0 stages so that ~32K threads are busy,
// with a 4-ary tree above them (log-depth in the horizon).
static Plan auto_plan(int B, int T, int K0, int K, int nx = 0) {
  const bool wide = nx >= 8;
  // tree fan-out: each level above the leaves costs K serial combines of
  // one unit, and the log-depth levels are latency-bound, so a narrow tree
  // wins: K = 4 measured 4-17% faster than 8 for nx = 12 at T = 2^10 ..
  // 2^20 and 20-29% faster for nx = 2 / 4 at T = 2^12 .. 2^16, batch 1
  // (gpurun r119, r121); K = 2 doubles the levels and loses again.  Batched
  // thread-kernel trees (the strong-scaling shares, 2K-8K problems) keep
  // K = 8: there the levels are wide and K = 4 measured ~10% slower (r122)
  if (K <= 0) K = (wide || B < 256) ? 4 : 8;
  if (K0 <= 0) {
    const long long work = (long long)B * T;
    // thread-per-unit kernels want ~32K units; the warp-per-unit kernels of
    // nx >= 8 (wide.cuh) ~8K warps and level-0 chunks of at least 16 stages
    const long long units = wide ? 8192 : 32768;
    // one sweep per problem (work-optimal) once the batch alone keeps the
    // GPU busy: measured crossover between 8K (tree 15% faster) and 16K
    // (sweep 25% faster) problems per launch (nx = 2 / 4, T = 256)
    if (B >= 16384) K0 = T;
    else K0 = (int)std::max<long long>(wide ? 16 : 4, (work + units - 1) / units);
  }
  return make_plan(T, K0, K);
}

struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

template <typename R>
static void carve_lqr_tree(Carver& c, LqrArgs<R>& a, int nx, int nu) {
  const Plan& pl = a.plan;
  const size_t B = a.B;
  a.red = c.template take<double>(3 * (size_t)pl.units0() * B);
  // single long wide problem: stage-major copies of the expansion and of the
  // gains (wide.cuh "staged" mode) make every per-stage access contiguous
  a.xst = a.gst = nullptr;
  if (B == 1 && nx >= 8 && a.T >= 1024) {
    const size_t sc = (size_t)nx * nx + nu * nu + nx * nu + nu + nx * nx + nx * nu;
    a.xst = c.template take<R>((size_t)a.T * sc);
    a.gst = c.template take<R>((size_t)a.T * (nu * nx + nu));
  }
  for (int l = 0; l <= kMaxLevels; ++l)
    a.vagg[l] = a.vcar[l] = a.pagg[l] = a.pcar[l] = a.vhalf[l] = nullptr;
  a.vcin_buf = a.xin_buf = nullptr;
  if (a.block_mode) {
    a.vcin_buf = c.template take<R>(B * (nx * nx + nx));
    a.xin_buf = c.template take<R>(B * nx);
  }
  const int top = (a.block_mode && pl.L == 0) ? 1 : pl.L;
  for (int l = 1; l <= top; ++l) {
    const size_t n = (size_t)pl.n[l] * B;
    a.vagg[l] = c.template take<R>(n * (3 * nx * nx + 2 * nx));
    a.vcar[l] = c.template take<R>(n * (nx * nx + nx));
    a.pagg[l] = c.template take<R>(n * (nx * nx + nx));
    a.pcar[l] = c.template take<R>(n * nx);
  }
  // split-fold levels of the warp kernels keep their upper-half aggregates
  if (nx >= 8)
    for (int l = 1; l < pl.L; ++l)
      if ((long long)pl.n[l + 1] * a.B <= kUp2MaxUnits)
        a.vhalf[l] = c.template take<R>((size_t)pl.n[l + 1] * B * (3 * nx * nx + 2 * nx));
}

}  // namespace ptc

using namespace ptc;

extern "C" {

const char* ptc_last_error(void) { return g_err.c_str(); }

int ptc_version(void) { return 100; }

int ptc_supported(int dtype, int model, int nx, int nu) {
  if (model < 0) return lqr_registry().count(LqrKey(dtype, nx, nu)) ? 1 : 0;
  return newton_registry().count(NewtonKey(dtype, model, nx, nu)) ? 1 : 0;
}

int ptc_lqr_plan(int batch, int horizon, int nx, int chunk0, int chunk, int* out_chunk0,
                 int* out_chunk, int* out_levels) {
  if (batch < 1 || horizon < 1) return fail(PTC_ERR_ARG, "batch and horizon must be >= 1");
  Plan p = auto_plan(batch, horizon, chunk0, chunk, nx);
  if (out_chunk0) *out_chunk0 = p.K0;
  if (out_chunk) *out_chunk = p.K;
  if (out_levels) *out_levels = p.L;
  return PTC_OK;
}

int64_t ptc_lqr_workspace_bytes(int dtype, int batch, int horizon, int nx, int nu, int chunk0,
                                int chunk) {
  if (batch < 1 || horizon < 1 || nx < 1 || nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  Carver c{nullptr};
  if (dtype == PTC_F64) {
    LqrArgs<double> a{};
    a.B = batch;
    a.T = horizon;
    a.plan = auto_plan(batch, horizon, chunk0, chunk, nx);
    carve_lqr_tree(c, a, nx, nu);
  } else {
    LqrArgs<float> a{};
    a.B = batch;
    a.T = horizon;
    a.plan = auto_plan(batch, horizon, chunk0, chunk, nx);
    carve_lqr_tree(c, a, nx, nu);
  }
  return (int64_t)c.off + 256;
}

}  // extern "C"

// Graph cache of LQR launch sequences keyed by the full argument block
// (plain-old-data, zero-initialised so padding compares equal).
struct LqrGraph {
  std::vector<unsigned char> key;
  cudaGraphExec_t exec;
};

template <typename R>
static cudaGraphExec_t lqr_graph_for(const LqrArgs<R>& a, const LqrOps& ops, cudaStream_t) {
  static thread_local std::vector<LqrGraph> cache;
  static thread_local cudaStream_t cap = nullptr;
  const unsigned char* kb = reinterpret_cast<const unsigned char*>(&a);
  std::vector<unsigned char> key(kb, kb + sizeof(a));
  // the kernel set (dtype, nx, nu) is not part of LqrArgs: key on it too
  const uintptr_t fn = reinterpret_cast<uintptr_t>(ops.solve);
  const unsigned char* fb = reinterpret_cast<const unsigned char*>(&fn);
  key.insert(key.end(), fb, fb + sizeof(fn));
  key.push_back((unsigned char)sizeof(R));
  for (auto& g : cache)
    if (g.key == key) return g.exec;
  if (!cap && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ex = nullptr;
  bool ok = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    ops.solve(&a, cap);
    ok = cudaStreamEndCapture(cap, &g) == cudaSuccess && g != nullptr;
  }
  if (ok) ok = cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
  if (g) cudaGraphDestroy(g);
  if (!ok) {
    (void)cudaGetLastError();
    return nullptr;
  }
  if (cache.size() >= 32) {
    cudaGraphExecDestroy(cache.front().exec);
    cache.erase(cache.begin());
  }
  cache.push_back(LqrGraph{std::move(key), ex});
  return ex;
}

template <typename R>
static int lqr_solve_t(int batch, int horizon, int nx, int nu, const void* P, const void* Rm,
                       const void* M, const void* d, const void* Fx, const void* Fu,
                       const void* PT, const double* alpha, void* S, void* s, void* Gamma,
                       void* gamma, void* dx, void* du, int* flags, void* ws, int64_t ws_bytes,
                       int chunk0, int chunk, cudaStream_t st, const void* rows = nullptr) {
  auto it = lqr_registry().find(LqrKey(dtype_code<R>(), nx, nu));
  if (it == lqr_registry().end())
    return fail(PTC_ERR_UNSUPPORTED, "LQR kernels not instantiated for nx=" + std::to_string(nx) +
                                         " nu=" + std::to_string(nu));
  LqrArgs<R> a;
  std::memset(&a, 0, sizeof(a));  // padding too: the graph cache keys on the bytes
  a.B = batch;
  a.T = horizon;
  a.plan = auto_plan(batch, horizon, chunk0, chunk, nx);
  a.auto_plan = chunk0 == 0 && chunk == 0;
  a.P = (const R*)P;
  a.Rm = (const R*)Rm;
  a.M = (const R*)M;
  a.d = (const R*)d;
  a.Fx = (const R*)Fx;
  a.Fu = (const R*)Fu;
  a.PT = (const R*)PT;
  a.alpha = alpha;
  a.status = nullptr;
  a.S = (R*)S;
  a.s = (R*)s;
  a.Gam = (R*)Gamma;
  a.gam = (R*)gamma;
  a.dX = (R*)dx;
  a.dU = (R*)du;
  a.flags = flags;
  Carver c{(char*)ws};
  carve_lqr_tree(c, a, nx, nu);
  if ((int64_t)c.off > ws_bytes) return fail(PTC_ERR_WORKSPACE, "LQR workspace too small");
  if ((S == nullptr) != (s == nullptr)) return fail(PTC_ERR_ARG, "S and s must both be given or both NULL");
  a.red = nullptr;  // trust-region partial sums are a Newton-loop product only
  if (rows) {  // stage rows: the caller's buffer is the staging buffer
    if (!a.xst) return fail(PTC_ERR_ARG, "stage-row inputs need batch 1, nx >= 8, horizon >= 1024");
    a.xst = (R*)rows;
    a.prestaged = 1;
  }
  if (a.plan.L >= 1 && !getenv("PTC_NO_GRAPH")) {
    // a tree plan is 4L+4 short launches: replay them as one CUDA graph,
    // cached per argument set (same buffers -> same graph)
    cudaGraphExec_t ex = lqr_graph_for(a, it->second, st);
    if (ex) {
      PTC_CUDA(cudaGraphLaunch(ex, st));
      return PTC_OK;
    }
  }
  it->second.solve(&a, st);
  PTC_CUDA(cudaGetLastError());
  return PTC_OK;
}

template <typename R>
static int propagate_t(int batch, int horizon, int nx, int nu, const void* Fx, const void* Fu,
                       const void* Gamma, const void* gamma, const void* d, void* dx, void* du,
                       void* ws, int64_t ws_bytes, int chunk0, int chunk, cudaStream_t st) {
  auto it = lqr_registry().find(LqrKey(dtype_code<R>(), nx, nu));
  if (it == lqr_registry().end())
    return fail(PTC_ERR_UNSUPPORTED, "LQR kernels not instantiated for nx=" + std::to_string(nx) +
                                         " nu=" + std::to_string(nu));
  LqrArgs<R> a{};
  a.B = batch;
  a.T = horizon;
  a.plan = auto_plan(batch, horizon, chunk0, chunk, nx);
  a.Fx = (const R*)Fx;
  a.Fu = (const R*)Fu;
  a.d = (const R*)d;
  a.Gam = (R*)Gamma;
  a.gam = (R*)gamma;
  a.dX = (R*)dx;
  a.dU = (R*)du;
  Carver c{(char*)ws};
  carve_lqr_tree(c, a, nx, nu);
  if ((int64_t)c.off > ws_bytes) return fail(PTC_ERR_WORKSPACE, "LQR workspace too small");
  a.red = nullptr;  // no trust-region partial sums outside the Newton loop
  it->second.propagate(&a, st);
  PTC_CUDA(cudaGetLastError());
  return PTC_OK;
}

extern "C" {

int ptc_propagate(int dtype, int batch, int horizon, int nx, int nu, const void* Fx,
                  const void* Fu, const void* Gamma, const void* gamma, const void* d, void* dx,
                  void* du, void* workspace, int64_t workspace_bytes, int chunk0, int chunk,
                  void* stream) {
  if (batch < 1 || horizon < 1 || nx < 1 || nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == PTC_F64)
    return propagate_t<double>(batch, horizon, nx, nu, Fx, Fu, Gamma, gamma, d, dx, du, workspace,
                               workspace_bytes, chunk0, chunk, st);
  if (dtype == PTC_F32)
    return propagate_t<float>(batch, horizon, nx, nu, Fx, Fu, Gamma, gamma, d, dx, du, workspace,
                              workspace_bytes, chunk0, chunk, st);
  return fail(PTC_ERR_ARG, "dtype must be PTC_F32 or PTC_F64");
}

int ptc_lqr_block_comps(int nx, int* value_comps, int* prop_comps) {
  if (nx < 1) return fail(PTC_ERR_ARG, "nx must be >= 1");
  if (value_comps) *value_comps = 3 * nx * nx + 2 * nx;
  if (prop_comps) *prop_comps = nx * nx + nx;
  return PTC_OK;
}

int64_t ptc_lqr_block_workspace_bytes(int dtype, int batch, int horizon, int nx, int nu,
                                      int chunk0, int chunk) {
  if (batch < 1 || horizon < 1 || nx < 1 || nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  Carver c{nullptr};
  if (dtype == PTC_F64) {
    LqrArgs<double> a{};
    a.B = batch;
    a.T = horizon;
    a.block_mode = 1;
    a.plan = auto_plan(batch, horizon, chunk0, chunk, nx);
    carve_lqr_tree(c, a, nx, nu);
  } else {
    LqrArgs<float> a{};
    a.B = batch;
    a.T = horizon;
    a.block_mode = 1;
    a.plan = auto_plan(batch, horizon, chunk0, chunk, nx);
    carve_lqr_tree(c, a, nx, nu);
  }
  return (int64_t)c.off + 256;
}

static int lqr_block_solve_impl(int phase, int dtype, int batch, int horizon, int nx, int nu,
                                int t_base, int is_last, int rank, int world, const void* P,
                                const void* R, const void* M, const void* d, const void* Fx,
                                const void* Fu, const void* rows, const void* PT,
                                const double* alpha, const void* blocks_in, void* block_out,
                                void* S, void* s, void* Gamma, void* gamma, void* dx, void* du,
                                int* flags, void* workspace, int64_t workspace_bytes, int chunk0,
                                int chunk, void* stream);

int ptc_lqr_block_solve(int phase, int dtype, int batch, int horizon, int nx, int nu, int t_base,
                        int is_last, int rank, int world, const void* P, const void* R,
                        const void* M, const void* d, const void* Fx, const void* Fu,
                        const void* PT, const double* alpha, const void* blocks_in,
                        void* block_out, void* S, void* s, void* Gamma, void* gamma, void* dx,
                        void* du, int* flags, void* workspace, int64_t workspace_bytes,
                        int chunk0, int chunk, void* stream) {
  if (!P || !R || !M || !d || !Fx || !Fu) return fail(PTC_ERR_ARG, "missing expansion buffer");
  return lqr_block_solve_impl(phase, dtype, batch, horizon, nx, nu, t_base, is_last, rank, world,
                              P, R, M, d, Fx, Fu, nullptr, PT, alpha, blocks_in, block_out, S, s,
                              Gamma, gamma, dx, du, flags, workspace, workspace_bytes, chunk0,
                              chunk, stream);
}

int ptc_lqr_block_solve_rows(int phase, int dtype, int horizon, int nx, int nu, int t_base,
                             int is_last, int rank, int world, const void* rows, const void* PT,
                             const double* alpha, const void* blocks_in, void* block_out,
                             void* S, void* s, void* Gamma, void* gamma, void* dx, void* du,
                             int* flags, void* workspace, int64_t workspace_bytes, int chunk0,
                             int chunk, void* stream) {
  if (!rows) return fail(PTC_ERR_ARG, "rows is required");
  if (nx < 8) return fail(PTC_ERR_UNSUPPORTED, "stage-row inputs are read by the nx >= 8 kernels");
  if (horizon < 1024) return fail(PTC_ERR_ARG, "stage-row inputs need a block of >= 1024 stages");
  return lqr_block_solve_impl(phase, dtype, 1, horizon, nx, nu, t_base, is_last, rank, world,
                              nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, rows, PT,
                              alpha, blocks_in, block_out, S, s, Gamma, gamma, dx, du, flags,
                              workspace, workspace_bytes, chunk0, chunk, stream);
}

static int lqr_block_solve_impl(int phase, int dtype, int batch, int horizon, int nx, int nu,
                                int t_base, int is_last, int rank, int world, const void* P,
                                const void* R, const void* M, const void* d, const void* Fx,
                                const void* Fu, const void* rows, const void* PT,
                                const double* alpha, const void* blocks_in, void* block_out,
                                void* S, void* s, void* Gamma, void* gamma, void* dx, void* du,
                                int* flags, void* workspace, int64_t workspace_bytes, int chunk0,
                                int chunk, void* stream) {
  if (batch < 1 || horizon < 1 || nx < 1 || nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  if (phase < 0 || phase > 2) return fail(PTC_ERR_ARG, "phase must be 0, 1 or 2");
  if (world < 1 || rank < 0 || rank >= world) return fail(PTC_ERR_ARG, "bad rank / world");
  if (t_base < 0) return fail(PTC_ERR_ARG, "t_base must be >= 0");
  if (phase > 0 && blocks_in == nullptr) return fail(PTC_ERR_ARG, "phase 1/2 need blocks_in");
  if (phase < 2 && block_out == nullptr) return fail(PTC_ERR_ARG, "phase 0/1 need block_out");
  if (is_last && PT == nullptr) return fail(PTC_ERR_ARG, "the last block needs PT");
  if ((S == nullptr) != (s == nullptr)) return fail(PTC_ERR_ARG, "S and s must both be given or both NULL");
  cudaStream_t st = (cudaStream_t)stream;
  auto run = [&](auto zero) -> int {
    using Rt = decltype(zero);
    auto it = lqr_registry().find(LqrKey(dtype_code<Rt>(), nx, nu));
    if (it == lqr_registry().end())
      return fail(PTC_ERR_UNSUPPORTED, "LQR kernels not instantiated for nx=" +
                                           std::to_string(nx) + " nu=" + std::to_string(nu));
    LqrArgs<Rt> a{};
    a.B = batch;
    a.T = horizon;
    a.plan = auto_plan(batch, horizon, chunk0, chunk, nx);
    a.block_mode = 1;
    a.t_base = t_base;
    a.no_terminal = is_last ? 0 : 1;
    a.P = (const Rt*)P;
    a.Rm = (const Rt*)R;
    a.M = (const Rt*)M;
    a.d = (const Rt*)d;
    a.Fx = (const Rt*)Fx;
    a.Fu = (const Rt*)Fu;
    a.PT = (const Rt*)PT;
    a.alpha = alpha;
    a.S = (Rt*)S;
    a.s = (Rt*)s;
    a.Gam = (Rt*)Gamma;
    a.gam = (Rt*)gamma;
    a.dX = (Rt*)dx;
    a.dU = (Rt*)du;
    a.flags = flags;
    Carver c{(char*)workspace};
    carve_lqr_tree(c, a, nx, nu);
    if ((int64_t)c.off > workspace_bytes) return fail(PTC_ERR_WORKSPACE, "LQR workspace too small");
    if (rows) {  // the caller's stage rows are the staging buffer: no transpose
      a.xst = (Rt*)rows;
      a.prestaged = 1;
    }
    it->second.block(&a, phase, blocks_in, block_out, rank, world, st);
    PTC_CUDA(cudaGetLastError());
    return PTC_OK;
  };
  if (dtype == PTC_F64) return run(0.0);
  if (dtype == PTC_F32) return run(0.0f);
  return fail(PTC_ERR_ARG, "dtype must be PTC_F32 or PTC_F64");
}

}  // extern "C"

// device staging of the host-buffer entry: inputs, alpha, flags, outputs
template <typename R>
static size_t host_staging(Carver& c, int batch, int horizon, int nx, int nu, R** in, double** al,
                           int** fl, R** out) {
  const size_t TB = (size_t)horizon * batch, B = batch;
  const size_t ci[7] = {(size_t)nx * nx * TB, (size_t)nu * nu * TB, (size_t)nx * nu * TB,
                        (size_t)nu * TB, (size_t)nx * nx * TB, (size_t)nx * nu * TB,
                        (size_t)nx * nx * B};
  for (int k = 0; k < 7; ++k) in[k] = c.template take<R>(ci[k]);
  *al = c.template take<double>(B);
  *fl = c.template take<int>(B);
  const size_t co[4] = {(size_t)nu * nx * TB, (size_t)nu * TB, (size_t)nx * (horizon + 1) * B,
                        (size_t)nu * TB};
  for (int k = 0; k < 4; ++k) out[k] = c.template take<R>(co[k]);
  return c.off;
}

template <typename R>
static int lqr_solve_host_t(int batch, int horizon, int nx, int nu, const void* const* hin,
                            const double* alpha, void* const* hout, int* flags, void* ws,
                            int64_t ws_bytes, int chunk0, int chunk, cudaStream_t st) {
  Carver c{(char*)ws};
  R* in[7];
  R* out[4];
  double* al;
  int* fl;
  host_staging<R>(c, batch, horizon, nx, nu, in, &al, &fl, out);
  c.off = (c.off + 255) & ~(size_t)255;
  const int64_t rest = ws_bytes - (int64_t)c.off;
  if (rest <= 0) return fail(PTC_ERR_WORKSPACE, "LQR host workspace too small");
  const size_t TB = (size_t)horizon * batch, es = sizeof(R);
  auto h2d = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  };
  // only what the kernels read crosses PCIe: the thread-per-unit kernels
  // (nx < 8) read the upper triangles of the symmetric P and R
  // (elements.cuh ld_stage); the warp kernels read whole stage rows
  auto sym_copy = [&](R* dst, const void* src, int n) -> cudaError_t {
    if (nx >= 8) return h2d(dst, src, (size_t)n * n * TB * es);
    for (int i = 0; i < n; ++i) {
      // components i*n + i .. i*n + n-1 of one row are contiguous slabs
      const size_t c0 = (size_t)i * n + i;
      cudaError_t e = h2d(dst + c0 * TB, static_cast<const R*>(src) + c0 * TB,
                          (size_t)(n - i) * TB * es);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  };
  PTC_CUDA(sym_copy(in[0], hin[0], nx));
  PTC_CUDA(sym_copy(in[1], hin[1], nu));
  PTC_CUDA(h2d(in[2], hin[2], (size_t)nx * nu * TB * es));
  PTC_CUDA(h2d(in[3], hin[3], (size_t)nu * TB * es));
  PTC_CUDA(h2d(in[4], hin[4], (size_t)nx * nx * TB * es));
  PTC_CUDA(h2d(in[5], hin[5], (size_t)nx * nu * TB * es));
  PTC_CUDA(h2d(in[6], hin[6], (size_t)nx * nx * batch * es));
  PTC_CUDA(h2d(al, alpha, (size_t)batch * sizeof(double)));
  PTC_CUDA(cudaMemsetAsync(fl, 0, sizeof(int) * batch, st));
  int rc = lqr_solve_t<R>(batch, horizon, nx, nu, in[0], in[1], in[2], in[3], in[4], in[5], in[6],
                          al, nullptr, nullptr, out[0], out[1], out[2], out[3], fl,
                          (char*)ws + c.off, rest, chunk0, chunk, st);
  if (rc != PTC_OK) return rc;
  const size_t ob[4] = {(size_t)nu * nx * TB * es, (size_t)nu * TB * es,
                        (size_t)nx * (horizon + 1) * batch * es, (size_t)nu * TB * es};
  for (int k = 0; k < 4; ++k)
    PTC_CUDA(cudaMemcpyAsync(hout[k], out[k], ob[k], cudaMemcpyDeviceToHost, st));
  if (flags) PTC_CUDA(cudaMemcpyAsync(flags, fl, sizeof(int) * batch, cudaMemcpyDeviceToHost, st));
  return PTC_OK;
}

// problem-major <-> SoA batch-minor restack of one field with C components
// over `rows` stages: stacked[(b * rows + t) * C + c] <-> soa[(c * rows + t) *
// B + b].  Flattening k = t * C + c makes it a [B][K] <-> [K][B] transpose
// with the SoA row of k remapped to c * rows + t; 32 x 32 smem tiles keep
// both sides coalesced (256 B per warp access in fp64).
template <typename R, bool kToSoa>
__global__ void __launch_bounds__(256) k_restack(const R* __restrict__ in, R* __restrict__ out,
                                                 int B, int rows, int C) {
  __shared__ R tile[32][33];
  const long long K = (long long)rows * C, k0 = (long long)blockIdx.x * 32;
  const int b0 = blockIdx.y * 32, tx = threadIdx.x;
  auto soa = [&](long long k, int b) {
    return ((long long)(k % C) * rows + k / C) * B + b;
  };
#pragma unroll
  for (int j = threadIdx.y; j < 32; j += 8) {
    if (kToSoa) {
      const int b = b0 + j;
      const long long k = k0 + tx;
      if (b < B && k < K) tile[j][tx] = in[(long long)b * K + k];
    } else {
      const long long k = k0 + j;
      const int b = b0 + tx;
      if (b < B && k < K) tile[j][tx] = in[soa(k, b)];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = threadIdx.y; j < 32; j += 8) {
    if (kToSoa) {
      const long long k = k0 + j;
      const int b = b0 + tx;
      if (b < B && k < K) out[soa(k, b)] = tile[tx][j];
    } else {
      const int b = b0 + j;
      const long long k = k0 + tx;
      if (b < B && k < K) out[(long long)b * K + k] = tile[tx][j];
    }
  }
}

template <typename R>
static void restack(const R* in, R* out, int B, int rows, int C, bool to_soa, cudaStream_t st) {
  const dim3 grid((unsigned)(((long long)rows * C + 31) / 32), (unsigned)((B + 31) / 32));
  if (to_soa) k_restack<R, true><<<grid, dim3(32, 8), 0, st>>>(in, out, B, rows, C);
  else k_restack<R, false><<<grid, dim3(32, 8), 0, st>>>(in, out, B, rows, C);
}

// the host entry for the reference's own per-problem arrays stacked over the
// batch: each field crosses PCIe whole into one device staging buffer and is
// restacked into the SoA inputs there; the outputs go the other way
// (every input field side by side: the copies of one call run back to back,
// then the restacks; the outputs reuse the space)
static size_t stacked_raw_words(int batch, int horizon, int nx, int nu) {
  const size_t TB = (size_t)horizon * batch;
  const size_t in = (size_t)(2 * nx * nx + nu * nu + 2 * nx * nu + nu) * TB + (size_t)nx * nx * batch;
  const size_t out = (size_t)(nu * nx + 2 * nu) * TB + (size_t)nx * (horizon + 1) * batch;
  return std::max(in, out);
}

template <typename R>
static int lqr_solve_host_stacked_t(int batch, int horizon, int nx, int nu,
                                    const void* const* hin, const double* alpha,
                                    void* const* hout, int* flags, void* ws, int64_t ws_bytes,
                                    int chunk0, int chunk, cudaStream_t st) {
  if (batch > 65535 * 32) return fail(PTC_ERR_ARG, "stacked layout: batch above 2,097,120");
  Carver c{(char*)ws};
  R* in[7];
  R* out[4];
  double* al;
  int* fl;
  host_staging<R>(c, batch, horizon, nx, nu, in, &al, &fl, out);
  R* raw = c.template take<R>(stacked_raw_words(batch, horizon, nx, nu));
  c.off = (c.off + 255) & ~(size_t)255;
  const int64_t rest = ws_bytes - (int64_t)c.off;
  if (rest <= 0) return fail(PTC_ERR_WORKSPACE, "LQR host workspace too small");
  const size_t es = sizeof(R);
  const int cin[7] = {nx * nx, nu * nu, nx * nu, nu, nx * nx, nx * nu, nx * nx};
  size_t off[8] = {0};
  for (int k = 0; k < 7; ++k) off[k + 1] = off[k] + (size_t)cin[k] * (k == 6 ? 1 : horizon) * batch;
  for (int k = 0; k < 7; ++k)
    PTC_CUDA(cudaMemcpyAsync(raw + off[k], hin[k], (off[k + 1] - off[k]) * es,
                             cudaMemcpyHostToDevice, st));
  for (int k = 0; k < 7; ++k) restack<R>(raw + off[k], in[k], batch, k == 6 ? 1 : horizon, cin[k], true, st);
  PTC_CUDA(cudaMemcpyAsync(al, alpha, (size_t)batch * sizeof(double), cudaMemcpyHostToDevice, st));
  PTC_CUDA(cudaMemsetAsync(fl, 0, sizeof(int) * batch, st));
  int rc = lqr_solve_t<R>(batch, horizon, nx, nu, in[0], in[1], in[2], in[3], in[4], in[5], in[6],
                          al, nullptr, nullptr, out[0], out[1], out[2], out[3], fl,
                          (char*)ws + c.off, rest, chunk0, chunk, st);
  if (rc != PTC_OK) return rc;
  const int cout_[4] = {nu * nx, nu, nx, nu};
  size_t oo[5] = {0};
  for (int k = 0; k < 4; ++k) oo[k + 1] = oo[k] + (size_t)cout_[k] * (k == 2 ? horizon + 1 : horizon) * batch;
  for (int k = 0; k < 4; ++k)
    restack<R>(out[k], raw + oo[k], batch, k == 2 ? horizon + 1 : horizon, cout_[k], false, st);
  for (int k = 0; k < 4; ++k)
    PTC_CUDA(cudaMemcpyAsync(hout[k], raw + oo[k], (oo[k + 1] - oo[k]) * es,
                             cudaMemcpyDeviceToHost, st));
  if (flags) PTC_CUDA(cudaMemcpyAsync(flags, fl, sizeof(int) * batch, cudaMemcpyDeviceToHost, st));
  PTC_CUDA(cudaGetLastError());
  return PTC_OK;
}

extern "C" {

int64_t ptc_lqr_host_stacked_workspace_bytes(int dtype, int batch, int horizon, int nx, int nu,
                                             int chunk0, int chunk) {
  const int64_t hw = ptc_lqr_host_workspace_bytes(dtype, batch, horizon, nx, nu, chunk0, chunk);
  if (hw < 0) return hw;
  const size_t es = dtype == PTC_F64 ? 8 : 4;
  return hw + (int64_t)((stacked_raw_words(batch, horizon, nx, nu) * es + 511) & ~(size_t)255);
}

int ptc_lqr_solve_host_stacked(int dtype, int batch, int horizon, int nx, int nu, const void* P,
                               const void* R, const void* M, const void* d, const void* Fx,
                               const void* Fu, const void* PT, const double* alpha, void* Gamma,
                               void* gamma, void* dx, void* du, int* flags, void* workspace,
                               int64_t workspace_bytes, int chunk0, int chunk, void* stream) {
  if (batch < 1 || horizon < 1 || nx < 1 || nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  const void* hin[7] = {P, R, M, d, Fx, Fu, PT};
  for (const void* p : hin)
    if (!p) return fail(PTC_ERR_ARG, "every input buffer is required");
  void* hout[4] = {Gamma, gamma, dx, du};
  for (void* p : hout)
    if (!p) return fail(PTC_ERR_ARG, "every output buffer is required");
  if (!alpha) return fail(PTC_ERR_ARG, "alpha is required");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == PTC_F64)
    return lqr_solve_host_stacked_t<double>(batch, horizon, nx, nu, hin, alpha, hout, flags,
                                            workspace, workspace_bytes, chunk0, chunk, st);
  if (dtype == PTC_F32)
    return lqr_solve_host_stacked_t<float>(batch, horizon, nx, nu, hin, alpha, hout, flags,
                                           workspace, workspace_bytes, chunk0, chunk, st);
  return fail(PTC_ERR_ARG, "dtype must be PTC_F32 or PTC_F64");
}

// element-level entry points: any registered kernel set of this dtype / nx
static const LqrOps* ops_for_nx(int dtype, int nx) {
  const int code = dtype == PTC_F64 ? 1 : 0;
  for (auto& kv : lqr_registry())
    if (std::get<0>(kv.first) == code && std::get<1>(kv.first) == nx) return &kv.second;
  return nullptr;
}

int ptc_value_elements(int dtype, int horizon, int nx, int nu, const void* P, const void* R,
                       const void* M, const void* d, const void* Fx, const void* Fu,
                       const void* PT, const double* alpha, void* out, int* flags, void* stream) {
  if (horizon < 0 || nx < 1 || nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  if (dtype != PTC_F32 && dtype != PTC_F64) return fail(PTC_ERR_ARG, "bad dtype");
  if (!PT || !alpha || !out || !flags || (horizon > 0 && (!P || !R || !M || !d || !Fx || !Fu)))
    return fail(PTC_ERR_ARG, "missing buffer");
  auto it = lqr_registry().find(LqrKey(dtype == PTC_F64 ? 1 : 0, nx, nu));
  if (it == lqr_registry().end())
    return fail(PTC_ERR_UNSUPPORTED, "kernels not instantiated for nx=" + std::to_string(nx) +
                                         " nu=" + std::to_string(nu));
  const void* st[7] = {P, R, M, d, Fx, Fu, PT};
  it->second.velem_init(horizon, st, alpha, out, flags, (cudaStream_t)stream);
  PTC_CUDA(cudaGetLastError());
  return PTC_OK;
}

int ptc_lqr_diagnose(int dtype, int batch, int horizon, int nx, int nu, const void* P,
                     const void* R, const void* M, const void* d, const void* Fx, const void* Fu,
                     const void* PT, const double* alpha, int* out, void* stream) {
  if (batch < 1 || horizon < 1 || nx < 1 || nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  if (dtype != PTC_F32 && dtype != PTC_F64) return fail(PTC_ERR_ARG, "bad dtype");
  if (!P || !R || !M || !d || !Fx || !Fu || !PT || !alpha || !out)
    return fail(PTC_ERR_ARG, "missing buffer");
  auto it = lqr_registry().find(LqrKey(dtype == PTC_F64 ? 1 : 0, nx, nu));
  if (it == lqr_registry().end())
    return fail(PTC_ERR_UNSUPPORTED, "kernels not instantiated for nx=" + std::to_string(nx) +
                                         " nu=" + std::to_string(nu));
  const void* st[7] = {P, R, M, d, Fx, Fu, PT};
  it->second.diagnose(batch, horizon, st, alpha, out, (cudaStream_t)stream);
  PTC_CUDA(cudaGetLastError());
  return PTC_OK;
}

int ptc_value_combine(int dtype, int n, int nx, const void* left, const void* right, void* out,
                      int* flags, void* stream) {
  if (n < 1 || nx < 1) return fail(PTC_ERR_ARG, "bad dims");
  if (!left || !right || !out || !flags) return fail(PTC_ERR_ARG, "missing buffer");
  const LqrOps* ops = ops_for_nx(dtype, nx);
  if (!ops) return fail(PTC_ERR_UNSUPPORTED, "kernels not instantiated for nx=" + std::to_string(nx));
  ops->vcombine(n, left, right, out, flags, (cudaStream_t)stream);
  PTC_CUDA(cudaGetLastError());
  return PTC_OK;
}

int ptc_affine_combine(int dtype, int n, int nx, int kind, const void* a, const void* b, void* out,
                       void* stream) {
  if (n < 1 || nx < 1) return fail(PTC_ERR_ARG, "bad dims");
  if (kind != 0 && kind != 1) return fail(PTC_ERR_ARG, "kind must be 0 (rollout) or 1 (costate)");
  if (!a || !b || !out) return fail(PTC_ERR_ARG, "missing buffer");
  const LqrOps* ops = ops_for_nx(dtype, nx);
  if (!ops) return fail(PTC_ERR_UNSUPPORTED, "kernels not instantiated for nx=" + std::to_string(nx));
  ops->affine(n, kind, a, b, out, (cudaStream_t)stream);
  PTC_CUDA(cudaGetLastError());
  return PTC_OK;
}

int64_t ptc_lqr_host_workspace_bytes(int dtype, int batch, int horizon, int nx, int nu,
                                     int chunk0, int chunk) {
  const int64_t lw = ptc_lqr_workspace_bytes(dtype, batch, horizon, nx, nu, chunk0, chunk);
  if (lw < 0) return lw;
  Carver c{nullptr};
  double* al;
  int* fl;
  if (dtype == PTC_F64) {
    double *in[7], *out[4];
    host_staging<double>(c, batch, horizon, nx, nu, in, &al, &fl, out);
  } else {
    float *in[7], *out[4];
    host_staging<float>(c, batch, horizon, nx, nu, in, &al, &fl, out);
  }
  return (int64_t)((c.off + 255) & ~(size_t)255) + lw;
}

int ptc_lqr_solve_host(int dtype, int batch, int horizon, int nx, int nu, const void* P,
                       const void* R, const void* M, const void* d, const void* Fx,
                       const void* Fu, const void* PT, const double* alpha, void* Gamma,
                       void* gamma, void* dx, void* du, int* flags, void* workspace,
                       int64_t workspace_bytes, int chunk0, int chunk, void* stream) {
  if (batch < 1 || horizon < 1 || nx < 1 || nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  const void* hin[7] = {P, R, M, d, Fx, Fu, PT};
  for (const void* p : hin)
    if (!p) return fail(PTC_ERR_ARG, "every input buffer is required");
  void* hout[4] = {Gamma, gamma, dx, du};
  for (void* p : hout)
    if (!p) return fail(PTC_ERR_ARG, "every output buffer is required");
  if (!alpha) return fail(PTC_ERR_ARG, "alpha is required");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == PTC_F64)
    return lqr_solve_host_t<double>(batch, horizon, nx, nu, hin, alpha, hout, flags, workspace,
                                    workspace_bytes, chunk0, chunk, st);
  if (dtype == PTC_F32)
    return lqr_solve_host_t<float>(batch, horizon, nx, nu, hin, alpha, hout, flags, workspace,
                                   workspace_bytes, chunk0, chunk, st);
  return fail(PTC_ERR_ARG, "dtype must be PTC_F32 or PTC_F64");
}

int ptc_lqr_solve_rows(int dtype, int horizon, int nx, int nu, const void* rows, const void* PT,
                       const double* alpha, void* S, void* s, void* Gamma, void* gamma, void* dx,
                       void* du, int* flags, void* workspace, int64_t workspace_bytes, int chunk0,
                       int chunk, void* stream) {
  if (horizon < 1 || nx < 1 || nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  if (!rows) return fail(PTC_ERR_ARG, "rows is required");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == PTC_F64)
    return lqr_solve_t<double>(1, horizon, nx, nu, nullptr, nullptr, nullptr, nullptr, nullptr,
                               nullptr, PT, alpha, S, s, Gamma, gamma, dx, du, flags, workspace,
                               workspace_bytes, chunk0, chunk, st, rows);
  if (dtype == PTC_F32)
    return lqr_solve_t<float>(1, horizon, nx, nu, nullptr, nullptr, nullptr, nullptr, nullptr,
                              nullptr, PT, alpha, S, s, Gamma, gamma, dx, du, flags, workspace,
                              workspace_bytes, chunk0, chunk, st, rows);
  return fail(PTC_ERR_ARG, "dtype must be PTC_F32 or PTC_F64");
}

int ptc_lqr_solve(int dtype, int batch, int horizon, int nx, int nu, const void* P, const void* R,
                  const void* M, const void* d, const void* Fx, const void* Fu, const void* PT,
                  const double* alpha, void* S, void* s, void* Gamma, void* gamma, void* dx,
                  void* du, int* flags, void* workspace, int64_t workspace_bytes, int chunk0,
                  int chunk, void* stream) {
  if (batch < 1 || horizon < 1 || nx < 1 || nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == PTC_F64)
    return lqr_solve_t<double>(batch, horizon, nx, nu, P, R, M, d, Fx, Fu, PT, alpha, S, s, Gamma,
                               gamma, dx, du, flags, workspace, workspace_bytes, chunk0, chunk, st);
  if (dtype == PTC_F32)
    return lqr_solve_t<float>(batch, horizon, nx, nu, P, R, M, d, Fx, Fu, PT, alpha, S, s, Gamma,
                              gamma, dx, du, flags, workspace, workspace_bytes, chunk0, chunk, st);
  return fail(PTC_ERR_ARG, "dtype must be PTC_F32 or PTC_F64");
}

}  // extern "C"

// ---------------------------------------------------------------------------
// solver object
// ---------------------------------------------------------------------------

struct ptc_solver {
  virtual ~ptc_solver() = default;
  ptc_problem_desc desc;
  virtual int load(const void* X, const void* U, const void* z, const void* v, int on_dev,
                   cudaStream_t s) = 0;
  virtual int check(int32_t* bad, cudaStream_t s) = 0;
  virtual int iterate(int n, cudaStream_t s) = 0;
  virtual int running(int32_t* n, cudaStream_t s) = 0;
  virtual int running_async(int32_t* n, cudaStream_t s) = 0;
  virtual int loop(int group, int cap, int32_t* launched, cudaStream_t s) = 0;
  virtual int expand(cudaStream_t s) = 0;
  virtual int lqr(const double* alpha_host, cudaStream_t s) = 0;
  virtual int rollout(cudaStream_t s) = 0;
  virtual int total_cost(cudaStream_t s) = 0;
  virtual int info(const char* name, int64_t* numel, int32_t* es) = 0;
  virtual int read(const char* name, void* dst, int64_t bytes, int on_dev, cudaStream_t s) = 0;
  virtual int write(const char* name, const void* src, int64_t bytes, int on_dev,
                    cudaStream_t s) = 0;
  virtual int block_phase(int phase, const void* in, void* out, const void* aux, int rank,
                          int world, cudaStream_t s) = 0;
};

namespace ptc {

// device-resident solve loop (Solver::loop): the launch counter and the
// WHILE node's condition
__global__ void k_loop_init(int* count) { *count = 0; }

__global__ void k_loop_cond(cudaGraphConditionalHandle h, const int* n_running, int* count,
                            int group, int cap) {
  const int c = *count + group;
  *count = c;
  cudaGraphSetConditional(h, (*n_running > 0 && c < cap) ? 1u : 0u);
}

// component-major affine model (comps x T) -> stage-major rows [t][A | Bm | c]
template <typename R>
__global__ void k_model_stage_major(const R* A, const R* Bm, const R* c, R* st, int T, int nx,
                                    int nu) {
  __shared__ R tile[32][33];
  const int nA = nx * nx, nB = nx * nu, nc = nA + nB + nx;
  const int c0 = blockIdx.x * 32, t0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int k = c0 + i, t = t0 + threadIdx.x;
    R v = R(0);
    if (k < nc && t < T) {
      if (k < nA) v = A[(size_t)k * T + t];
      else if (k < nA + nB) v = Bm[(size_t)(k - nA) * T + t];
      else v = c[(size_t)(k - nA - nB) * T + t];
    }
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int t = t0 + i, k = c0 + threadIdx.x;
    if (k < nc && t < T) st[(size_t)t * nc + k] = tile[threadIdx.x][i];
  }
}

template <typename R>
__global__ void k_normalize_parity(NewtonArgs<R> a, int nx, int nu) {
  // make buffer 0 hold every problem's current trajectory
  const long long n = (long long)a.B * (a.T + 1);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = (int)(i % a.B);
  const int t = (int)(i / a.B);
  if (a.parity[b] == 0) return;
  for (int c = 0; c < nx; ++c) {
    size_t o = ((size_t)c * (a.T + 1) + t) * a.B + b;
    a.X[o] = a.X[a.xsz + o];
  }
  if (t < a.T)
    for (int c = 0; c < nu; ++c) {
      size_t o = ((size_t)c * a.T + t) * a.B + b;
      a.U[o] = a.U[a.usz + o];
    }
}

template <typename R>
__global__ void k_clear_parity(NewtonArgs<R> a) {
  const int b = unit_id();
  if (b < a.B) a.parity[b] = 0;
}

struct Buf {
  void* p;
  int64_t numel;
  int32_t es;
};

template <typename R>
struct Solver final : ptc_solver {
  NewtonArgs<R> na{};
  LqrArgs<R> la{};
  const NewtonOps* ops = nullptr;
  int nx = 0, nu = 0, W = 0;
  R *S = nullptr, *s_ = nullptr;
  int* bad_t = nullptr;
  ProblemParams hp{};
  std::map<std::string, Buf> bufs;

  static void build_params(const ptc_problem_desc& d, ProblemParams& p) {
    std::memset(&p, 0, sizeof(p));
    p.dyn_kind = d.model;
    for (int i = 0; i < 8; ++i) p.dyn[i] = d.dyn_params[i];
    const int nx = d.nx, nu = d.nu;
    for (int i = 0; i < nx * nx; ++i) {
      p.Q[i] = d.Q ? d.Q[i] : 0.0;
      p.Qf[i] = d.Qf ? d.Qf[i] : 0.0;
    }
    for (int i = 0; i < nu * nu; ++i) p.Rc[i] = d.R ? d.R[i] : 0.0;
    for (int i = 0; i < nx; ++i) p.goal[i] = d.goal ? d.goal[i] : 0.0;
    int W = 0;
    auto add = [&](int var, int idx, double sign, double bound) {
      p.row_var[W] = var;
      p.row_idx[W] = idx;
      p.row_sign[W] = sign;
      p.row_bound[W] = bound;
      const int v = var == 0 ? idx : kMaxNX + idx;
      if (sign > 0) {
        p.box_up |= 1u << v;
        p.box_ub[v] = bound;
      } else {
        p.box_lo |= 1u << v;
        p.box_lb[v] = bound;
      }
      ++W;
    };
    // stacking order of BoxConstraint (problem.py:254-260): state upper,
    // state lower, control upper, control lower; infinite bounds dropped
    for (int i = 0; i < nx; ++i)
      if (d.state_upper && std::isfinite(d.state_upper[i])) add(0, i, 1.0, d.state_upper[i]);
    for (int i = 0; i < nx; ++i)
      if (d.state_lower && std::isfinite(d.state_lower[i])) add(0, i, -1.0, d.state_lower[i]);
    p.Ws = W;
    for (int i = 0; i < nu; ++i)
      if (d.control_upper && std::isfinite(d.control_upper[i])) add(1, i, 1.0, d.control_upper[i]);
    for (int i = 0; i < nu; ++i)
      if (d.control_lower && std::isfinite(d.control_lower[i])) add(1, i, -1.0, d.control_lower[i]);
    p.W = W;
    p.lin_T = std::max(1, d.lin_rows);
    p.lin_B = std::max(1, d.lin_batch);
    p.user_data = static_cast<const double*>(d.user_data);
    for (int i = 0; i < 8; ++i) p.cost_prm[i] = d.cost_params[i];
    p.cost_data = static_cast<const double*>(d.cost_data);
    for (int i = 0; i < 8; ++i) p.con_prm[i] = d.con_params[i];
    p.con_data = static_cast<const double*>(d.con_data);
    if (d.con_rows_state + d.con_rows_control > 0) {   // user constraint rows
      p.Ws = d.con_rows_state;
      p.W = d.con_rows_state + d.con_rows_control;
    }
  }

  static size_t layout(const ptc_problem_desc& d, Carver& c, Solver* self) {
    const size_t B = d.batch, T = d.horizon, nx = d.nx, nu = d.nu;
    ProblemParams pp;
    build_params(d, pp);
    const size_t W = pp.W;
    NewtonArgs<R> a{};
    LqrArgs<R> l{};
    a.B = l.B = (int)B;
    a.T = l.T = (int)T;
    a.plan = l.plan = auto_plan((int)B, (int)T, d.chunk0, d.chunk, (int)nx);
    const size_t P0 = a.plan.units0();
    ProblemParams* dpp = c.template take<ProblemParams>(1);
    R *linA = nullptr, *linB = nullptr, *linc = nullptr, *linst = nullptr;
    if (d.model == PTC_DYN_LINEAR) {
      const size_t lt = pp.lin_T, lb = pp.lin_B;
      linA = c.template take<R>(nx * nx * lt * lb);
      linB = c.template take<R>(nx * nu * lt * lb);
      linc = c.template take<R>(nx * lt * lb);
      if (lt > 1 && lb == 1 && nx >= 8) linst = c.template take<R>((nx * nx + nx * nu + nx) * lt);
    }
    a.xsz = nx * (T + 1) * B;
    a.usz = nu * T * B;
    a.X = c.template take<R>(2 * a.xsz);
    a.U = c.template take<R>(2 * a.usz);
    auto ib = [&]() { return c.template take<int>(B); };
    auto db = [&]() { return c.template take<double>(B); };
    a.status = ib(); a.phase = ib(); a.parity = ib(); a.flags = ib(); a.iters = ib();
    a.term = ib(); a.round = ib(); a.hist_len = ib(); a.bad_index = ib();
    a.n_running = c.template take<int>(1);
    int* bad_t = ib();
    a.rstate = ib();
    a.rres = c.template take<double>(P0 * B);
    // candidate rollout: log-depth Newton sweeps for tree plans with long
    // horizons (rollout 0 = auto), the sequential recurrence otherwise
    // (affine dynamics: the log-depth rollout is exact in one scan -- the
    // wide affine-scan kernels for nx >= 8, one checked sweep otherwise --
    // and beats the sequential recurrence at any horizon with a tree plan)
    const bool affine = d.model == PTC_DYN_LINEAR;
    const bool par = a.plan.L >= 1 &&
                     (d.rollout == 2 || (d.rollout == 0 && (T >= 1024 || affine)));
    // Newton on the recurrence converges quadratically from the LQR's
    // prediction when it converges at all (non-chaotic stretches): 4 sweeps,
    // then the sequential recurrence -- a larger budget only adds early-exit
    // launches to every iteration of the problems that never converge
    a.pr_iters = par ? 4 : 0;
    a.xr = par ? c.template take<R>(a.xsz) : nullptr;
    // cached sin / cos of each trajectory buffer's pole angle (CartPole's
    // kAux values, single-sweep Newton kernels, fp64)
    const bool aux = !d.block_mode && d.model == PTC_DYN_CARTPOLE && sizeof(R) == 8;
    a.auxsz = aux ? 2 * T * B : 0;
    a.aux = aux ? c.template take<R>(2 * a.auxsz) : nullptr;
    a.aux_ok = aux ? ib() : nullptr;
    a.alpha = db(); a.nu = db(); a.cur_cost = db(); a.cand_cost = db(); a.mu = db();
    a.bad_value = db();
    a.opt.hist_cap = std::max(0, d.hist_cap);
    a.opt.round_cap = std::max(1, d.round_cap);
    a.hist = c.template take<double>((size_t)a.opt.hist_cap * 5 * B + 1);
    const size_t rc = a.opt.round_cap;
    a.round_mu = c.template take<double>(rc * B);
    a.round_cost = c.template take<double>(rc * B);
    a.round_rp = c.template take<double>(rc * B);
    a.round_rd = c.template take<double>(rc * B);
    a.round_iters = c.template take<int>(rc * B);
    a.round_term = c.template take<int>(rc * B);
    a.round_U = (d.method == PTC_METHOD_BARRIER && d.keep_round_controls)
                    ? c.template take<R>(rc * nu * T * B) : nullptr;
    const bool admm = d.method == PTC_METHOD_ADMM || d.aug == PTC_AUG_ADMM;
    a.z = admm ? c.template take<R>(std::max<size_t>(W, 1) * T * B) : nullptr;
    a.v = admm ? c.template take<R>(std::max<size_t>(W, 1) * T * B) : nullptr;
    a.lam = c.template take<R>(nx * (T + 1) * B);
    a.P = c.template take<R>(nx * nx * T * B);
    a.Rm = c.template take<R>(nu * nu * T * B);
    a.M = c.template take<R>(nx * nu * T * B);
    a.d = c.template take<R>(nu * T * B);
    a.Fx = c.template take<R>(nx * nx * T * B);
    a.Fu = c.template take<R>(nx * nu * T * B);
    a.PT = c.template take<R>(nx * nx * B);
    for (int k = 0; k <= kMaxLevels; ++k) a.cagg[k] = a.ccar[k] = nullptr;
    for (int k = 1; k <= a.plan.L; ++k) {
      a.cagg[k] = c.template take<R>((size_t)a.plan.n[k] * B * (nx * nx + nx));
      a.ccar[k] = c.template take<R>((size_t)a.plan.n[k] * B * nx);
    }
    a.cpart[0] = c.template take<double>(3 * P0 * B);
    a.cpart[1] = c.template take<double>(3 * P0 * B);
    a.apart = c.template take<double>(2 * P0 * B);
    // LQR outputs + tree
    const bool keep_S = B * (T + 1) * (nx * nx + nx) <= (size_t)64 << 20;
    R* S = keep_S ? c.template take<R>(nx * nx * (T + 1) * B) : nullptr;
    R* s = keep_S ? c.template take<R>(nx * (T + 1) * B) : nullptr;
    l.Gam = c.template take<R>(nu * nx * T * B);
    l.gam = c.template take<R>(nu * T * B);
    l.dX = c.template take<R>(nx * (T + 1) * B);
    l.dU = c.template take<R>(nu * T * B);
    a.blk = d.block_mode ? 1 : 0;
    a.uterm = 0;
    a.blk_last = d.block_last ? 1 : 0;
    a.t_base = d.block_mode ? d.t_base : 0;
    a.lam_in = a.x_in = nullptr;
    a.x0g = nullptr;
    if (d.block_mode) {
      l.block_mode = 1;
      l.t_base = d.t_base;
      l.no_terminal = d.block_last ? 0 : 1;
      a.lam_in = c.template take<R>(nx * B);
      a.x_in = c.template take<R>(nx * B);
    }
    carve_lqr_tree(c, l, (int)nx, (int)nu);
    a.red = l.red;
    if (self) {
      self->hp = pp;
      self->W = (int)W;
      self->S = S;
      self->s_ = s;
      self->bad_t = bad_t;
      a.pp = dpp;
      a.aug_kind = d.method == PTC_METHOD_BARRIER ? AUG_BARRIER
                   : d.method == PTC_METHOD_ADMM  ? AUG_ADMM
                                                  : d.aug;
      a.opt.method = d.method;
      a.opt.alpha0 = d.alpha0;
      a.opt.nu0 = d.nu0;
      a.opt.inner_tol = d.inner_tol;
      a.opt.max_iters = d.max_iters;
      a.opt.mu0 = d.method == PTC_METHOD_BARRIER ? d.mu0 : d.aug_mu;
      a.opt.zeta = d.zeta;
      a.opt.mu_tol = d.mu_tol;
      a.opt.rho = d.rho;
      a.opt.residual_tol = d.residual_tol;
      a.opt.max_outer = d.max_outer;
      a.opt.keep_round_controls = d.keep_round_controls;
      self->hp.lin_A = linA;
      self->hp.lin_Bm = linB;
      self->hp.lin_c = linc;
      self->hp.lin_st = linst;
      // LQR args view the solver's expansion
      l.P = a.P; l.Rm = a.Rm; l.M = a.M; l.d = a.d; l.Fx = a.Fx; l.Fu = a.Fu; l.PT = a.PT;
      l.alpha = a.alpha;
      l.status = a.status;
      l.flags = a.flags;
      l.S = nullptr;
      l.s = nullptr;
      self->na = a;
      self->la = l;
      auto reg = [&](const char* n, void* p, int64_t numel, int32_t es) {
        self->bufs[n] = Buf{p, numel, es};
      };
      const int rs = sizeof(R);
      reg("states", a.X, a.xsz, rs);
      reg("controls", a.U, a.usz, rs);
      reg("lam", a.lam, nx * (T + 1) * B, rs);
      reg("P", a.P, nx * nx * T * B, rs);
      reg("R", a.Rm, nu * nu * T * B, rs);
      reg("M", a.M, nx * nu * T * B, rs);
      reg("d", a.d, nu * T * B, rs);
      reg("Fx", a.Fx, nx * nx * T * B, rs);
      reg("Fu", a.Fu, nx * nu * T * B, rs);
      reg("PT", a.PT, nx * nx * B, rs);
      if (S) {
        reg("S", S, nx * nx * (T + 1) * B, rs);
        reg("s", s, nx * (T + 1) * B, rs);
      }
      reg("Gamma", l.Gam, nu * nx * T * B, rs);
      reg("gamma", l.gam, nu * T * B, rs);
      reg("dx", l.dX, nx * (T + 1) * B, rs);
      reg("du", l.dU, nu * T * B, rs);
      if (a.z) {
        reg("z", a.z, W * T * B, rs);
        reg("v", a.v, W * T * B, rs);
      }
      reg("status", a.status, B, 4);
      reg("phase", a.phase, B, 4);
      reg("iters", a.iters, B, 4);
      reg("term", a.term, B, 4);
      reg("round", a.round, B, 4);
      reg("hist_len", a.hist_len, B, 4);
      reg("bad_index", a.bad_index, B, 4);
      reg("flags", a.flags, B, 4);
      reg("rollout_state", a.rstate, B, 4);
      reg("parity", a.parity, B, 4);
      reg("hist", a.hist, (int64_t)a.opt.hist_cap * 5 * B, 8);
      reg("cur_cost", a.cur_cost, B, 8);
      reg("cand_cost", a.cand_cost, B, 8);
      reg("alpha", a.alpha, B, 8);
      reg("nu", a.nu, B, 8);
      reg("mu", a.mu, B, 8);
      reg("bad_value", a.bad_value, B, 8);
      reg("round_mu", a.round_mu, rc * B, 8);
      reg("round_cost", a.round_cost, rc * B, 8);
      reg("round_rp", a.round_rp, rc * B, 8);
      reg("round_rd", a.round_rd, rc * B, 8);
      reg("round_iters", a.round_iters, rc * B, 4);
      reg("round_term", a.round_term, rc * B, 4);
      if (a.round_U) reg("round_controls", a.round_U, rc * nu * T * B, rs);
    }
    return c.off + 256;
  }

  int init(const ptc_problem_desc& d, void* ws, int64_t bytes) {
    desc = d;
    nx = d.nx;
    nu = d.nu;
    ops = nullptr;
    auto it = newton_registry().find(NewtonKey(dtype_code<R>(), d.model, d.nx, d.nu));
    if (it == newton_registry().end())
      return fail(PTC_ERR_UNSUPPORTED, "solver kernels not instantiated for model " +
                                           std::to_string(d.model) + " nx=" + std::to_string(d.nx) +
                                           " nu=" + std::to_string(d.nu));
    if (!lqr_registry().count(LqrKey(dtype_code<R>(), d.nx, d.nu)))
      return fail(PTC_ERR_UNSUPPORTED, "LQR kernels not instantiated for nx=" +
                                           std::to_string(d.nx) + " nu=" + std::to_string(d.nu));
    ops = &it->second;
    if (d.block_mode && !ops->block)
      return fail(PTC_ERR_UNSUPPORTED, "time-block mode is implemented for affine models with "
                                       "nx >= 8 (the config-4 systems)");
    if (d.block_mode && auto_plan(d.batch, d.horizon, d.chunk0, d.chunk, d.nx).L < 1)
      return fail(PTC_ERR_ARG, "time-block mode needs a tree plan (chunk0 < horizon)");
    Carver c{(char*)ws};
    size_t need = layout(d, c, this);
    if ((int64_t)need > bytes) return fail(PTC_ERR_WORKSPACE, "solver workspace too small");
    na.uterm = ops->user_cost;
    if (d.model == PTC_DYN_LINEAR) {
      const size_t lt = hp.lin_T, lb = hp.lin_B;
      if (!d.lin_a || !d.lin_b) return fail(PTC_ERR_ARG, "linear model needs lin_a and lin_b");
      // host or device pointers (unified addressing decides the direction)
      PTC_CUDA(cudaMemcpy((void*)hp.lin_A, d.lin_a, sizeof(R) * nx * nx * lt * lb, cudaMemcpyDefault));
      PTC_CUDA(cudaMemcpy((void*)hp.lin_Bm, d.lin_b, sizeof(R) * nx * nu * lt * lb, cudaMemcpyDefault));
      if (d.lin_c)
        PTC_CUDA(cudaMemcpy((void*)hp.lin_c, d.lin_c, sizeof(R) * nx * lt * lb, cudaMemcpyDefault));
      else
        PTC_CUDA(cudaMemset((void*)hp.lin_c, 0, sizeof(R) * nx * lt * lb));
      if (hp.lin_st) {
        const int nc = nx * nx + nx * nu + nx;
        k_model_stage_major<R><<<dim3((nc + 31) / 32, (unsigned)((lt + 31) / 32)), dim3(32, 8)>>>(
            static_cast<const R*>(hp.lin_A), static_cast<const R*>(hp.lin_Bm),
            static_cast<const R*>(hp.lin_c), (R*)hp.lin_st, (int)lt, nx, nu);
        PTC_CUDA(cudaGetLastError());
        PTC_CUDA(cudaStreamSynchronize(0));
      }
    }
    PTC_CUDA(cudaMemcpy((void*)na.pp, &hp, sizeof(ProblemParams), cudaMemcpyHostToDevice));
    return PTC_OK;
  }

  int load(const void* X, const void* U, const void* z, const void* v, int on_dev,
           cudaStream_t s) override {
    auto kind = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    PTC_CUDA(cudaMemcpyAsync(na.X, X, sizeof(R) * na.xsz, kind, s));
    PTC_CUDA(cudaMemcpyAsync(na.U, U, sizeof(R) * na.usz, kind, s));
    PTC_CUDA(clear_aux(s));
    ops->init(&na, s);
    if (desc.method == PTC_METHOD_NEWTON && na.aug_kind == AUG_ADMM) {
      const size_t n = sizeof(R) * (size_t)std::max(W, 1) * na.T * na.B;
      if (z) PTC_CUDA(cudaMemcpyAsync(na.z, z, n, kind, s));
      else PTC_CUDA(cudaMemsetAsync(na.z, 0, n, s));
      if (v) PTC_CUDA(cudaMemcpyAsync(na.v, v, n, kind, s));
      else PTC_CUDA(cudaMemsetAsync(na.v, 0, n, s));
    }
    PTC_CUDA(cudaGetLastError());
    return PTC_OK;
  }

  int check(int32_t* bad, cudaStream_t s) override {
    std::vector<int> init(na.B, 0x7fffffff);
    PTC_CUDA(cudaMemcpyAsync(bad_t, init.data(), sizeof(int) * na.B, cudaMemcpyHostToDevice, s));
    ops->check(&na, bad_t, s);
    PTC_CUDA(cudaMemcpyAsync(bad, bad_t, sizeof(int) * na.B, cudaMemcpyDeviceToHost, s));
    PTC_CUDA(cudaStreamSynchronize(s));
    for (int b = 0; b < na.B; ++b)
      if (bad[b] == 0x7fffffff) bad[b] = -1;
    return PTC_OK;
  }

  // One Newton iteration is a fixed launch sequence over fixed buffers, so
  // it is captured once into a CUDA graph (on a private stream: the legacy
  // default stream cannot be captured) and replayed on the caller's stream.
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t iter_exec = nullptr;
  bool graph_off = false;

  void build_iteration_graph() {
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      ops->iterate(&na, &la, cap_stream);
      ok = cudaStreamEndCapture(cap_stream, &g) == cudaSuccess && g != nullptr;
    }
    if (ok) ok = cudaGraphInstantiate(&iter_exec, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) {
      iter_exec = nullptr;
      graph_off = true;
      (void)cudaGetLastError();
    }
  }

  // The whole solve as one device-resident loop: a CUDA graph whose
  // conditional WHILE node replays `group` iterations and then lets one
  // thread decide, from the control kernel's running count, whether to go
  // round again -- no host round trip between iterations, so a host stall
  // cannot drain the stream (the host-polled loop's failure mode).
  cudaGraphExec_t loop_exec = nullptr;
  int loop_group = 0, loop_cap = 0;
  int* loop_count = nullptr;

  int build_loop_graph(int group, int cap) {
    if (loop_exec) cudaGraphExecDestroy(loop_exec);
    loop_exec = nullptr;
    if (!loop_count) PTC_CUDA(cudaMalloc(&loop_count, sizeof(int)));
    if (!cap_stream) PTC_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    PTC_CUDA(cudaGraphCreate(&g, 0));
    cudaError_t e = add_loop_nodes(g, group, cap);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&loop_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      loop_exec = nullptr;
      (void)cudaGetLastError();
      return fail(PTC_ERR_CUDA, std::string("device loop graph: ") + cudaGetErrorString(e));
    }
    loop_group = group;
    loop_cap = cap;
    return PTC_OK;
  }

  cudaError_t add_loop_nodes(cudaGraph_t g, int group, int cap) {
    cudaGraphNode_t init;
    cudaKernelNodeParams kp = {};
    void* init_args[] = {&loop_count};
    kp.func = reinterpret_cast<void*>(ptc::k_loop_init);
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = init_args;
    cudaError_t e = cudaGraphAddKernelNode(&init, g, nullptr, 0, &kp);
    if (e != cudaSuccess) return e;
    cudaGraphConditionalHandle h;
    e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    if (e != cudaSuccess) return e;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t loop;
    e = cudaGraphAddNode(&loop, g, &init, 1, &cp);
    if (e != cudaSuccess) return e;
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(cap_stream, body, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return e;
    for (int i = 0; i < group; ++i) ops->iterate(&na, &la, cap_stream);
    ptc::k_loop_cond<<<1, 1, 0, cap_stream>>>(h, na.n_running, loop_count, group, cap);
    cudaGraph_t out = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(cap_stream, &out);
    return e2 != cudaSuccess ? e2 : cudaGetLastError();
  }

  int loop(int group, int cap, int32_t* launched, cudaStream_t s) override {
    if (na.blk) return fail(PTC_ERR_ARG, "block_mode solvers iterate through ptc_solver_block_phase");
    if (group < 1 || cap < 1) return fail(PTC_ERR_ARG, "group and max_launch must be >= 1");
    if (!loop_exec || group != loop_group || cap != loop_cap) {
      int rc = build_loop_graph(group, cap);
      if (rc) return rc;
    }
    PTC_CUDA(cudaGraphLaunch(loop_exec, s));
    if (launched)
      PTC_CUDA(cudaMemcpyAsync(launched, loop_count, sizeof(int), cudaMemcpyDeviceToHost, s));
    return PTC_OK;
  }

  ~Solver() override {
    if (loop_exec) cudaGraphExecDestroy(loop_exec);
    if (loop_count) cudaFree(loop_count);
    if (iter_exec) cudaGraphExecDestroy(iter_exec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
  }

  // states written outside the iteration: no trajectory buffer's cached
  // auxiliary values belong to it any more
  cudaError_t clear_aux(cudaStream_t s) {
    return na.aux_ok ? cudaMemsetAsync(na.aux_ok, 0, sizeof(int) * na.B, s) : cudaSuccess;
  }

  int iterate(int n, cudaStream_t s) override {
    if (na.blk) return fail(PTC_ERR_ARG, "block_mode solvers iterate through ptc_solver_block_phase");
    if (n > 0 && !iter_exec && !graph_off && !getenv("PTC_NO_GRAPH")) build_iteration_graph();
    for (int i = 0; i < n; ++i) {
      if (iter_exec) PTC_CUDA(cudaGraphLaunch(iter_exec, s));
      else ops->iterate(&na, &la, s);
    }
    PTC_CUDA(cudaGetLastError());
    return PTC_OK;
  }

  int block_phase(int phase, const void* in, void* out, const void* aux, int rank, int world,
                  cudaStream_t s) override {
    if (!na.blk) return fail(PTC_ERR_ARG, "ptc_solver_block_phase needs a block_mode solver");
    if (phase < 0 || phase > 9) return fail(PTC_ERR_ARG, "block phase must be 0..9");
    if (world < 1 || rank < 0 || rank >= world) return fail(PTC_ERR_ARG, "bad rank / world");
    if (na.blk_last != (rank == world - 1))
      return fail(PTC_ERR_ARG, "block_last must be set exactly on rank world-1");
    const bool needs_in = phase == 1 || phase == 2 || phase == 3 || phase == 4 || phase == 5 ||
                          phase == 6 || phase == 7 || phase == 9;
    const bool needs_out = phase <= 6 || phase == 8;
    if (needs_in && !in) return fail(PTC_ERR_ARG, "this block phase needs its input buffer");
    if (needs_out && !out) return fail(PTC_ERR_ARG, "this block phase needs its output buffer");
    if ((phase == 5 || phase == 9) && !aux) return fail(PTC_ERR_ARG, "phases 5 and 9 need x0 (aux)");
    na.x0g = static_cast<const R*>(aux);
    ops->block(&na, &la, phase, in, out, rank, world, s);
    PTC_CUDA(cudaGetLastError());
    return PTC_OK;
  }

  int running(int32_t* n, cudaStream_t s) override {
    PTC_CUDA(cudaMemcpyAsync(n, na.n_running, sizeof(int), cudaMemcpyDeviceToHost, s));
    PTC_CUDA(cudaStreamSynchronize(s));
    return PTC_OK;
  }
  int running_async(int32_t* n, cudaStream_t s) override {
    PTC_CUDA(cudaMemcpyAsync(n, na.n_running, sizeof(int), cudaMemcpyDeviceToHost, s));
    return PTC_OK;
  }

  int expand(cudaStream_t s) override {
    ops->expand(&na, s);
    PTC_CUDA(cudaGetLastError());
    return PTC_OK;
  }

  int lqr(const double* alpha_host, cudaStream_t s) override {
    if (alpha_host)
      PTC_CUDA(cudaMemcpyAsync(na.alpha, alpha_host, sizeof(double) * na.B, cudaMemcpyHostToDevice, s));
    PTC_CUDA(cudaMemsetAsync(na.flags, 0, sizeof(int) * na.B, s));
    LqrArgs<R> l = la;
    l.status = nullptr;
    l.S = S;
    l.s = s_;
    ops->lqr(&l, s);
    PTC_CUDA(cudaGetLastError());
    return PTC_OK;
  }

  int rollout(cudaStream_t s) override {
    if (na.blk) return fail(PTC_ERR_ARG, "block_mode solvers roll out through block phases 8 / 9");
    PTC_CUDA(cudaMemsetAsync(na.bad_index, 0xff, sizeof(int) * na.B, s));
    PTC_CUDA(clear_aux(s));
    ops->rollout(&na, s);
    PTC_CUDA(cudaGetLastError());
    return PTC_OK;
  }

  int total_cost(cudaStream_t s) override {
    ops->cost(&na, s);
    PTC_CUDA(cudaGetLastError());
    return PTC_OK;
  }

  int info(const char* name, int64_t* numel, int32_t* es) override {
    auto it = bufs.find(name);
    if (it == bufs.end()) return fail(PTC_ERR_ARG, std::string("unknown buffer ") + name);
    if (numel) *numel = it->second.numel;
    if (es) *es = it->second.es;
    return PTC_OK;
  }

  int read(const char* name, void* dst, int64_t bytes, int on_dev, cudaStream_t s) override {
    auto it = bufs.find(name);
    if (it == bufs.end()) return fail(PTC_ERR_ARG, std::string("unknown buffer ") + name);
    const Buf& bf = it->second;
    if (bytes < bf.numel * bf.es) return fail(PTC_ERR_ARG, "destination too small");
    if (!strcmp(name, "states") || !strcmp(name, "controls")) {
      const long long n = (long long)na.B * (na.T + 1);
      k_normalize_parity<R><<<grid_for(n), kBlock, 0, s>>>(na, nx, nu);
      k_clear_parity<R><<<grid_for(na.B), kBlock, 0, s>>>(na);
      PTC_CUDA(clear_aux(s));
    }
    PTC_CUDA(cudaMemcpyAsync(dst, bf.p, bf.numel * bf.es,
                             on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    if (!on_dev) PTC_CUDA(cudaStreamSynchronize(s));
    PTC_CUDA(cudaGetLastError());
    return PTC_OK;
  }
  // per-problem loop state a caller may set between load and iterate
  // (restart from a recorded iteration: alpha, nu, mu)
  int write(const char* name, const void* src, int64_t bytes, int on_dev,
            cudaStream_t s) override {
    if (strcmp(name, "alpha") && strcmp(name, "nu") && strcmp(name, "mu"))
      return fail(PTC_ERR_ARG, std::string("buffer not writable: ") + name);
    const Buf& bf = bufs.at(name);
    if (bytes != bf.numel * bf.es) return fail(PTC_ERR_ARG, "size mismatch");
    PTC_CUDA(cudaMemcpyAsync(bf.p, src, bytes,
                             on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    if (!on_dev) PTC_CUDA(cudaStreamSynchronize(s));
    PTC_CUDA(cudaGetLastError());
    return PTC_OK;
  }
};

}  // namespace ptc

extern "C" {

static int validate(const ptc_problem_desc* d) {
  if (!d) return fail(PTC_ERR_ARG, "desc is NULL");
  if (d->dtype != PTC_F32 && d->dtype != PTC_F64) return fail(PTC_ERR_ARG, "bad dtype");
  if (d->batch < 1 || d->horizon < 1 || d->nx < 1 || d->nu < 1) return fail(PTC_ERR_ARG, "bad dims");
  if (d->nx > kMaxNX || d->nu > kMaxNU) return fail(PTC_ERR_ARG, "nx <= 12 and nu <= 6 required");
  if (d->method < 0 || d->method > 2) return fail(PTC_ERR_ARG, "bad method");
  if (d->block_mode != 0 && d->block_mode != 1) return fail(PTC_ERR_ARG, "block_mode must be 0 or 1");
  if (d->block_mode && d->t_base < 0) return fail(PTC_ERR_ARG, "t_base must be >= 0");
  if (d->model == PTC_DYN_LINEAR) {
    if (d->lin_rows != 1 && d->lin_rows != d->horizon) return fail(PTC_ERR_ARG, "lin_rows must be 1 or horizon");
    if (d->lin_batch != 1 && d->lin_batch != d->batch) return fail(PTC_ERR_ARG, "lin_batch must be 1 or batch");
  }
  return PTC_OK;
}

int64_t ptc_solver_workspace_bytes(const ptc_problem_desc* d) {
  int rc = validate(d);
  if (rc) return rc;
  Carver c{nullptr};
  if (d->dtype == PTC_F64) return (int64_t)Solver<double>::layout(*d, c, nullptr);
  return (int64_t)Solver<float>::layout(*d, c, nullptr);
}

int ptc_solver_create(const ptc_problem_desc* d, void* ws, int64_t bytes, ptc_solver** out) {
  int rc = validate(d);
  if (rc) return rc;
  if (!out) return fail(PTC_ERR_ARG, "out is NULL");
  std::unique_ptr<ptc_solver> s;
  if (d->dtype == PTC_F64) {
    auto* p = new Solver<double>();
    s.reset(p);
    rc = p->init(*d, ws, bytes);
  } else {
    auto* p = new Solver<float>();
    s.reset(p);
    rc = p->init(*d, ws, bytes);
  }
  if (rc) return rc;
  *out = s.release();
  return PTC_OK;
}

int ptc_solver_destroy(ptc_solver* s) {
  delete s;
  return PTC_OK;
}

#define PTC_S(s) if (!(s)) return fail(PTC_ERR_ARG, "solver is NULL")

int ptc_solver_load(ptc_solver* s, const void* X, const void* U, const void* z, const void* v,
                    int on_device, void* stream) {
  PTC_S(s);
  return s->load(X, U, z, v, on_device, (cudaStream_t)stream);
}
int ptc_solver_check_consistency(ptc_solver* s, int32_t* bad, void* stream) {
  PTC_S(s);
  return s->check(bad, (cudaStream_t)stream);
}
int ptc_solver_iterate(ptc_solver* s, int n, void* stream) {
  PTC_S(s);
  return s->iterate(n, (cudaStream_t)stream);
}
int ptc_solver_block_phase(ptc_solver* s, int phase, const void* in, void* out, const void* aux,
                           int rank, int world, void* stream) {
  PTC_S(s);
  return s->block_phase(phase, in, out, aux, rank, world, (cudaStream_t)stream);
}
int ptc_solver_running(ptc_solver* s, int32_t* n, void* stream) {
  PTC_S(s);
  return s->running(n, (cudaStream_t)stream);
}

int ptc_solver_running_async(ptc_solver* s, int32_t* n, void* stream) {
  PTC_S(s);
  if (!n) return fail(PTC_ERR_ARG, "n is required");
  return s->running_async(n, (cudaStream_t)stream);
}
int ptc_solver_loop(ptc_solver* s, int group, int max_launch, int32_t* launched, void* stream) {
  PTC_S(s);
  return s->loop(group, max_launch, launched, (cudaStream_t)stream);
}
int ptc_solver_expand(ptc_solver* s, void* stream) {
  PTC_S(s);
  return s->expand((cudaStream_t)stream);
}
int ptc_solver_lqr(ptc_solver* s, const double* alpha_host, void* stream) {
  PTC_S(s);
  return s->lqr(alpha_host, (cudaStream_t)stream);
}
int ptc_solver_rollout(ptc_solver* s, void* stream) {
  PTC_S(s);
  return s->rollout((cudaStream_t)stream);
}
int ptc_solver_total_cost(ptc_solver* s, void* stream) {
  PTC_S(s);
  return s->total_cost((cudaStream_t)stream);
}
int ptc_model_load(const char* path, int* model_id, int* nx, int* nu) {
  static std::mutex mu;
  static std::map<std::string, int> loaded;
  static int next_id = PTC_DYN_USER_BASE;
  if (!path || !model_id || !nx || !nu) return fail(PTC_ERR_ARG, "missing argument");
  std::lock_guard<std::mutex> lock(mu);
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) return fail(PTC_ERR_ARG, std::string("dlopen failed: ") + dlerror());
  using OpsFn = int (*)(int, int*, int*, NewtonOps*);
  auto fn = reinterpret_cast<OpsFn>(dlsym(h, "ptc_user_model_ops"));
  if (!fn) return fail(PTC_ERR_ARG, std::string(path) + " exports no ptc_user_model_ops");
  auto it = loaded.find(path);
  const int id = it != loaded.end() ? it->second : next_id++;
  int mx = 0, mu_ = 0;
  for (int dt : {PTC_F64, PTC_F32}) {
    NewtonOps ops{};
    if (fn(dt, &mx, &mu_, &ops) == 0) newton_registry()[NewtonKey(dt, id, mx, mu_)] = ops;
  }
  if (mx < 1) return fail(PTC_ERR_ARG, std::string(path) + " holds no kernel set");
  loaded[path] = id;
  *model_id = id;
  *nx = mx;
  *nu = mu_;
  return PTC_OK;
}

int ptc_solver_write(ptc_solver* s, const char* name, const void* src, int64_t bytes, int on_dev,
                     void* stream) {
  PTC_S(s);
  if (!name || !src) return fail(PTC_ERR_ARG, "missing argument");
  return s->write(name, src, bytes, on_dev, (cudaStream_t)stream);
}
int ptc_solver_buffer_info(ptc_solver* s, const char* name, int64_t* numel, int32_t* es) {
  PTC_S(s);
  return s->info(name, numel, es);
}
int ptc_solver_read(ptc_solver* s, const char* name, void* dst, int64_t bytes, int on_dev,
                    void* stream) {
  PTC_S(s);
  return s->read(name, dst, bytes, on_dev, (cudaStream_t)stream);
}

}  // extern "C"
