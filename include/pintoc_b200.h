/*
 * pintoc_b200 -- C ABI of the B200-native parallel-in-time Newton solver.
 *
 * Drop-in boundary for the hot path of the reference package `pintoc`
 * (arxiv 2409.20027 artifact, /root/reference/pkg/src/pintoc).  Every entry
 * point below replaces one reference function; the file:line it replaces is
 * given beside it.  The reference is pure Python, so the binding a
 * maintainer would add is a ctypes stub; the Python
 * package `paper_2409_20027_b200` is exactly that binding.
 *
 * Conventions
 *   - Plain pointers and sizes only.  `void* stream` is a cudaStream_t
 *     (NULL = legacy default stream).  Return value 0 = success, < 0 = error
 *     (message via ptc_last_error()).
 *   - dtype: PTC_F32 or PTC_F64; every array argument is in that dtype
 *     unless typed explicitly.
 *   - HBM layout "SoA, batch-minor": a per-stage field with C scalar
 *     components over `rows` stages of `batch` problems is stored as
 *         field[(c * rows + t) * batch + b],
 *     matrices row-major inside c (c = i * ncols + j).  For batch = 1 this is
 *     one contiguous time series per matrix entry.
 *   - Workspaces are caller-allocated device memory (the Python binding
 *     allocates them as torch tensors).
 */
#ifndef PINTOC_B200_H
#define PINTOC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PTC_F32 0
#define PTC_F64 1

#define PTC_OK 0
#define PTC_ERR_ARG (-1)
#define PTC_ERR_UNSUPPORTED (-2)
#define PTC_ERR_CUDA (-3)
#define PTC_ERR_WORKSPACE (-4)

/* dynamics models (reference systems.py) */
#define PTC_DYN_PENDULUM 0   /* PendulumDynamics, systems.py:172-231   */
#define PTC_DYN_CARTPOLE 1   /* CartPoleDynamics, systems.py:341-437   */
#define PTC_DYN_LINEAR 2     /* LinearDynamics, systems.py:32-77 (+ time-varying) */

/* augmentation of a plain Newton solve (reference problem.py:343-433, outer.py) */
#define PTC_AUG_ZERO 0
#define PTC_AUG_BARRIER 1
#define PTC_AUG_ADMM 2

/* solve method */
#define PTC_METHOD_NEWTON 0   /* newton.py:129  newton_solve   */
#define PTC_METHOD_BARRIER 1  /* outer.py:221   barrier_solve  */
#define PTC_METHOD_ADMM 2     /* outer.py:392   admm_solve     */

/* per-problem status codes (int32, read back with ptc_solver_read "status") */
#define PTC_ST_RUNNING 0
#define PTC_ST_DONE 1
#define PTC_ST_ERR_STALLED (-1)    /* SolverStalledError (newton.py:168-171) */
#define PTC_ST_ERR_INFEASIBLE (-2) /* InfeasibleError from total_cost          */

/* Newton termination codes ("round_term"); names as newton.py:41-44 */
#define PTC_TERM_NONE 0
#define PTC_TERM_COST 1       /* "converged_cost" */
#define PTC_TERM_STEP 2       /* "converged_step" */
#define PTC_TERM_MAX_ITERS 3  /* "max_iters"      */
#define PTC_TERM_STALLED 4    /* "stalled"        */

const char* ptc_last_error(void);
int ptc_version(void);

/* 1 if kernels for (dtype, model, nx, nu) are compiled in; model = -1 asks
 * about the model-free LQR kernels only. */
int ptc_supported(int dtype, int model, int nx, int nu);

/* ------------------------------------------------------------------------
 * LQR subproblem solve = value_pass + propagation_pass
 *   replaces passes.py:291 value_pass  (Alg. 2: suffix scan over dual value
 *   elements, passes.py:244-288, gains passes.py:316-323) and
 *   passes.py:338 propagation_pass (Alg. 3: prefix scan of closed-loop
 *   affine maps).
 * Inputs (device, SoA batch-minor, `horizon` rows unless noted):
 *   P (nx*nx), R (nu*nu, unregularised), M (nx*nu), d (nu), Fx (nx*nx),
 *   Fu (nx*nu), PT (nx*nx, 1 row), alpha (float64[batch], R_reg = R + alpha I).
 * Outputs (device): S (nx*nx, horizon+1 rows) and s (nx, horizon+1) may be
 *   NULL; Gamma (nu*nx), gamma (nu), dx (nx, horizon+1), du (nu).
 *   flags (int32[batch], must be zeroed by the caller): bit 1 R+alpha I not
 *   positive definite, bit 2 some Q_t not positive definite (both
 *   DefinitenessError), bit 4 singular I + C Y (ConditioningError).
 * chunk0 / chunk: scan-tree plan (stages per level-0 thread, items per
 *   thread above level 0); 0 = automatic.  chunk0 >= horizon gives the
 *   sequential (one thread per problem) schedule.
 * ---------------------------------------------------------------------- */
int64_t ptc_lqr_workspace_bytes(int dtype, int batch, int horizon, int nx, int nu,
                                int chunk0, int chunk);
int ptc_lqr_solve(int dtype, int batch, int horizon, int nx, int nu,
                  const void* P, const void* R, const void* M, const void* d,
                  const void* Fx, const void* Fu, const void* PT, const double* alpha,
                  void* S, void* s, void* Gamma, void* gamma, void* dx, void* du,
                  int* flags, void* workspace, int64_t workspace_bytes,
                  int chunk0, int chunk, void* stream);
/* The same solve for one long problem (batch 1, nx >= 8, horizon >= 1024)
 * whose expansion is given as stage rows rows[t * SC + c], row =
 * [P | R | M | d | Fx | Fu] (the reference StageExpansion's per-stage
 * arrays side by side): the layout the warp kernels read, no transpose. */
int ptc_lqr_solve_rows(int dtype, int horizon, int nx, int nu, const void* rows, const void* PT,
                       const double* alpha, void* S, void* s, void* Gamma, void* gamma, void* dx,
                       void* du, int* flags, void* workspace, int64_t workspace_bytes, int chunk0,
                       int chunk, void* stream);
/* value_pass + propagation_pass with HOST buffers (the numpy arrays of the
 * reference's StageExpansion, passes.py:291-361): same layouts and outputs
 * (Gamma, gamma, dx, du; flags may be NULL), host->device copies, solve and
 * device->host copies enqueued on `stream` (pinned host memory makes them
 * asynchronous, so calls on several streams overlap PCIe with compute).
 * Only what the kernels read is copied: for nx < 8 the upper triangles of
 * the symmetric P and R.  Workspace: ptc_lqr_host_workspace_bytes (device). */
int64_t ptc_lqr_host_workspace_bytes(int dtype, int batch, int horizon, int nx, int nu,
                                     int chunk0, int chunk);
int ptc_lqr_solve_host(int dtype, int batch, int horizon, int nx, int nu,
                       const void* P, const void* R, const void* M, const void* d,
                       const void* Fx, const void* Fu, const void* PT, const double* alpha,
                       void* Gamma, void* gamma, void* dx, void* du, int* flags,
                       void* workspace, int64_t workspace_bytes, int chunk0, int chunk,
                       void* stream);
/* The same host-buffer solve on the reference's own per-problem arrays
 * stacked over the batch ("stacked", problem-major: numpy's
 * np.stack([exp.P for exp in expansions]) of passes.py:291's StageExpansion
 * fields), so a pintoc caller hands its arrays over without a host
 * transpose:
 *   P (batch, horizon, nx, nx), R (batch, horizon, nu, nu),
 *   M (batch, horizon, nx, nu), d (batch, horizon, nu),
 *   Fx (batch, horizon, nx, nx), Fu (batch, horizon, nx, nu),
 *   PT (batch, nx, nx), alpha float64[batch];
 *   out Gamma (batch, horizon, nu, nx), gamma (batch, horizon, nu),
 *   dx (batch, horizon + 1, nx), du (batch, horizon, nu).
 * Each field crosses PCIe whole and is restacked to the SoA layout on the
 * device (an HBM-bound tiled transpose); results are bit-identical to
 * ptc_lqr_solve_host.  batch <= 2,097,120.  Workspace (device):
 * ptc_lqr_host_stacked_workspace_bytes. */
int64_t ptc_lqr_host_stacked_workspace_bytes(int dtype, int batch, int horizon, int nx, int nu,
                                             int chunk0, int chunk);
int ptc_lqr_solve_host_stacked(int dtype, int batch, int horizon, int nx, int nu,
                               const void* P, const void* R, const void* M, const void* d,
                               const void* Fx, const void* Fu, const void* PT,
                               const double* alpha, void* Gamma, void* gamma, void* dx, void* du,
                               int* flags, void* workspace, int64_t workspace_bytes, int chunk0,
                               int chunk, void* stream);
/* Element-level operations of the three scans, batched over items; item i
 * of a field with C components at f[c * n + i] (device pointers).
 *   ptc_value_elements   value_element_init (passes.py:192-228) of stages
 *     0..horizon-1 and the boundary element (stage horizon): out
 *     (3nx^2 + 2nx, horizon + 1) in the order A, Y, C, eta, b; flags[t]
 *     bit 1 when R_t + alpha I is not positive definite.  alpha: 1 double.
 *   ptc_value_combine    value_combine (passes.py:264-288), left = earlier
 *     stages: n pairs; flags[i] bit 4 when I + C_left Y_right is singular.
 *   ptc_affine_combine   kind 0: rollout_combine (passes.py:330-335),
 *     [F | e] maps, out = b after a; kind 1: costate_combine
 *     (passes.py:113-119), [df | dl | dc], a = the earlier segment. */
int ptc_value_elements(int dtype, int horizon, int nx, int nu, const void* P, const void* R,
                       const void* M, const void* d, const void* Fx, const void* Fu,
                       const void* PT, const double* alpha, void* out, int* flags, void* stream);
int ptc_value_combine(int dtype, int n, int nx, const void* left, const void* right, void* out,
                      int* flags, void* stream);
int ptc_affine_combine(int dtype, int n, int nx, int kind, const void* a, const void* b,
                       void* out, void* stream);
/* propagation_pass alone (passes.py:338-361) for a given feedback law:
 * Fx, Fu, Gamma (nu*nx), gamma (nu) in; dx, du out; d (nu) may be NULL.
 * Same workspace as ptc_lqr_solve. */
int ptc_propagate(int dtype, int batch, int horizon, int nx, int nu,
                  const void* Fx, const void* Fu, const void* Gamma, const void* gamma,
                  const void* d, void* dx, void* du, void* workspace, int64_t workspace_bytes,
                  int chunk0, int chunk, void* stream);
/* Which stage the definiteness gates of value_pass name (passes.py:231-241
 * _assert_spd_batch over R + alpha I, then over Q_t, passes.py:316-320) and
 * whether a combine was singular (ConditioningError, passes.py:280-283) --
 * the payload of the reference's DefinitenessError(stage, what) after a
 * solve returned flags.  Same SoA inputs as ptc_lqr_solve, alpha = device
 * float64[batch]; out = device int32[3 * batch]: row 0 first failing stage
 * of R + alpha I, row 1 first failing stage of Q_t (-1 = none), row 2 = 1
 * when some I + C Y is singular.  Error path only: one thread per problem
 * runs the exact dual-form recursion. */
int ptc_lqr_diagnose(int dtype, int batch, int horizon, int nx, int nu, const void* P,
                     const void* R, const void* M, const void* d, const void* Fx, const void* Fu,
                     const void* PT, const double* alpha, int* out, void* stream);
/* the plan the automatic choice would use for state size nx (for reporting
 * / depth probes; the same choice ptc_lqr_workspace_bytes and the solves make) */
int ptc_lqr_plan(int batch, int horizon, int nx, int chunk0, int chunk, int* out_chunk0,
                 int* out_chunk, int* out_levels);

/* ------------------------------------------------------------------------
 * Time-sharded LQR solve (BASELINE config 4): the horizon is split into
 * contiguous blocks, one per rank; same math as ptc_lqr_solve (value_pass +
 * propagation_pass, passes.py:291 / 338) with the scans' block-boundary
 * carries exchanged by the caller (one all-gather per scan).  Per rank:
 *   phase 0: value up-sweep of the local block -> block_out = block value
 *            aggregate (value_comps, 1, batch)
 *   [caller all-gathers block_out of every rank, rank-major:
 *    blocks_in = (world, value_comps, 1, batch)]
 *   phase 1: carry from the later blocks, value down-sweep, gains (and S, s
 *            if given; row `horizon` = the cost-to-go handed in), then the
 *            propagation up-sweep -> block_out = block affine aggregate
 *            (prop_comps, 1, batch)
 *   [caller all-gathers: blocks_in = (world, prop_comps, 1, batch)]
 *   phase 2: deviation entering the block from the earlier blocks, forward
 *            sweep -> dx (nx, horizon+1, batch; row `horizon` = the next
 *            block's first deviation), du.
 * Inputs are the local block's stages (global stages t_base ..
 * t_base+horizon-1); PT is read only when is_last.  The same workspace
 * (ptc_lqr_block_workspace_bytes) must be passed to all three phases.
 * ---------------------------------------------------------------------- */
int ptc_lqr_block_comps(int nx, int* value_comps, int* prop_comps);
int64_t ptc_lqr_block_workspace_bytes(int dtype, int batch, int horizon, int nx, int nu,
                                      int chunk0, int chunk);
int ptc_lqr_block_solve(int phase, int dtype, int batch, int horizon, int nx, int nu, int t_base,
                        int is_last, int rank, int world, const void* P, const void* R,
                        const void* M, const void* d, const void* Fx, const void* Fu,
                        const void* PT, const double* alpha, const void* blocks_in,
                        void* block_out, void* S, void* s, void* Gamma, void* gamma, void* dx,
                        void* du, int* flags, void* workspace, int64_t workspace_bytes,
                        int chunk0, int chunk, void* stream);
/* The same for one long problem (batch 1, nx >= 8, >= 1024 stages per
 * block) whose expansion is given as stage rows: rows[t * SC + c] with the
 * row [P (nx*nx) | R (nu*nu) | M (nx*nu) | d (nu) | Fx (nx*nx) | Fu (nx*nu)],
 * SC their total -- the layout the warp-per-unit kernels read, so no
 * transpose precedes the scans. */
int ptc_lqr_block_solve_rows(int phase, int dtype, int horizon, int nx, int nu, int t_base,
                             int is_last, int rank, int world, const void* rows, const void* PT,
                             const double* alpha, const void* blocks_in, void* block_out,
                             void* S, void* s, void* Gamma, void* gamma, void* dx, void* du,
                             int* flags, void* workspace, int64_t workspace_bytes, int chunk0,
                             int chunk, void* stream);

/* ------------------------------------------------------------------------
 * Batched device-resident solver
 *   one object = `batch` independent problems sharing model, cost and
 *   constraints (per-problem initial trajectories).  Replaces
 *   newton.py:129 newton_solve, outer.py:221 barrier_solve and
 *   outer.py:392 admm_solve; the augmentations are outer.py:30-157
 *   (BarrierAugmentation) and outer.py:252-333 (AdmmAugmentation); the
 *   passes inside one iteration are passes.py:122 costate_pass,
 *   passes.py:155 hamiltonian_expansion, value_pass, propagation_pass,
 *   problem.py:449 rollout and problem.py:476 total_cost.
 * ---------------------------------------------------------------------- */
typedef struct ptc_solver ptc_solver;

typedef struct ptc_problem_desc {
  int32_t dtype, batch, horizon, nx, nu;
  int32_t model;               /* PTC_DYN_* */
  double dyn_params[8];        /* pendulum: g, l, m, b, dt; cart-pole: g, l, m_cart, m_pole, dt */
  /* affine model x' = A x + B u + c: host or device arrays in dtype, shapes
   * (nx*nx, lin_rows, lin_batch), (nx*nu, lin_rows, lin_batch),
   * (nx, lin_rows, lin_batch) with lin_rows in {1, horizon} (time-invariant
   * or time-varying) and lin_batch in {1, batch}; lin_c may be NULL */
  const void* lin_a;
  const void* lin_b;
  const void* lin_c;
  int32_t lin_rows, lin_batch;
  /* quadratic cost (systems.py:80-139), float64 host arrays */
  const double* Q;             /* nx*nx */
  const double* R;             /* nu*nu */
  const double* Qf;            /* nx*nx */
  const double* goal;          /* nx, may be NULL (= 0) */
  /* box constraints (problem.py:233-340), float64 host, +-inf = absent;
   * any pointer may be NULL */
  const double* state_lower;
  const double* state_upper;
  const double* control_lower;
  const double* control_upper;
  /* solve */
  int32_t method;              /* PTC_METHOD_* */
  int32_t aug;                 /* PTC_AUG_* for PTC_METHOD_NEWTON */
  double aug_mu;               /* barrier weight for PTC_AUG_BARRIER */
  double alpha0, nu0, inner_tol;
  int32_t max_iters;
  double mu0, zeta, mu_tol;    /* barrier (outer.py:180-193) */
  double rho, residual_tol;    /* ADMM (outer.py:351-364), also the ADMM-aug rho */
  int32_t max_outer;
  int32_t hist_cap;            /* per-problem Newton iteration records kept */
  int32_t round_cap;           /* per-problem outer rounds recorded */
  int32_t keep_round_controls; /* barrier: store each round's controls */
  int32_t chunk0, chunk;       /* scan plan, 0 = automatic */
  int32_t rollout;             /* candidate rollout: 0 auto (log-depth Newton sweeps for
                                  tree plans with horizon >= 1024), 1 sequential,
                                  2 log-depth (tree plans) */
  /* time-block mode (config 4, horizon split across ranks): this solver
   * holds stages [t_base, t_base + horizon) of a longer horizon; the model
   * data, trajectories and z/v are the block's (states: horizon+1 rows, row 0
   * = the block's first state).  block_last: the block ends the horizon
   * (terminal cost and gradient live here).  Iterations then run through
   * ptc_solver_block_phase.  Affine models with nx >= 8, tree plans. */
  int32_t block_mode, t_base, block_last;
  /* user-defined model (model id from ptc_model_load): its device array of
   * float64 data (per-stage matrices, tables ...), read by the model's code
   * as `data`; may be NULL.  Its parameters are dyn_params (`prm`). */
  const void* user_data;
  /* user-defined cost (a model library built with a cost source): its
   * parameters (`cprm`) and device float64 array (`cdata`, may be NULL) */
  double cost_params[8];
  const void* cost_data;
  /* user-defined constraints (a model library built with a constraint
   * source): state / control row counts (the box fields stay NULL), their
   * parameters and device float64 array */
  int32_t con_rows_state, con_rows_control;
  double con_params[8];
  const void* con_data;
} ptc_problem_desc;

/* Register a user-defined dynamics model (reference problem.py:59-112: a
 * DynamicsModel subclass with f, fx, fu, fxx, fuu, fxu) compiled into its own
 * shared library from the model's per-stage CUDA code
 * (paper_2409_20027_b200/usermodel.py, csrc/user_model.cuh).  The library's
 * fused Newton kernel sets (f64, f32) are registered under a fresh model id
 * (>= PTC_DYN_USER_BASE) for use as ptc_problem_desc.model; loading the
 * same path twice returns the same id.  nx / nu receive the model's sizes. */
#define PTC_DYN_USER_BASE 100
int ptc_model_load(const char* path, int* model_id, int* nx, int* nu);

int64_t ptc_solver_workspace_bytes(const ptc_problem_desc* desc);
int ptc_solver_create(const ptc_problem_desc* desc, void* workspace, int64_t workspace_bytes,
                      ptc_solver** out);
int ptc_solver_destroy(ptc_solver* s);

/* Load initial trajectories: states (nx, horizon+1, batch), controls
 * (nu, horizon, batch); host (on_device = 0) or device pointers.  Resets the
 * solver state.  For PTC_AUG_ADMM Newton solves, z and v (W, horizon, batch)
 * may be given (else zero). */
int ptc_solver_load(ptc_solver* s, const void* states, const void* controls,
                    const void* z, const void* v, int on_device, void* stream);

/* first stage t where x_{t+1} != f_t(x_t, u_t) per problem (-1 if
 * consistent), int32 host array [batch] -- newton.py:118-126 */
int ptc_solver_check_consistency(ptc_solver* s, int32_t* first_bad_stage, void* stream);

/* Enqueue n device iterations (costate + expansion, value scan, propagation
 * scan, rollout + cost, trust-region control, outer-loop control). */
int ptc_solver_iterate(ptc_solver* s, int n, void* stream);

/* Number of problems still running (synchronises the stream). */
int ptc_solver_running(ptc_solver* s, int32_t* n_running, void* stream);
/* the same count enqueued on `stream` without waiting (n_running: pinned
 * host memory, valid once the stream reaches the copy -- record an event):
 * lets a host loop keep the next group of iterations queued while it polls
 * the previous one */
int ptc_solver_running_async(ptc_solver* s, int32_t* n_running, void* stream);

/* The whole solve loop enqueued as ONE device-resident CUDA graph (replaces
 * the host loop of newton.py:157-208 / outer.py:221-245, 392-427 driven by
 * ptc_solver_iterate + ptc_solver_running): a conditional WHILE node replays
 * `group` iterations, then the device stops once no problem is running or
 * max_launch iterations were launched.  launched (pinned host int32, may be
 * NULL) receives the iteration count once the stream reaches it.  Returns
 * PTC_ERR_CUDA if the driver cannot build conditional graphs. */
int ptc_solver_loop(ptc_solver* s, int group, int max_launch, int32_t* launched, void* stream);

/* Pass-level entry points on the loaded trajectory (buffer 0):
 *   expand  = costate_pass + hamiltonian_expansion (passes.py:122, 155)
 *   lqr     = value_pass + propagation_pass on that expansion
 *   rollout = problem.py:449 rollout (controls -> states, from x_0)
 *   cost    = problem.py:476 total_cost -> "cur_cost", "bad_index" */
int ptc_solver_expand(ptc_solver* s, void* stream);
int ptc_solver_lqr(ptc_solver* s, const double* alpha_host, void* stream);
int ptc_solver_rollout(ptc_solver* s, void* stream);
int ptc_solver_total_cost(ptc_solver* s, void* stream);

/* One phase of a time-sharded Newton iteration (block_mode solvers); the
 * caller runs the collective named after each phase between phases, every
 * rank the same sequence (sharded.TimeShardedNewton).  R = solver dtype,
 * CC = nx*nx + nx, VC = 3*nx*nx + 2*nx, all buffers device, (comps, 1, batch):
 *   phase 0  cost partials, co-state up-sweep    out: CC  (R)   -> all-gather
 *   phase 1  in: gathered co-state aggregates (world, CC); carry, co-state
 *            down-sweep + expansion, value up-sweep  out: VC (R) -> all-gather
 *   phase 2  in: gathered value aggregates; value carry + down-sweep + gains,
 *            propagation up-sweep                out: CC  (R)   -> all-gather
 *   phase 3  in: gathered propagation aggregates; propagation down-sweep
 *            out: 6 (double): [sum du^2, sum du.d | max |du|, 3 LQR flag bits]
 *            -> all-reduce SUM rows 0-1, MAX rows 2-5
 *   phase 4  in: reduced phase-3 vector; rollout up-sweep of u + du
 *            out: CC (R) -> all-gather
 *   phase 5  in: gathered rollout aggregates; x0 = aux (nx, 1, batch): the
 *            horizon's initial state; rollout down-sweep, cost partials
 *            out: 7 (double): [cur l, cur c, cand l, cand c | diverged |
 *            cur first infeasible, cand first infeasible (global stage*W +
 *            row, 1e300 = none)] -> all-reduce SUM 0-3, MAX 4, MIN 5-6
 *   phase 6  in: reduced phase-5 vector; trust-region control, round end
 *            out: 2 (double): ADMM residual maxima -> all-reduce MAX
 *   phase 7  in: reduced phase-6 vector; outer-loop control
 *   phase 8  (rollout of buffer 0, problem.py:449) up-sweep  out: CC -> all-gather
 *   phase 9  in: gathered phase-8 aggregates, aux = x0; down-sweep */
int ptc_solver_block_phase(ptc_solver* s, int phase, const void* in, void* out, const void* aux,
                           int rank, int world, void* stream);

/* Set per-problem loop state between ptc_solver_load and ptc_solver_iterate:
 * "alpha", "nu" (float64[batch], the Levenberg-Marquardt weight and growth
 * factor newton.py:154-208 carries between iterations) and "mu" (float64
 * [batch], the barrier weight of PTC_AUG_BARRIER Newton solves).  Together
 * with the loaded trajectory and z / v this is the complete state entering
 * one reference iteration, so the device can restart from any recorded
 * reference iteration.  src host (on_device = 0) or device. */
int ptc_solver_write(ptc_solver* s, const char* name, const void* src, int64_t bytes,
                     int on_device, void* stream);

/* Copy a named buffer out (dst host or device).  Names: states, controls
 * (current trajectory), lam, P, R, M, d, Fx, Fu, PT, S, s, Gamma, gamma, dx,
 * du, z, v, status, iters, term, round, hist_len, hist, cur_cost, cand_cost (the
 * last iteration's candidate cost, float64), alpha, nu, mu,
 * bad_value (float64: the constraint value w at bad_index, InfeasibleError.value),
 * round_mu, round_cost, round_iters, round_term, round_rp, round_rd,
 * round_controls, bad_index, flags, rollout_state (bit 0 skipped, bit 1 log-depth
 * rollout converged, bit 2 converged in the scratch buffer).  ptc_solver_buffer_info reports the
 * element count and element size. */
int ptc_solver_buffer_info(ptc_solver* s, const char* name, int64_t* numel, int32_t* elem_bytes);
int ptc_solver_read(ptc_solver* s, const char* name, void* dst, int64_t bytes, int dst_on_device,
                    void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PINTOC_B200_H */
