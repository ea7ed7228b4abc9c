/*
 * gsls.h — C ABI of the B200-native GPU-SLS solver core (libgsls.so).
 *
 * Plain C: device pointers (float32, row-major, batch-major, the layouts of
 * the reference's LtvQpData, /root/reference/pkg/src/scanmpc/lqr.py:53-68),
 * sizes, and a cudaStream_t passed as void*.  No torch types.  Every entry
 * point returns a gsls_status_t; details of the last failure (instance,
 * stage, column) are read with gsls_last_error().
 *
 * Each function below names the reference interface it replaces.  The
 * reference is a Python package with no FFI of its own; these are the
 * calls its module-level entry points bind to (see INTEGRATION.md for the
 * ctypes stubs).
 */
#ifndef GSLS_H_
#define GSLS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GSLS_OK = 0,
  GSLS_ERR_ARG = 1,               /* ValueError: bad shape/argument                       */
  GSLS_ERR_CUDA = 2,              /* CUDA runtime failure                                   */
  GSLS_ERR_SINGULAR_STAGE = 3,    /* lqr.SingularStageError (lqr.py:35, :213-215; sls.py:321-326) */
  GSLS_ERR_ILL_CONDITIONED = 4,   /* lqr.IllConditionedCombineError (lqr.py:31, :229-232)   */
  GSLS_ERR_CACHE_INVALIDATED = 5, /* lqr.CacheInvalidatedError (lqr.py:39, :426-427)        */
  GSLS_ERR_NONFINITE = 6,         /* ArithmeticError non-finite dynamics (sqp.py:125-131)   */
  GSLS_ERR_TOO_LARGE = 7,         /* dimensions beyond the compiled limits                  */
  GSLS_ERR_NO_DEVICE = 8,
  GSLS_ERR_LOWRANK = 9            /* internal: a factored combine met an indefinite P (never
                                     returned; the scan is re-run with dense combines)     */
} gsls_status_t;

/* labels carried with GSLS_ERR_SINGULAR_STAGE (error.aux2) */
enum {
  GSLS_LABEL_R = 1,            /* "singular R at stage i"                       lqr.py:323 */
  GSLS_LABEL_R_BPB = 2,        /* "singular R + B'PB at stage i"                lqr.py:399 */
  GSLS_LABEL_QU = 3,           /* "singular Qu block at (k=.., j=..)"           sls.py:258-261 */
  GSLS_LABEL_QU_BPB = 4,       /* "singular Qu + B'PB block at (k=.., j=..)"    sls.py:288-293 */
  GSLS_LABEL_NONFINITE_DYN = 5,
  GSLS_LABEL_NONFINITE_CON = 6
};

typedef struct {
  int32_t code;      /* gsls_status_t                                   */
  int32_t instance;  /* batch index, -1 if not instance-specific         */
  int32_t where;     /* stage k / scan op                                */
  int32_t aux;       /* SLS column j, or -1                              */
  int32_t aux2;      /* GSLS_LABEL_* for singular blocks                 */
  char message[256];
} gsls_error_t;

/* Problem dimensions; one set per batch of independent instances. */
typedef struct {
  int32_t nx, nu, nc, nf, N; /* lqr.py:70-88 properties */
  int32_t batch;
} gsls_dims_t;

/* Stagewise QP data (lqr.py:53-68), device, batch-major.  Precision split:
 * matrices are float32 (they feed the fp32 factorization), vectors are
 * float64 (the replay and the ADMM iterate run in fp64 — see DESIGN.md §3).
 *   float32:  A (B,N,nx,nx) B (B,N,nx,nu) Q (B,N,nx,nx) R (B,N,nu,nu)
 *             S (B,N,nu,nx) or NULL (= 0) QN (B,nx,nx) C (B,N,nc,nx)
 *             D (B,N,nc,nu) CN (B,nf,nx)
 *   float64:  b (B,N,nx) q (B,N,nx) r (B,N,nu) qN (B,nx) f (B,N,nc) fN (B,nf)
 *             dx0 (B,nx) */
typedef struct {
  const float* A;
  const float* B;
  const double* b;
  const float* Q;
  const float* R;
  const float* S;
  const double* q;
  const double* r;
  const float* QN;
  const double* qN;
  const float* C;
  const float* D;
  const double* f;
  const float* CN;
  const double* fN;
  const double* dx0;
} gsls_qp_t;

/* admm.AdmmSettings (admm.py:24-39). */
typedef struct {
  double rho0, rho_min, rho_max;
  int32_t sigma;
  double tol_primal, tol_dual;
  int32_t max_iter;
} gsls_admm_settings_t;

/* admm.AdmmState (admm.py:42-55), device arrays, in/out (mutated in place,
 * as the reference mutates its warm_start, admm.py:164/:186/:197).
 * z, lam, y: (B, N*nc+nf) float64; rho, r_primal, r_dual: (B) float64;
 * generation, iteration: (B) int32. */
typedef struct {
  double *z, *lam, *y;
  double *rho, *r_primal, *r_dual;
  int32_t *generation, *iteration;
} gsls_admm_state_t;

/* admm.AdmmStats (admm.py:58-67), device int32 arrays (B). */
typedef struct {
  int32_t *iterations, *converged, *rho_changes, *cache_builds;
} gsls_admm_stats_t;

typedef struct gsls_ctx gsls_ctx; /* workspace + LQR factorization cache for one dims */

/* ---- context ---------------------------------------------------------- */
int gsls_version(void);
int gsls_last_error(gsls_error_t* out);
int gsls_ctx_create(const gsls_dims_t* dims, gsls_ctx** out);
int gsls_ctx_destroy(gsls_ctx* ctx);
/* Synchronizes the stream and reports the first per-instance error recorded
 * by earlier kernels (singular blocks, ill-conditioned combines, non-finite
 * model output), clearing the record. */
int gsls_ctx_check(gsls_ctx* ctx, void* stream);
/* bytes of device memory held by the context */
int64_t gsls_ctx_bytes(const gsls_ctx* ctx);

/* ---- scan plan (scan.py:141-234 tree order), host-side, for inspection --
 * Writes the combine ops of a scan of `length` elements: ops[3*i..3*i+2] =
 * (dst, earlier, later) slot ids, layer_off[0..layers] offsets into ops,
 * out_slot[0..length-1] (-1 = identity).  Returns number of ops in *n_ops. */
int gsls_scan_plan(int32_t length, int32_t reverse, int32_t max_ops, int32_t* ops,
                   int32_t* layer_off, int32_t* out_slot, int32_t* n_ops, int32_t* n_layers);

/* ---- LQR (lqr.py) ------------------------------------------------------ */
/* lqr.solve (lqr.py:366): full solve. Outputs (float64) dx (B,N+1,nx)
 * du (B,N,nu) k (B,N,nu) p (B,N+1,nx); (float32) K (B,N,nu,nx)
 * P (B,N+1,nx,nx); K/k/P/p may be NULL.
 * Leaves the factorization cache in ctx stamped with `generation`. */
int gsls_lqr_solve(gsls_ctx* ctx, const gsls_qp_t* qp, int32_t generation, double* dx, double* du,
                   float* K, double* k, float* P, double* p, void* stream);
/* lqr.build_cache (lqr.py:372) == gsls_lqr_solve with the cache kept. */
/* lqr.solve_cached (lqr.py:419): replay with new linear terms only.
 * q (B,N,nx) r (B,N,nu) qN (B,nx); generation must match the cache stamp. */
int gsls_lqr_solve_cached(gsls_ctx* ctx, const gsls_qp_t* qp, const double* q, const double* r,
                          const double* qN, int32_t generation, double* dx, double* du, double* k,
                          double* p, void* stream);

/* ---- ADMM QP (admm.py:153-203), batched -------------------------------- */
/* Runs every instance to convergence / max_iter with per-instance rho,
 * cache rebuilds on committed rho changes, exact reference control flow.
 * dx (B,N+1,nx), du (B,N,nu) (float64) receive the last LQR iterate. */
int gsls_admm_solve_qp(gsls_ctx* ctx, const gsls_qp_t* qp, const gsls_admm_settings_t* settings,
                       gsls_admm_state_t* state, gsls_admm_stats_t* stats, double* dx, double* du,
                       void* stream);

/* The first ADMM cache build (LQR factorization at the augmented costs, all
 * instances, at rho (B) float64) issued ahead of gsls_admm_solve_qp, which then
 * skips it.  Lets the caller overlap the build with independent work on another
 * stream (the robust RTI step overlaps it with the SLS synthesis: the
 * factorization of admm.py:171-178 does not depend on the tightened offsets f);
 * the caller orders the streams.  Same result as the solve's own first build. */
int gsls_admm_build_cache(gsls_ctx* ctx, const gsls_qp_t* qp, const double* rho, void* stream);

/* Exports the last solve held by ctx: K (B,N,nu,nx) and P (B,N+1,nx,nx) of
 * the current factorization, k (B,N,nu) and p (B,N+1,nx) of the last replay
 * (the LqrSolution the reference returns in AdmmResult.solution, admm.py:203).
 * Any output may be NULL. */
int gsls_ctx_export_solution(gsls_ctx* ctx, float* K, double* k, float* P, double* p, void* stream);

/* ---- SLS (sls.py) -------------------------------------------------------
 * Per-instance SLS objects use a triangular CELL layout: cell(k, j) for
 * 0 <= j < k <= N, index j*N - j*(j-1)/2 + (k-j-1), ncell = N(N+1)/2
 * (gsls_sls_ncell).  Cells with k <= N-1 carry stage quantities (costs, gains,
 * Phi^u, tau); cells with k = N carry the terminal ones (Qx_term, tau_term via
 * column j).  Phi^x is defined on every cell. */
int gsls_sls_ncell(int32_t N);
/* Column sharding of the SLS objects: restricts this context's
 * SLS work and storage to disturbance columns [j0, j1) (j1 = -1: N).  Every SLS
 * array then holds only the shard's cells, in the same order at shard-local index
 * cell(k, j) - cell(j0 + 1, j0); gsls_sls_tighten returns the shard's partial sums
 * of h and hf (sum them over shards, e.g. an all-reduce); tau_term is written for
 * the shard's columns only.  Columns are independent (sls.py:227-318), so a
 * shard's cells equal those of the unsharded synthesis.  Call before the first
 * SLS call on ctx. */
int gsls_sls_set_columns(gsls_ctx* ctx, int32_t j0, int32_t j1);
/* Host-side inspection of the merged column schedules: cvf = 1 the reverse
 * CVF grid scan (leaves at cell(k, j) for k in [j+1, N]), cvf = 0 the forward
 * product scan (leaf of position p at cell(p+1, j)).  ops as gsls_scan_plan;
 * out_cell[cell(k, j)] = slot holding the column-j output of position k
 * (CVF) / of position k-1 (product).  Sizes only when max_ops is too small. */
int gsls_sls_plan(int32_t N, int32_t cvf, int32_t max_ops, int32_t* ops, int32_t* layer_off, int32_t* out_cell,
                  int32_t* n_ops, int32_t* n_layers, int32_t* n_slots);
/* sls.assemble_costs (sls.py:176-200): [C D]' diag(tau) [C D] + blkdiag(Qbar, Rbar)
 * per cell, CN' diag(tau_term) CN + QbarN on terminal cells.  tau (B,ncell,nc)
 * float64 or NULL (= unweighted, sls.py:189); tau_term (B,N,nf) or NULL.
 * Qbar (nx,nx) Rbar (nu,nu) QbarN (nx,nx) float32, one set per instance when
 * weights_per_instance != 0.  C, D, CN are taken from qp. */
int gsls_sls_assemble(gsls_ctx* ctx, const gsls_qp_t* qp, const double* tau, const double* tau_term,
                      const float* Qbar, const float* Rbar, const float* QbarN, int32_t weights_per_instance,
                      void* stream);
/* Explicit SlsCosts (sls.py:129-143) in cell layout: Qx (B,ncell,nx,nx) (terminal
 * cells hold Qx_term), Qu (B,ncell,nu,nu), Qux (B,ncell,nu,nx), float64. */
int gsls_sls_set_costs(gsls_ctx* ctx, const double* Qx, const double* Qu, const double* Qux, void* stream);
/* Reads back the costs held by ctx in the gsls_sls_set_costs layout; any may be NULL. */
int gsls_sls_export_costs(gsls_ctx* ctx, double* Qx, double* Qu, double* Qux, void* stream);
/* sls.synthesize (sls.py:227-318) on the costs held by ctx; A, B from qp,
 * E (B,N,nx,nx) float32.  The response stays on the device. */
int gsls_sls_synthesize(gsls_ctx* ctx, const gsls_qp_t* qp, const float* E, void* stream);
/* sls.tighten (sls.py:329-341) of the response held by ctx with C, D, CN
 * from qp: h (B,N,nc), hf (B,nf), float64. */
int gsls_sls_tighten(gsls_ctx* ctx, const gsls_qp_t* qp, double* h, double* hf, void* stream);
/* sls.compute_duals (sls.py:150-173): lam is the stacked multiplier
 * (B, N*nc+nf) (AdmmState.lam, admm.py:82-88) -> tau (B,ncell,nc),
 * tau_term (B,N,nf) [beta, beta_term same shapes, may be NULL], float64;
 * C, D, CN from qp.  use_response = 0 reproduces response=None (beta = 0);
 * reuse_rownorms = 1 skips recomputing the row norms of the last
 * gsls_sls_tighten (same C, D, CN). */
int gsls_sls_duals(gsls_ctx* ctx, const gsls_qp_t* qp, const double* lam, double eps, int32_t use_response,
                   int32_t reuse_rownorms, double* tau, double* tau_term, double* beta, double* beta_term,
                   void* stream);
/* Loads an SlsResponse built elsewhere: Phi_x (B,ncell,nx,nx), Phi_u (B,ncell,nu,nx). */
int gsls_sls_import_response(gsls_ctx* ctx, const float* phix, const float* phiu, void* stream);
/* SlsResponse export (sls.py:51-92): Phi_x (B,ncell,nx,nx), Phi_u and gains
 * (B,ncell,nu,nx) (zero on terminal cells), float32; any may be NULL. */
int gsls_sls_export(gsls_ctx* ctx, float* phix, float* phiu, float* gains, void* stream);
/* sls.sls_cost (sls.py:344-358) of the response held by ctx: cost (B,) float64 =
 * sum over cells of tr(Phi' W Phi) = ||L' Phi||_F^2 (W = L L': Qbar for Phi^x at k < N,
 * QbarN at k = N, Rbar for Phi^u); weights nx x nx / nu x nu float64 device arrays. */
int gsls_sls_cost(gsls_ctx* ctx, const double* Qbar, const double* Rbar, const double* QbarN, double* cost,
                  void* stream);

/* ---- SQP linearization (sqp.py:105-147) ----------------------------------- */
enum { GSLS_MODEL_DUBINS = 1, GSLS_MODEL_PLANAR_QUAD = 2, GSLS_MODEL_PENDULUM = 3,
       GSLS_MODEL_QUAD12 = 4, GSLS_MODEL_SYNTHETIC = 5 };

typedef struct {
  int32_t model_id;             /* GSLS_MODEL_*                                        */
  const double* params;         /* model parameters + constraint block (device)        */
  int32_t cons_offset;          /* index of the constraint block in params:
                                   n_obs, u_min[nu], u_max[nu], (cx, cy, r) per obstacle */
  const double *x, *u;          /* linearization trajectory (B,N+1,nx), (B,N,nu)       */
  const double *h, *hf;         /* tightenings (B,N,nc), (B,nf) or NULL                */
  const double* xbar0;          /* measured state (B,nx) or NULL (dx0 = 0)              */
  const double *Qw, *Rw, *QNw;  /* tracking weights (nx,nx) (nu,nu) (nx,nx)             */
  const double *xref, *uref;    /* reference (N+1,nx), (N,nu)                           */
  const double* E_const;        /* constant disturbance map (nx,nx) or NULL             */
  int32_t write_weights;        /* 1: also write Q, R, S (= 0), QN and E                */
} gsls_linearize_args_t;

/* sqp.linearize: writes A, B, b, C, D, f (= -g - h), q, r, CN, fN, qN, dx0 of
 * `out` (device buffers of the gsls_qp_t layout; the pointers are written
 * through), and Q, R, S, QN, E (B,N,nx,nx) when write_weights is set.
 * Non-finite dynamics raise GSLS_ERR_NONFINITE naming the stage. */
int gsls_linearize(gsls_ctx* ctx, const gsls_linearize_args_t* args, const gsls_qp_t* out, float* E, void* stream);

/* Trajectory terms of the SQP loop (sqp.py:150-187) for the trajectory in
 * args (x, u, h, hf, xbar0; weights/reference for the tracking cost):
 * out (B,8) float64 = {tracking cost J, max|defect|, sum|defect|,
 * max(g + h) (unclamped), sum max(g + h, 0), sum|x0 - xbar0|, max|x0 - xbar0|, n_obs}. */
int gsls_traj_eval(gsls_ctx* ctx, const gsls_linearize_args_t* args, double* out, void* stream);

/* ---- closed-loop verification (rollout.py:47-93) ------------------------------
 * Replaces rollout.closed_loop (rollout.py:47) for `rollouts` disturbance
 * sequences per instance of the context's batch: u_k = v_k + sum_{j<k}
 * Phi^u_{k,j} w_hat_j, x_{k+1} = f(x_k, u_k) + E d_k, w_hat_k = E^+ (x_{k+1} - f),
 * stage/terminal constraint values, tube slack min(g_nom + h_k + tol_lin - g)
 * (+inf without h), flags.  E must be state-independent (true for every
 * device model); E_pinv is its range-restricted pseudo-inverse (rollout.py:41-44). */
typedef struct {
  int32_t model_id;             /* GSLS_MODEL_*                                        */
  const double* params;         /* model parameters + constraint block (device)        */
  int32_t cons_offset;          /* index of the constraint block in params             */
  const double *x, *u;          /* nominal trajectory (B,N+1,nx), (B,N,nu)             */
  const float* phi_u;           /* (B, N(N+1)/2, nu, nx) cell layout, or NULL           */
  const double *E, *E_pinv;     /* (nx,nx) disturbance map and its pseudo-inverse       */
  const double* disturbances;   /* true injected w (B, rollouts, N, nx)                 */
  const double* h;              /* stage tightening (B,N,nc) or NULL (no tube check)    */
  double tol_lin;               /* rollout.py:48 default 1e-2                           */
  int32_t rollouts;             /* disturbance sequences per instance                   */
} gsls_rollout_args_t;

typedef struct {                /* all device buffers, float64 unless noted             */
  double* x;                    /* (B, R, N+1, nx) realized states                      */
  double* u;                    /* (B, R, N, nu) applied controls                       */
  double* w;                    /* (B, R, N, nx) reconstructed disturbances             */
  double* stage_g;              /* (B, R, N, nc)                                        */
  double* terminal_g;           /* (B, R, nf)                                           */
  double* tube_margin;          /* (B, R, N), +inf where unchecked                      */
  double* max_w_norm;           /* (B, R)                                               */
  int32_t* flags;               /* (B, R, 3) int32: safe, tube_ok, disturbance_model_violated */
} gsls_rollout_out_t;

int gsls_rollout(gsls_ctx* ctx, const gsls_rollout_args_t* args, const gsls_rollout_out_t* out, void* stream);

/* f -= h, fN -= hf in place (the tightened re-linearization, sqp.py:136/:140). */
int gsls_apply_tightening(gsls_ctx* ctx, double* f, double* fN, const double* h, const double* hf, void* stream);
/* RTI update (sqp.py:293-301, :40-43): plan = prev + (dx, du); warm start =
 * plan shifted with the last stage duplicated; u0 = plan.u[0]; cost (B) =
 * tracking cost of the plan (models.py:85-93) or NULL.  All float64. */
int gsls_rti_apply(gsls_ctx* ctx, const double* prev_x, const double* prev_u, const double* dx, const double* du,
                   double* plan_x, double* plan_u, double* warm_x, double* warm_u, double* u0, const double* Qw,
                   const double* Rw, const double* QNw, const double* xref, const double* uref, double* cost,
                   void* stream);

/* ---- one MPC step for the whole batch (the metric's unit of work) ------------
 * Replaces sls.rti_robust_step (sls.py:500-525) for every instance of the
 * context when robust = 1, sqp.rti_step (sqp.py:272-302) when robust = 0:
 * linearize at (lin.x, lin.u) = (prev_x, prev_u) with lin.xbar0; [robust: SLS
 * costs with the duals tau / tau_term when use_tau (else unweighted),
 * synthesize, tighten into h / hf, f -= h]; admm.solve_qp from a cold state
 * (state reset to rho0) or the given one (warm_admm); [robust: compute_duals
 * into tau, tau_term, beta, beta_term for the next step]; plan / warm start / u0
 * / tracking cost.  The ADMM's first factorization runs on the context's side
 * stream concurrently with the SLS chain unless no_overlap.  Capturable into a
 * CUDA graph.  All pointers are device buffers of the layouts above; `qp` is the
 * QP workspace the step writes.  E_in (B,N,nx,nx) or NULL overrides the
 * disturbance maps after the linearization. */
typedef struct {
  gsls_linearize_args_t lin;      /* model, x = prev_x, u = prev_u, xbar0, weights     */
  const gsls_qp_t* qp;            /* QP workspace (written)                             */
  float* E;                       /* (B,N,nx,nx) disturbance maps (written)             */
  const float* E_in;              /* or NULL                                            */
  int32_t robust, use_tau, warm_admm, no_overlap;
  const float *Qbar, *Rbar, *QbarN;  /* SLS weights (nx,nx) (nu,nu) (nx,nx)            */
  double *tau, *tau_term, *beta, *beta_term;  /* cell-layout duals, in / out           */
  double eps;                     /* compute_duals epsilon                              */
  gsls_admm_settings_t admm;
  gsls_admm_state_t state;
  gsls_admm_stats_t stats;
  double *h, *hf;                 /* tightenings (B,N,nc), (B,nf)                       */
  double *dx, *du;                /* QP solution (B,N+1,nx), (B,N,nu)                   */
  double *plan_x, *plan_u, *warm_x, *warm_u, *u0;
  double* cost;                   /* (B) tracking cost of the plan, or NULL             */
} gsls_rti_step_args_t;

int gsls_rti_step(gsls_ctx* ctx, const gsls_rti_step_args_t* args, void* stream);

/* The per-instance result record a multi-GPU batch exchanges (one all-gather per
 * step, dist.py): rec (B, nu + 4) float64 = u0, ADMM iterations, converged, rho
 * changes, cost (0 when cost is NULL). */
int gsls_rti_pack_results(gsls_ctx* ctx, const double* u0, const gsls_admm_stats_t* stats, const double* cost,
                          double* rec, void* stream);

/* ---- profiling (bench.py roofline evidence) -----------------------------
 * When enabled, every kernel launch records a CUDA event pair on its stream.
 * gsls_prof_read synchronizes and returns, per kernel family (order:
 * leaf, cvf_lqr, gains, cot, replay, sls_assemble, sls_leaf, sls_cvf,
 * sls_gains, sls_matprod, sls_phiu, sls_rownorm, sls_small, linearize,
 * rti_misc): accumulated ms, work units (combines for scan families,
 * instances for the replay) and launch counts, then resets.  Returns the
 * number of families. */
int gsls_prof_enable(int32_t on);
int gsls_prof_read(double* ms, double* units, int64_t* launches, int32_t max_ids);

#ifdef __cplusplus
}
#endif
#endif /* GSLS_H_ */
