// extern "C" entry points of libgsls.so (declared in include/gsls.h).
#include <cstring>

#include "ctx.h"

struct gsls_ctx {
  gsls::Ctx* impl;
};

namespace gsls {
int ctx_create(const gsls_dims_t* dims, Ctx** out);
void ctx_destroy(Ctx* c);
int get_last_error(gsls_error_t* out);
int check_errors(Ctx* c, cudaStream_t st, const char* what);
void set_error(int code, int inst, int where, int aux, int label, const char* msg);
int lqr_solve(Ctx* c, const gsls_qp_t* qp, int generation, double* dx, double* du, float* K, double* k, float* P,
              double* p, cudaStream_t st);
int lqr_solve_cached(Ctx* c, const gsls_qp_t* qp, const double* q, const double* r, const double* qN,
                     int generation, double* dx, double* du, double* k, double* p, cudaStream_t st);
int admm_build(Ctx* c, const gsls_qp_t* qp, const double* rho, cudaStream_t st);
int admm_solve(Ctx* c, const gsls_qp_t* qp, const gsls_admm_settings_t* s, gsls_admm_state_t* state,
               gsls_admm_stats_t* stats, double* dx, double* du, cudaStream_t st);
int ctx_export(Ctx* c, float* K, double* k, float* P, double* p, cudaStream_t st);
int sls_assemble(Ctx* c, const gsls_qp_t* qp, const double* tau, const double* tau_term, const float* Qbar,
                 const float* Rbar, const float* QbarN, int weights_per_instance, cudaStream_t st);
int sls_set_costs(Ctx* c, const double* Qx, const double* Qu, const double* Qux, cudaStream_t st);
int sls_synthesize(Ctx* c, const gsls_qp_t* qp, const float* E, cudaStream_t st, bool check);
int sls_tighten(Ctx* c, const gsls_qp_t* qp, double* h, double* hf, cudaStream_t st);
int sls_duals(Ctx* c, const gsls_qp_t* qp, const double* lam, double eps, int use_response, int reuse_rownorms,
              double* tau, double* tau_term, double* beta, double* beta_term, cudaStream_t st);
int sls_import(Ctx* c, const float* phix, const float* phiu, cudaStream_t st);
int sls_export_costs(Ctx* c, double* Qx, double* Qu, double* Qux, cudaStream_t st);
int sls_plan(int N, int cvf, int max_ops, int* ops, int* layer_off, int* out, int* n_ops, int* n_layers,
             int* n_slots);
int linearize(Ctx* c, const gsls_linearize_args_t* in, gsls_qp_t* out_qp, float* E, cudaStream_t st);
int traj_eval(Ctx* c, const gsls_linearize_args_t* in, double* out, cudaStream_t st);
int apply_tightening(Ctx* c, double* f, double* fN, const double* h, const double* hf, cudaStream_t st);
int rti_apply(Ctx* c, const double* px, const double* pu, const double* dx, const double* du, double* plan_x,
              double* plan_u, double* warm_x, double* warm_u, double* u0, const double* Qw, const double* Rw,
              const double* QNw, const double* xref, const double* uref, double* cost, cudaStream_t st);
int sls_export(Ctx* c, float* phix, float* phiu, float* gains, cudaStream_t st);
int sls_cost(Ctx* c, const double* Qbar, const double* Rbar, const double* QbarN, double* cost, cudaStream_t st);
int rollout(Ctx* c, const gsls_rollout_args_t* in, const gsls_rollout_out_t* out, cudaStream_t st);
int sls_set_columns(Ctx* c, int j0, int j1);
int rti_step(Ctx* c, const gsls_rti_step_args_t* a, cudaStream_t st);
int rti_pack_results(Ctx* c, const double* u0, const gsls_admm_stats_t* stats, const double* cost, double* rec,
                     cudaStream_t st);
}  // namespace gsls

using namespace gsls;

static int fail_null(const char* what) {
  char msg[128];
  snprintf(msg, sizeof msg, "null %s", what);
  set_error(GSLS_ERR_ARG, -1, 0, 0, 0, msg);
  return GSLS_ERR_ARG;
}

static int check_qp(const gsls_qp_t* qp, const gsls_dims_t& d) {
  if (!qp) return fail_null("qp");
  if (!qp->QN || !qp->qN || !qp->dx0) return fail_null("QN/qN/dx0");
  if (d.N > 0 && (!qp->A || !qp->B || !qp->b || !qp->Q || !qp->R || !qp->q || !qp->r)) return fail_null("stage data");
  if (d.N > 0 && d.nc > 0 && (!qp->C || !qp->D || !qp->f)) return fail_null("C/D/f");
  if (d.nf > 0 && (!qp->CN || !qp->fN)) return fail_null("CN/fN");
  return GSLS_OK;
}

extern "C" {

int gsls_version(void) { return 1; }

int gsls_last_error(gsls_error_t* out) {
  if (!out) return GSLS_ERR_ARG;
  return get_last_error(out);
}

int gsls_ctx_create(const gsls_dims_t* dims, gsls_ctx** out) {
  if (!dims || !out) return fail_null("argument");
  Ctx* c = nullptr;
  int rc = ctx_create(dims, &c);
  if (rc) return rc;
  *out = new gsls_ctx{c};
  return GSLS_OK;
}

int gsls_ctx_destroy(gsls_ctx* ctx) {
  if (!ctx) return GSLS_OK;
  ctx_destroy(ctx->impl);
  delete ctx;
  return GSLS_OK;
}

int64_t gsls_ctx_bytes(const gsls_ctx* ctx) { return ctx ? ctx->impl->bytes : 0; }

int gsls_ctx_check(gsls_ctx* ctx, void* stream) {
  if (!ctx) return fail_null("ctx");
  return check_errors(ctx->impl, (cudaStream_t)stream, "check");
}

int gsls_scan_plan(int32_t length, int32_t reverse, int32_t max_ops, int32_t* ops, int32_t* layer_off,
                   int32_t* out_slot, int32_t* n_ops, int32_t* n_layers) {
  if (length < 1) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "empty scan");
    return GSLS_ERR_ARG;
  }
  ScanPlan p = make_scan_plan(length, reverse != 0);
  if (n_ops) *n_ops = (int32_t)p.ops.size();
  if (n_layers) *n_layers = p.layers;
  if ((int)p.ops.size() > max_ops) return GSLS_OK;  // sizes only
  for (size_t i = 0; i < p.ops.size(); ++i) {
    ops[3 * i] = p.ops[i].dst;
    ops[3 * i + 1] = p.ops[i].earlier;
    ops[3 * i + 2] = p.ops[i].later;
  }
  for (int l = 0; l <= p.layers; ++l) layer_off[l] = p.layer_off[l];
  for (int i = 0; i < length; ++i) out_slot[i] = p.out[i];
  return GSLS_OK;
}

int gsls_lqr_solve(gsls_ctx* ctx, const gsls_qp_t* qp, int32_t generation, double* dx, double* du, float* K,
                   double* k, float* P, double* p, void* stream) {
  if (!ctx || !dx || (!du && ctx->impl->dims.N > 0)) return fail_null("ctx/dx/du");
  int rc = check_qp(qp, ctx->impl->dims);
  if (rc) return rc;
  return lqr_solve(ctx->impl, qp, generation, dx, du, K, k, P, p, (cudaStream_t)stream);
}

int gsls_lqr_solve_cached(gsls_ctx* ctx, const gsls_qp_t* qp, const double* q, const double* r, const double* qN,
                          int32_t generation, double* dx, double* du, double* k, double* p, void* stream) {
  if (!ctx || !dx || !qN || (!du && ctx->impl->dims.N > 0)) return fail_null("ctx/dx/du/qN");
  int rc = check_qp(qp, ctx->impl->dims);
  if (rc) return rc;
  return lqr_solve_cached(ctx->impl, qp, q, r, qN, generation, dx, du, k, p, (cudaStream_t)stream);
}

int gsls_admm_solve_qp(gsls_ctx* ctx, const gsls_qp_t* qp, const gsls_admm_settings_t* settings,
                       gsls_admm_state_t* state, gsls_admm_stats_t* stats, double* dx, double* du, void* stream) {
  if (!ctx || !settings || !state || !stats || !dx || (!du && ctx->impl->dims.N > 0)) return fail_null("argument");
  int rc = check_qp(qp, ctx->impl->dims);
  if (rc) return rc;
  return admm_solve(ctx->impl, qp, settings, state, stats, dx, du, (cudaStream_t)stream);
}

int gsls_admm_build_cache(gsls_ctx* ctx, const gsls_qp_t* qp, const double* rho, void* stream) {
  if (!ctx || !rho) return fail_null("argument");
  int rc = check_qp(qp, ctx->impl->dims);
  if (rc) return rc;
  return admm_build(ctx->impl, qp, rho, (cudaStream_t)stream);
}

int gsls_ctx_export_solution(gsls_ctx* ctx, float* K, double* k, float* P, double* p, void* stream) {
  if (!ctx) return fail_null("ctx");
  return ctx_export(ctx->impl, K, k, P, p, (cudaStream_t)stream);
}

int gsls_sls_ncell(int32_t N) { return N * (N + 1) / 2; }

int gsls_sls_set_columns(gsls_ctx* ctx, int32_t j0, int32_t j1) {
  if (!ctx) return fail_null("ctx");
  return sls_set_columns(ctx->impl, j0, j1);
}

int gsls_sls_plan(int32_t N, int32_t cvf, int32_t max_ops, int32_t* ops, int32_t* layer_off, int32_t* out_cell,
                  int32_t* n_ops, int32_t* n_layers, int32_t* n_slots) {
  if (N < 1 || !n_ops || !n_layers || !n_slots) return fail_null("argument");
  return sls_plan(N, cvf, max_ops, ops, layer_off, out_cell, n_ops, n_layers, n_slots);
}

int gsls_sls_assemble(gsls_ctx* ctx, const gsls_qp_t* qp, const double* tau, const double* tau_term,
                      const float* Qbar, const float* Rbar, const float* QbarN, int32_t weights_per_instance,
                      void* stream) {
  if (!ctx || !qp || !Qbar || !Rbar || !QbarN) return fail_null("argument");
  const gsls_dims_t& d = ctx->impl->dims;
  if (!qp->C || !qp->D || (d.nf > 0 && !qp->CN)) {
    if (d.nc > 0 || d.nf > 0) return fail_null("C/D/CN");
  }
  return sls_assemble(ctx->impl, qp, tau, tau_term, Qbar, Rbar, QbarN, weights_per_instance, (cudaStream_t)stream);
}

int gsls_sls_set_costs(gsls_ctx* ctx, const double* Qx, const double* Qu, const double* Qux, void* stream) {
  if (!ctx || !Qx || !Qu || !Qux) return fail_null("argument");
  return sls_set_costs(ctx->impl, Qx, Qu, Qux, (cudaStream_t)stream);
}

int gsls_sls_export_costs(gsls_ctx* ctx, double* Qx, double* Qu, double* Qux, void* stream) {
  if (!ctx) return fail_null("ctx");
  return sls_export_costs(ctx->impl, Qx, Qu, Qux, (cudaStream_t)stream);
}

int gsls_sls_synthesize(gsls_ctx* ctx, const gsls_qp_t* qp, const float* E, void* stream) {
  if (!ctx || !qp || !qp->A || !qp->B || !E) return fail_null("argument");
  return sls_synthesize(ctx->impl, qp, E, (cudaStream_t)stream, true);
}

int gsls_sls_tighten(gsls_ctx* ctx, const gsls_qp_t* qp, double* h, double* hf, void* stream) {
  if (!ctx || !qp || !h) return fail_null("argument");
  return sls_tighten(ctx->impl, qp, h, hf, (cudaStream_t)stream);
}

int gsls_sls_duals(gsls_ctx* ctx, const gsls_qp_t* qp, const double* lam, double eps, int32_t use_response,
                   int32_t reuse_rownorms, double* tau, double* tau_term, double* beta, double* beta_term,
                   void* stream) {
  if (!ctx || !qp || !lam || !tau || !tau_term) return fail_null("argument");
  return sls_duals(ctx->impl, qp, lam, eps, use_response, reuse_rownorms, tau, tau_term, beta, beta_term,
                   (cudaStream_t)stream);
}

int gsls_sls_import_response(gsls_ctx* ctx, const float* phix, const float* phiu, void* stream) {
  if (!ctx || !phix || !phiu) return fail_null("argument");
  return sls_import(ctx->impl, phix, phiu, (cudaStream_t)stream);
}

int gsls_sls_export(gsls_ctx* ctx, float* phix, float* phiu, float* gains, void* stream) {
  if (!ctx) return fail_null("ctx");
  return sls_export(ctx->impl, phix, phiu, gains, (cudaStream_t)stream);
}

int gsls_sls_cost(gsls_ctx* ctx, const double* Qbar, const double* Rbar, const double* QbarN, double* cost,
                  void* stream) {
  if (!ctx || !Qbar || !Rbar || !QbarN || !cost) return fail_null("argument");
  return sls_cost(ctx->impl, Qbar, Rbar, QbarN, cost, (cudaStream_t)stream);
}

int gsls_linearize(gsls_ctx* ctx, const gsls_linearize_args_t* args, const gsls_qp_t* out, float* E, void* stream) {
  if (!ctx || !args || !out || !args->params || !args->x || !args->u || !args->Qw || !args->Rw || !args->QNw ||
      !args->xref || !args->uref)
    return fail_null("argument");
  gsls_qp_t o = *out;
  int rc = linearize(ctx->impl, args, &o, E, (cudaStream_t)stream);
  if (rc == GSLS_ERR_ARG) set_error(rc, -1, 0, 0, 0, "model / dimension mismatch");
  if (rc == GSLS_ERR_TOO_LARGE) set_error(rc, -1, 0, 0, 0, "model too large");
  return rc;
}

int gsls_traj_eval(gsls_ctx* ctx, const gsls_linearize_args_t* args, double* out, void* stream) {
  if (!ctx || !args || !out || !args->params || !args->x || !args->u || !args->Qw || !args->Rw || !args->QNw ||
      !args->xref || !args->uref)
    return fail_null("argument");
  return traj_eval(ctx->impl, args, out, (cudaStream_t)stream);
}

int gsls_apply_tightening(gsls_ctx* ctx, double* f, double* fN, const double* h, const double* hf, void* stream) {
  if (!ctx || (!f && ctx->impl->dims.nc > 0) || (!h && ctx->impl->dims.nc > 0)) return fail_null("argument");
  return apply_tightening(ctx->impl, f, fN, h, hf, (cudaStream_t)stream);
}

int gsls_rti_apply(gsls_ctx* ctx, const double* prev_x, const double* prev_u, const double* dx, const double* du,
                   double* plan_x, double* plan_u, double* warm_x, double* warm_u, double* u0, const double* Qw,
                   const double* Rw, const double* QNw, const double* xref, const double* uref, double* cost,
                   void* stream) {
  if (!ctx || !prev_x || !prev_u || !dx || !du || !plan_x || !plan_u || !warm_x || !warm_u || !u0)
    return fail_null("argument");
  if (cost && (!Qw || !Rw || !QNw || !xref || !uref)) return fail_null("cost weights");
  return rti_apply(ctx->impl, prev_x, prev_u, dx, du, plan_x, plan_u, warm_x, warm_u, u0, Qw, Rw, QNw, xref, uref,
                   cost, (cudaStream_t)stream);
}

int gsls_rollout(gsls_ctx* ctx, const gsls_rollout_args_t* args, const gsls_rollout_out_t* out, void* stream) {
  if (!ctx || !args || !out || !args->params || !args->x || !args->u || !args->E || !args->E_pinv ||
      !args->disturbances)
    return fail_null("argument");
  if (!out->x || !out->u || !out->w || !out->tube_margin || !out->max_w_norm || !out->flags ||
      (ctx->impl->dims.nc > 0 && !out->stage_g) || (ctx->impl->dims.nf > 0 && !out->terminal_g))
    return fail_null("output");
  const int rc = rollout(ctx->impl, args, out, (cudaStream_t)stream);
  if (rc == GSLS_ERR_ARG) set_error(rc, -1, 0, 0, 0, "model / dimension mismatch");
  if (rc == GSLS_ERR_TOO_LARGE) set_error(rc, -1, 0, 0, 0, "rollout too large");
  return rc;
}

int gsls_rti_step(gsls_ctx* ctx, const gsls_rti_step_args_t* args, void* stream) {
  if (!ctx || !args) return fail_null("argument");
  const gsls_linearize_args_t& l = args->lin;
  if (!l.params || !l.x || !l.u || !l.Qw || !l.Rw || !l.QNw || !l.xref || !l.uref) return fail_null("lin argument");
  if (!args->qp || !args->dx || !args->du || !args->plan_x || !args->plan_u || !args->warm_x || !args->warm_u ||
      !args->u0)
    return fail_null("step output");
  const gsls_admm_state_t& a = args->state;
  const gsls_admm_stats_t& t = args->stats;
  if (!a.z || !a.lam || !a.y || !a.rho || !a.r_primal || !a.r_dual || !a.generation || !a.iteration)
    return fail_null("ADMM state");
  if (!t.iterations || !t.converged || !t.rho_changes || !t.cache_builds) return fail_null("ADMM stats");
  const gsls_admm_settings_t& st = args->admm;
  if (st.sigma < 2 || st.max_iter < 1 || !(st.rho0 > 0) || !(st.tol_primal > 0) || !(st.tol_dual > 0)) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "invalid ADMM settings");
    return GSLS_ERR_ARG;
  }
  int rc = rti_step(ctx->impl, args, (cudaStream_t)stream);
  if (rc == GSLS_ERR_ARG) set_error(rc, -1, 0, 0, 0, "model / dimension mismatch");
  return rc;
}

int gsls_rti_pack_results(gsls_ctx* ctx, const double* u0, const gsls_admm_stats_t* stats, const double* cost,
                          double* rec, void* stream) {
  if (!ctx || !u0 || !stats || !stats->iterations || !stats->converged || !stats->rho_changes || !rec)
    return fail_null("argument");
  return rti_pack_results(ctx->impl, u0, stats, cost, rec, (cudaStream_t)stream);
}

}  // extern "C"
