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
void set_error(int code, int inst, int where, int aux, int label, const char* msg);
int lqr_solve(Ctx* c, const gsls_qp_t* qp, int generation, double* dx, double* du, float* K, double* k, float* P,
              double* p, cudaStream_t st);
int lqr_solve_cached(Ctx* c, const gsls_qp_t* qp, const double* q, const double* r, const double* qN,
                     int generation, double* dx, double* du, double* k, double* p, cudaStream_t st);
int admm_solve(Ctx* c, const gsls_qp_t* qp, const gsls_admm_settings_t* s, gsls_admm_state_t* state,
               gsls_admm_stats_t* stats, double* dx, double* du, cudaStream_t st);
int ctx_export(Ctx* c, float* K, double* k, float* P, double* p, cudaStream_t st);
int sls_assemble(Ctx* c, const gsls_qp_t* qp, const double* tau, const double* tau_term, const float* Qbar,
                 const float* Rbar, const float* QbarN, int weights_per_instance, cudaStream_t st);
int sls_set_costs(Ctx* c, const float* Qx, const float* Qu, const float* Qux, cudaStream_t st);
int sls_synthesize(Ctx* c, const gsls_qp_t* qp, const float* E, cudaStream_t st, bool check);
int sls_tighten(Ctx* c, double* h, double* hf, cudaStream_t st);
int sls_duals(Ctx* c, const double* lam_s, const double* lam_t, double eps, int use_response, double* tau,
              double* tau_term, double* beta, double* beta_term, cudaStream_t st);
int sls_export(Ctx* c, float* phix, float* phiu, float* gains, cudaStream_t st);
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

int gsls_ctx_export_solution(gsls_ctx* ctx, float* K, double* k, float* P, double* p, void* stream) {
  if (!ctx) return fail_null("ctx");
  return ctx_export(ctx->impl, K, k, P, p, (cudaStream_t)stream);
}

int gsls_sls_ncell(int32_t N) { return N * (N + 1) / 2; }

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

int gsls_sls_set_costs(gsls_ctx* ctx, const float* Qx, const float* Qu, const float* Qux, void* stream) {
  if (!ctx || !Qx || !Qu || !Qux) return fail_null("argument");
  return sls_set_costs(ctx->impl, Qx, Qu, Qux, (cudaStream_t)stream);
}

int gsls_sls_synthesize(gsls_ctx* ctx, const gsls_qp_t* qp, const float* E, void* stream) {
  if (!ctx || !qp || !qp->A || !qp->B || !E) return fail_null("argument");
  return sls_synthesize(ctx->impl, qp, E, (cudaStream_t)stream, true);
}

int gsls_sls_tighten(gsls_ctx* ctx, double* h, double* hf, void* stream) {
  if (!ctx || !h) return fail_null("argument");
  return sls_tighten(ctx->impl, h, hf, (cudaStream_t)stream);
}

int gsls_sls_duals(gsls_ctx* ctx, const double* lam_stage, const double* lam_term, double eps, int32_t use_response,
                   double* tau, double* tau_term, double* beta, double* beta_term, void* stream) {
  if (!ctx || !lam_stage || !tau || !tau_term) return fail_null("argument");
  return sls_duals(ctx->impl, lam_stage, lam_term, eps, use_response, tau, tau_term, beta, beta_term,
                   (cudaStream_t)stream);
}

int gsls_sls_export(gsls_ctx* ctx, float* phix, float* phiu, float* gains, void* stream) {
  if (!ctx) return fail_null("ctx");
  return sls_export(ctx->impl, phix, phiu, gains, (cudaStream_t)stream);
}

}  // extern "C"
