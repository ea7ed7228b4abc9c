// One receding-horizon MPC step for every instance of a context, as one C call:
// the metric's unit of work (sls.rti_robust_step, sls.py:500-525; nominal
// sqp.rti_step, sqp.py:272-302) behind the C ABI, so a C caller reaches it without
// the Python engine.  The order is the reference's:
//   linearize at (prev_x, prev_u) with the measured state      sqp.py:285-292 / sls.py:509
//   compute_duals' tau -> assemble_costs -> synthesize -> tighten sls.py:510-516
//   f -= h (the tightened re-linearization)                    sqp.py:136/:140
//   admm.solve_qp (cold or warm ADMM state)                    sqp.py:293 / sls.py:517
//   compute_duals for the next step                            sls.py:519-521
//   plan / warm start / u0                                     sqp.py:294-301
// The ADMM's first factorization depends on A, B, Q, R, S, C, D and rho only, not on
// the tightened offsets, so it is built on the context's side stream while the SLS
// chain runs on the caller's stream (fork/join by events: also capturable into a
// CUDA graph).  gsls_rti_pack_results packs the per-instance record the ranks of a
// multi-GPU batch exchange (dist.py RESULT_FIELDS).
#include <algorithm>
#include <cmath>

#include "ctx.h"

namespace gsls {

int linearize(Ctx* c, const gsls_linearize_args_t* in, gsls_qp_t* out_qp, float* E, cudaStream_t st);
int sls_assemble(Ctx* c, const gsls_qp_t* qp, const double* tau, const double* tau_term, const float* Qbar,
                 const float* Rbar, const float* QbarN, int weights_per_instance, cudaStream_t st);
int sls_synthesize(Ctx* c, const gsls_qp_t* qp, const float* E, cudaStream_t st, bool check);
int sls_tighten(Ctx* c, const gsls_qp_t* qp, double* h, double* hf, cudaStream_t st);
int sls_duals(Ctx* c, const gsls_qp_t* qp, const double* lam, double eps, int use_response, int reuse_rownorms,
              double* tau, double* tau_term, double* beta, double* beta_term, cudaStream_t st);
int apply_tightening(Ctx* c, double* f, double* fN, const double* h, const double* hf, cudaStream_t st);
int admm_build(Ctx* c, const gsls_qp_t* qp, const double* rho, cudaStream_t st);
int admm_solve(Ctx* c, const gsls_qp_t* qp, const gsls_admm_settings_t* s, gsls_admm_state_t* state,
               gsls_admm_stats_t* stats, double* dx, double* du, cudaStream_t st);
int rti_apply(Ctx* c, const double* px, const double* pu, const double* dx, const double* du, double* plan_x,
              double* plan_u, double* warm_x, double* warm_u, double* u0, const double* Qw, const double* Rw,
              const double* QNw, const double* xref, const double* uref, double* cost, cudaStream_t st);
void set_error(int code, int inst, int where, int aux, int label, const char* msg);

// Cold ADMM state (admm.py:160-166): z = lam = y = 0, rho = rho0, counters 0,
// residuals +inf.
__global__ void k_admm_reset(gsls_admm_state_t s, int B, int mtot, double rho0) {
  const long long tot = (long long)B * mtot;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    s.z[e] = 0.0;
    s.lam[e] = 0.0;
    s.y[e] = 0.0;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B; i += gridDim.x * blockDim.x) {
    s.rho[i] = rho0;
    s.generation[i] = 0;
    s.iteration[i] = 0;
    s.r_primal[i] = INFINITY;
    s.r_dual[i] = INFINITY;
  }
}

// (B, nu + 4) float64: u0, ADMM iterations, converged, rho changes, cost (dist.py).
__global__ void k_pack_results(const double* u0, const gsls_admm_stats_t st, const double* cost, int B, int nu,
                               double* rec) {
  const int w = nu + 4;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < B * w; e += gridDim.x * blockDim.x) {
    const int i = e / w, f = e - i * w;
    double v;
    if (f < nu) v = u0[(size_t)i * nu + f];
    else if (f == nu) v = st.iterations[i];
    else if (f == nu + 1) v = st.converged[i];
    else if (f == nu + 2) v = st.rho_changes[i];
    else v = cost ? cost[i] : 0.0;
    rec[e] = v;
  }
}

int rti_step(Ctx* c, const gsls_rti_step_args_t* a, cudaStream_t st) {
  const gsls_dims_t& d = c->dims;
  const int B = d.batch, mtot = d.N * d.nc + d.nf;
  gsls_qp_t qp = *a->qp;
  const bool robust = a->robust != 0;
  if (robust && (!a->E || !a->Qbar || !a->Rbar || !a->QbarN || !a->h || !a->hf || !a->tau || !a->tau_term ||
                 !a->beta || !a->beta_term)) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "robust step: null SLS buffer");
    return GSLS_ERR_ARG;
  }
  int rc = linearize(c, &a->lin, &qp, a->E, st);
  if (rc) return rc;
  if (a->E_in && a->E)
    GSLS_CUDA_CHECK(cudaMemcpyAsync(a->E, a->E_in, sizeof(float) * (size_t)B * d.N * d.nx * d.nx,
                                    cudaMemcpyDeviceToDevice, st));
  gsls_admm_state_t state = a->state;
  gsls_admm_stats_t stats = a->stats;
  if (!a->warm_admm) {
    const int blocks = std::min(1024, std::max(1, (B * mtot + 255) / 256));
    k_admm_reset<<<blocks, 256, 0, st>>>(state, B, mtot, a->admm.rho0);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  bool forked = false;
  if (robust) {
    if (!c->step_side) {
      GSLS_CUDA_CHECK(cudaStreamCreateWithFlags(&c->step_side, cudaStreamNonBlocking));
      GSLS_CUDA_CHECK(cudaEventCreateWithFlags(&c->step_fork, cudaEventDisableTiming));
      GSLS_CUDA_CHECK(cudaEventCreateWithFlags(&c->step_join, cudaEventDisableTiming));
    }
    if (!a->no_overlap) {  // first factorization beside the SLS chain
      GSLS_CUDA_CHECK(cudaEventRecord(c->step_fork, st));
      GSLS_CUDA_CHECK(cudaStreamWaitEvent(c->step_side, c->step_fork, 0));
      if ((rc = admm_build(c, &qp, state.rho, c->step_side))) return rc;
      GSLS_CUDA_CHECK(cudaEventRecord(c->step_join, c->step_side));
      forked = true;
    }
    if ((rc = sls_assemble(c, &qp, a->use_tau ? a->tau : nullptr, a->use_tau ? a->tau_term : nullptr, a->Qbar,
                           a->Rbar, a->QbarN, 0, st)))
      return rc;
    if ((rc = sls_synthesize(c, &qp, a->E, st, true))) return rc;
    if ((rc = sls_tighten(c, &qp, a->h, a->hf, st))) return rc;
    if ((rc = apply_tightening(c, const_cast<double*>(qp.f), const_cast<double*>(qp.fN), a->h, a->hf, st))) return rc;
    if (forked) GSLS_CUDA_CHECK(cudaStreamWaitEvent(st, c->step_join, 0));
  }
  if ((rc = admm_solve(c, &qp, &a->admm, &state, &stats, a->dx, a->du, st))) return rc;
  if (robust && (rc = sls_duals(c, &qp, state.lam, a->eps, 1, 1, a->tau, a->tau_term, a->beta, a->beta_term, st)))
    return rc;
  return rti_apply(c, a->lin.x, a->lin.u, a->dx, a->du, a->plan_x, a->plan_u, a->warm_x, a->warm_u, a->u0,
                   a->lin.Qw, a->lin.Rw, a->lin.QNw, a->lin.xref, a->lin.uref, a->cost, st);
}

int rti_pack_results(Ctx* c, const double* u0, const gsls_admm_stats_t* stats, const double* cost, double* rec,
                     cudaStream_t st) {
  const int B = c->dims.batch, nu = c->dims.nu;
  const int blocks = (B * (nu + 4) + 255) / 256;
  k_pack_results<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(u0, *stats, cost, B, nu, rec);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

}  // namespace gsls
