// Replay of the recorded scans (the per-ADMM-iteration hot path) and the
// persistent ADMM loop around it.
//
// One CTA owns one instance and keeps every scan vector in shared memory;
// the recorded matrices (Ups, Pr, Psi, Cl per CVF op, A_later per COT op) are
// streamed column-major from HBM/L2 by "warp tasks" (8 rows x 4 k-groups per
// warp, one 32-byte sector per k), so every load is a full sector.
//
// Reference map:
//   linear terms     augment_linear / _linear_element_terms (admm.py:113-121, lqr.py:338-342)
//   CVF replay       cvf_replay_kernel / _cvf_affine_core (lqr.py:242-262)
//   feedforward      _feedforward (lqr.py:345-346)
//   COT replay       _cot_elements + cot_replay_kernel (lqr.py:349-356, :281-285)
//   assembly         _assemble (lqr.py:359-363)
//   ADMM step        constraint_values / project_and_ascend / residuals /
//                    update_rho (admm.py:91-97, :130-150, :184-199)
#include <algorithm>
#include <cmath>
#include <vector>

#include "ctx.h"
#include "prof.h"

namespace gsls {

int check_errors(Ctx* c, cudaStream_t st, const char* what);
void set_error(int code, int inst, int where, int aux, int label, const char* msg);

enum { MODE_LQR = 0, MODE_ADMM = 1 };
enum { ST_DONE = 0, ST_REBUILD = 1 };

struct ReplayArgs {
  DevLqr L;
  gsls_qp_t qp;
  const double *q_in, *r_in, *qN_in;  // linear terms (LQR mode)
  int mode;
  gsls_admm_settings_t set;
  gsls_admm_state_t state;
  gsls_admm_stats_t stats;
  int32_t* status;
  double *dx, *du, *k_out, *p_out;
  const int* list;
  double* gscratch;
  long long scratch_floats;
  int max_layer;  // max ops in any scan layer (t1/t2 sizing)
};

// Replay vectors (all float64).
struct VecLayout {
  int pv, bv, cb, t1, t2, z, lam, y, rhat, om, kf, du, red, total;
};

__host__ __device__ inline VecLayout vec_layout(int n, int m, int N, int mtot, int s_cvf, int s_cot, int max_layer) {
  VecLayout v;
  int o = 0;
  auto take = [&](int sz) { int r = o; o += (sz + 1) & ~1; return r; };
  v.pv = take(s_cvf * n);
  v.bv = take(s_cvf * n);
  v.cb = take(s_cot * n);
  v.t1 = take(max_layer * n);
  v.t2 = take(max_layer * n);
  v.z = take(mtot);
  v.lam = take(mtot);
  v.y = take(mtot);
  v.rhat = take(N * m);
  v.om = take(N * m);  // also the feedforward inner vector
  v.kf = take(N * m);
  v.du = take(N * m);
  v.red = take(64);
  v.total = o;
  return v;
}

size_t replay_smem_floats(const Ctx* c) {
  const int ml = std::max(1, std::max(c->cvf_max_layer, c->cot_max_layer));
  return (size_t)vec_layout(c->dims.nx, c->dims.nu, c->dims.N, c->mtot, c->cvf.nslots, c->cot.nslots, ml).total;
}

// y[row] = add[row] + sgn * sum_k Mcm[k*ldg + row] x[k] for one 32-row block
// (fp32 recorded matrix, fp64 vectors and accumulation).  Lane (rq, g): rows
// 32rb + 4rq .. +3 as one 16-byte load, k = g, g+4, ...; 8 lanes of equal g
// read one full 128-byte line per k.  Padding rows (< ldg) are zero.
__device__ inline void warp_cm_matvec(const float* __restrict__ Mcm, int ldg, int n, int rb, const double* x,
                                      const double* add, double sgn, double* y) {
  const int lane = threadIdx.x & 31;
  const int rq = lane & 7, g = lane >> 3;
  const int row0 = rb * 32 + 4 * rq;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (row0 < ldg) {
    const float* p = Mcm + row0;
#pragma unroll 8
    for (int k = g; k < n; k += 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p + (size_t)k * ldg));
      const double xk = x[k];
      a0 = fma((double)v.x, xk, a0);
      a1 = fma((double)v.y, xk, a1);
      a2 = fma((double)v.z, xk, a2);
      a3 = fma((double)v.w, xk, a3);
    }
  }
#pragma unroll
  for (int o = 8; o <= 16; o <<= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    a3 += __shfl_xor_sync(0xffffffffu, a3, o);
  }
  if (g == 0) {
    const double av[4] = {a0, a1, a2, a3};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = row0 + r;
      if (row < n) y[row] = add[row] + sgn * av[r];
    }
  }
}

__device__ inline double block_max_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) r = fmax(r, red[i]);
  __syncthreads();
  return r;
}

__device__ inline void write_last(const DevLqr& L, int inst, const double* kf, const double* pv, int tid, int nthr) {
  const int n = L.n, m = L.m, N = L.N;
  for (int e = tid; e < N * m; e += nthr) L.last_k[(size_t)inst * N * m + e] = kf[e];
  for (int e = tid; e < (N + 1) * n; e += nthr) {
    const int k = e / n, i = e - k * n;
    L.last_p[(size_t)inst * (N + 1) * n + e] = pv[L.cvf_out[k] * n + i];
  }
}

__global__ void __launch_bounds__(512, 1) k_replay(ReplayArgs a) {
  const DevLqr& L = a.L;
  const int inst = a.list ? a.list[blockIdx.y] : (int)blockIdx.y;
  const int n = L.n, m = L.m, c = L.c, nf = L.nf, N = L.N, ldg = L.ldg, mtot = L.mtot;
  const size_t MS = (size_t)n * ldg;
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, nwarp = nthr >> 5;
  const VecLayout V = vec_layout(n, m, N, mtot, L.cvf_nslots, L.cot_nslots, a.max_layer);
  extern __shared__ double smem[];
  double* vs = a.gscratch ? a.gscratch + (size_t)inst * a.scratch_floats : smem;
  double *pv = vs + V.pv, *bv = vs + V.bv, *cb = vs + V.cb, *t1 = vs + V.t1, *t2 = vs + V.t2;
  double *z = vs + V.z, *lam = vs + V.lam, *y = vs + V.y;
  double *rhat = vs + V.rhat, *om = vs + V.om, *kf = vs + V.kf, *du = vs + V.du, *red = vs + V.red;
  __shared__ int s_flag;  // 0 continue, 1 done, 2 rebuild

  const size_t sN = (size_t)inst * N;
  const float* Cq = a.qp.C + sN * c * n;
  const float* Dq = a.qp.D + sN * c * m;
  const float* Bq = a.qp.B + sN * n * m;
  const double* bq = a.qp.b + sN * n;
  const float* CNq = a.qp.CN + (size_t)inst * nf * n;
  const double* q_lin = (a.q_in ? a.q_in : a.qp.q) + sN * n;
  const double* r_lin = (a.r_in ? a.r_in : a.qp.r) + sN * m;
  const double* qN_lin = (a.qN_in ? a.qN_in : a.qp.qN) + (size_t)inst * n;
  const float* Rinv = L.Rinv + sN * m * m;
  const float* Shat = L.Shat + sN * m * n;
  const float* Gam = L.Gamma + sN * m * m;
  const float* Kg = L.K + sN * m * n;
  const double* cvec = L.cvec + sN * n;
  const double* v0 = L.v0 + (size_t)inst * n;
  const float* cvf_rec = L.cvf_rec + (size_t)inst * L.cvf_nops * 4 * MS;
  const float* cot_rec = L.cot_rec + (size_t)inst * L.cot_nops * MS;
  const double* dx0 = a.qp.dx0 + (size_t)inst * n;
  // dx_k lives in the COT outputs (k >= 1) or dx0
  auto dxp = [&](int k) -> const double* { return k == 0 ? dx0 : cb + (size_t)L.cot_out[k - 1] * n; };

  const bool admm = a.mode == MODE_ADMM;
  double rho = 0.0;
  int it = 0;
  if (admm) {
    rho = a.state.rho[inst];
    it = a.stats.iterations[inst];
    const double* zg = a.state.z + (size_t)inst * mtot;
    const double* lg = a.state.lam + (size_t)inst * mtot;
    const double* yg = a.state.y + (size_t)inst * mtot;
    for (int e = tid; e < mtot; e += nthr) { z[e] = zg[e]; lam[e] = lg[e]; y[e] = yg[e]; }
    __syncthreads();
  }
  const int RB = (n + 31) >> 5;  // 32-row blocks per matvec

  for (;;) {
    // ---- linear terms q + rho C'(y - z), r + rho D'(y - z) and CVF leaves --------
    for (int e = tid; e < N * m; e += nthr) {
      const int k = e / m, i = e - k * m;
      double s = 0.0;
      if (admm)
        for (int r = 0; r < c; ++r) s = fma((double)Dq[((size_t)k * c + r) * m + i], y[k * c + r] - z[k * c + r], s);
      rhat[e] = admm ? r_lin[e] + rho * s : r_lin[e];
    }
    for (int e = tid; e < N * n; e += nthr) {
      const int k = e / n, i = e - k * n;
      double s = 0.0;
      if (admm)
        for (int r = 0; r < c; ++r) s = fma((double)Cq[((size_t)k * c + r) * n + i], y[k * c + r] - z[k * c + r], s);
      pv[e] = admm ? q_lin[e] + rho * s : q_lin[e];
    }
    for (int i = tid; i < n; i += nthr) {
      double s = 0.0;
      if (admm)
        for (int f = 0; f < nf; ++f) s = fma((double)CNq[f * n + i], y[N * c + f] - z[N * c + f], s);
      pv[N * n + i] = admm ? qN_lin[i] + rho * s : qN_lin[i];
      bv[N * n + i] = 0.0;
    }
    __syncthreads();
    for (int e = tid; e < N * m; e += nthr) {
      const int k = e / m, i = e - k * m;
      double s = 0.0;
      for (int t = 0; t < m; ++t) s = fma((double)Rinv[((size_t)k * m + i) * m + t], rhat[k * m + t], s);
      om[e] = s;
    }
    __syncthreads();
    for (int e = tid; e < N * n; e += nthr) {
      const int k = e / n, i = e - k * n;
      double s1 = 0.0, s2 = 0.0;
      for (int l = 0; l < m; ++l) {
        const double o = om[k * m + l];
        s1 = fma((double)Shat[((size_t)k * m + l) * n + i], o, s1);
        s2 = fma((double)Bq[((size_t)k * n + i) * m + l], o, s2);
      }
      pv[e] = pv[e] - s1;
      bv[e] = bq[e] - s2;
    }
    __syncthreads();

    // ---- CVF replay (reverse tree): 2 rounds per layer -----------------------
    for (int lay = 0; lay < L.cvf_layers; ++lay) {
      const int o0 = L.cvf_loff[lay], no = L.cvf_loff[lay + 1] - o0;
      if (no == 0) continue;
      const int tasks = no * 2 * RB;
      for (int t = warp; t < tasks; t += nwarp) {
        const int oi = t / (2 * RB), rem = t - oi * 2 * RB, which = rem / RB, rb = rem - which * RB;
        const int4 op = L.cvf_ops[o0 + oi];
        const float* rec = cvf_rec + (size_t)(o0 + oi) * 4 * MS;
        if (which == 0)  // t1 = p_later + Pr b_earlier
          warp_cm_matvec(rec + 1 * MS, ldg, n, rb, bv + op.y * n, pv + op.z * n, 1.0, t1 + oi * n);
        else             // t2 = b_earlier - Cl p_later
          warp_cm_matvec(rec + 3 * MS, ldg, n, rb, pv + op.z * n, bv + op.y * n, -1.0, t2 + oi * n);
      }
      __syncthreads();
      for (int t = warp; t < tasks; t += nwarp) {
        const int oi = t / (2 * RB), rem = t - oi * 2 * RB, which = rem / RB, rb = rem - which * RB;
        const int4 op = L.cvf_ops[o0 + oi];
        const float* rec = cvf_rec + (size_t)(o0 + oi) * 4 * MS;
        if (which == 0)  // p = Ups t1 + p_earlier
          warp_cm_matvec(rec + 0 * MS, ldg, n, rb, t1 + oi * n, pv + op.y * n, 1.0, pv + op.x * n);
        else             // b = Psi t2 + b_later
          warp_cm_matvec(rec + 2 * MS, ldg, n, rb, t2 + oi * n, bv + op.z * n, 1.0, bv + op.x * n);
      }
      __syncthreads();
    }

    // ---- feedforward k = -Gamma (B'(p+ + P+ b) + r) and COT leaves ---------------
    for (int e = tid; e < N * m; e += nthr) {
      const int k = e / m, l = e - k * m;
      const double* pn = pv + (size_t)L.cvf_out[k + 1] * n;
      const double* cvk = cvec + (size_t)k * n;
      double s = 0.0;
      for (int i = 0; i < n; ++i) s = fma((double)Bq[((size_t)k * n + i) * m + l], pn[i] + cvk[i], s);
      om[e] = s + rhat[e];
    }
    __syncthreads();
    for (int e = tid; e < N * m; e += nthr) {
      const int k = e / m, l = e - k * m;
      double s = 0.0;
      for (int t = 0; t < m; ++t) s = fma((double)Gam[((size_t)k * m + l) * m + t], om[k * m + t], s);
      kf[e] = -s;
    }
    __syncthreads();
    for (int e = tid; e < N * n; e += nthr) {
      const int k = e / n, i = e - k * n;
      double s = 0.0;
      for (int l = 0; l < m; ++l) s = fma((double)Bq[((size_t)k * n + i) * m + l], kf[k * m + l], s);
      const double bb = s + bq[e];
      cb[e] = (k == 0) ? v0[i] + bb : bb;
    }
    __syncthreads();

    // ---- COT replay (forward tree): 1 round per layer -------------------------
    for (int lay = 0; lay < L.cot_layers; ++lay) {
      const int o0 = L.cot_loff[lay], no = L.cot_loff[lay + 1] - o0;
      if (no == 0) continue;
      const int tasks = no * RB;
      for (int t = warp; t < tasks; t += nwarp) {
        const int oi = t / RB, rb = t - oi * RB;
        const int4 op = L.cot_ops[o0 + oi];
        warp_cm_matvec(cot_rec + (size_t)(o0 + oi) * MS, ldg, n, rb, cb + op.y * n, cb + op.z * n, 1.0,
                       cb + op.x * n);
      }
      __syncthreads();
    }

    // ---- du = K dx + k ------------------------------------------------------------
    for (int e = tid; e < N * m; e += nthr) {
      const int k = e / m, l = e - k * m;
      const double* xk = dxp(k);
      double s = 0.0;
      for (int i = 0; i < n; ++i) s = fma((double)Kg[((size_t)k * m + l) * n + i], xk[i], s);
      du[e] = s + kf[e];
    }
    __syncthreads();

    if (!admm) {
      write_last(L, inst, kf, pv, tid, nthr);
      double* gdx = a.dx + (size_t)inst * (N + 1) * n;
      double* gdu = a.du + (size_t)inst * N * m;
      for (int e = tid; e < (N + 1) * n; e += nthr) gdx[e] = dxp(e / n)[e % n];
      for (int e = tid; e < N * m; e += nthr) gdu[e] = du[e];
      if (a.k_out)
        for (int e = tid; e < N * m; e += nthr) a.k_out[(size_t)inst * N * m + e] = kf[e];
      if (a.p_out)
        for (int e = tid; e < (N + 1) * n; e += nthr) {
          const int k = e / n, i = e - k * n;
          a.p_out[(size_t)inst * (N + 1) * n + e] = pv[L.cvf_out[k] * n + i];
        }
      return;
    }

    // ---- ADMM: G = C dx + D du, projection, dual ascent, residuals ---------------
    const double* fst = a.qp.f + sN * c;
    const double* fN = a.qp.fN + (size_t)inst * nf;
    double rp = 0.0, rdz = 0.0;
    for (int e = tid; e < mtot; e += nthr) {
      double g, fe;
      if (e < N * c) {
        const int k = e / c, r = e - k * c;
        const float* Cr = Cq + ((size_t)k * c + r) * n;
        const float* Dr = Dq + ((size_t)k * c + r) * m;
        const double* xk = dxp(k);
        double s1 = 0.0, s2 = 0.0;
        for (int i = 0; i < n; ++i) s1 = fma((double)Cr[i], xk[i], s1);
        for (int l = 0; l < m; ++l) s2 = fma((double)Dr[l], du[k * m + l], s2);
        g = s1 + s2;
        fe = fst[e];
      } else {
        const int f = e - N * c;
        const double* xN = dxp(N);
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = fma((double)CNq[f * n + i], xN[i], s);
        g = s;
        fe = fN[f];
      }
      const double zo = z[e];
      const double zn = fmin(g + y[e], fe);
      const double ln = lam[e] + rho * (g - zn);
      lam[e] = ln;
      y[e] = ln / rho;
      z[e] = zn;
      rp = fmax(rp, fabs(g - zn));
      rdz = fmax(rdz, fabs(zn - zo));
    }
    rp = block_max_d(rp, red);
    rdz = block_max_d(rdz, red + 32);
    if (tid == 0) {
      ++it;
      a.state.iteration[inst] += 1;
      const double r_p = rp;
      const double r_d = rho * rdz;
      a.state.r_primal[inst] = r_p;
      a.state.r_dual[inst] = r_d;
      int flag = 0;
      if (r_p <= a.set.tol_primal && r_d <= a.set.tol_dual) {
        a.stats.converged[inst] = 1;
        flag = 1;
      } else {
        bool changed = false;
        if (it % a.set.sigma == 0) {
          const double ratio = sqrt(fmax(r_p, 1e-30) / fmax(r_d, 1e-30));
          const double prop = fmin(fmax(rho * ratio, a.set.rho_min), a.set.rho_max);
          if (prop > 5.0 * rho || prop < rho / 5.0) {
            a.state.rho[inst] = prop;
            a.state.generation[inst] += 1;
            a.stats.rho_changes[inst] += 1;
            changed = true;
          }
        }
        if (it >= a.set.max_iter) flag = 1;
        else if (changed) flag = 2;
      }
      a.stats.iterations[inst] = it;
      s_flag = flag;
    }
    __syncthreads();
    const int flag = s_flag;
    if (flag == 0) continue;
    const double rho_new = a.state.rho[inst];
    if (rho_new != rho)  // committed change rescales y = lam / rho (admm.py:149)
      for (int e = tid; e < mtot; e += nthr) y[e] = lam[e] / rho_new;
    __syncthreads();
    double* zg = a.state.z + (size_t)inst * mtot;
    double* lg = a.state.lam + (size_t)inst * mtot;
    double* yg = a.state.y + (size_t)inst * mtot;
    for (int e = tid; e < mtot; e += nthr) { zg[e] = z[e]; lg[e] = lam[e]; yg[e] = y[e]; }
    if (flag == 1) {
      write_last(L, inst, kf, pv, tid, nthr);
      double* gdx = a.dx + (size_t)inst * (N + 1) * n;
      double* gdu = a.du + (size_t)inst * N * m;
      for (int e = tid; e < (N + 1) * n; e += nthr) gdx[e] = dxp(e / n)[e % n];
      for (int e = tid; e < N * m; e += nthr) gdu[e] = du[e];
    }
    if (tid == 0) a.status[inst] = (flag == 2) ? ST_REBUILD : ST_DONE;
    return;
  }
}

// ---------------------------------------------------------------------------
// host side

static int launch_replay(Ctx* c, ReplayArgs& a, int count, cudaStream_t st) {
  if (count == 0) return GSLS_OK;
  a.L = c->dev;
  a.max_layer = std::max(1, std::max(c->cvf_max_layer, c->cot_max_layer));
  size_t sb = 0;
  if (c->d_scratch) {
    a.gscratch = c->d_scratch;
    a.scratch_floats = (long long)c->scratch_floats;
  } else {
    a.gscratch = nullptr;
    a.scratch_floats = 0;
    sb = c->scratch_floats * sizeof(double);
    if (sb > 48 * 1024)
      GSLS_CUDA_CHECK(cudaFuncSetAttribute((const void*)k_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
  }
  ProfScope ps(P_REPLAY, st, (double)count);
  k_replay<<<dim3(1, count), 512, sb, st>>>(a);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

__global__ void k_export_P(DevLqr L, float* P, const int* list) {
  const int inst = list ? list[blockIdx.y] : (int)blockIdx.y;
  const int pos = blockIdx.x, n = L.n, ldg = L.ldg;
  const float* src = L.Ps + ((size_t)inst * L.cvf_nslots + L.cvf_out[pos]) * n * ldg;
  float* dst = P + ((size_t)inst * (L.N + 1) + pos) * n * n;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) dst[e] = src[(e / n) * ldg + e % n];
}

int lqr_solve(Ctx* c, const gsls_qp_t* qp, int generation, double* dx, double* du, float* K, double* k, float* P,
              double* p, cudaStream_t st) {
  const int B = c->dims.batch;
  int rc = build_cache(c, qp, nullptr, nullptr, B, st);
  if (rc) return rc;
  rc = check_errors(c, st, "lqr build");
  if (rc) { c->cache_valid = false; return rc; }
  c->cache_valid = true;
  c->generation = generation;
  ReplayArgs a{};
  a.qp = *qp;
  a.mode = MODE_LQR;
  a.dx = dx; a.du = du; a.k_out = k; a.p_out = p;
  rc = launch_replay(c, a, B, st);
  if (rc) return rc;
  const int n = c->dims.nx, m = c->dims.nu, N = c->dims.N;
  if (K && N > 0)
    GSLS_CUDA_CHECK(cudaMemcpyAsync(K, c->dev.K, sizeof(float) * (size_t)B * N * m * n, cudaMemcpyDeviceToDevice, st));
  if (P) {
    k_export_P<<<dim3(N + 1, B), 256, 0, st>>>(c->dev, P, nullptr);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  return GSLS_OK;
}

int lqr_solve_cached(Ctx* c, const gsls_qp_t* qp, const double* q, const double* r, const double* qN,
                     int generation, double* dx, double* du, double* k, double* p, cudaStream_t st) {
  if (!c->cache_valid || generation != c->generation) {
    set_error(GSLS_ERR_CACHE_INVALIDATED, -1, 0, 0, 0, "cache invalidated");
    return GSLS_ERR_CACHE_INVALIDATED;
  }
  ReplayArgs a{};
  a.qp = *qp;
  a.q_in = q; a.r_in = r; a.qN_in = qN;
  a.mode = MODE_LQR;
  a.dx = dx; a.du = du; a.k_out = k; a.p_out = p;
  return launch_replay(c, a, c->dims.batch, st);
}

// Exports K, P (current cache) and k, p (last replay) for every instance.
int ctx_export(Ctx* c, float* K, double* k, float* P, double* p, cudaStream_t st) {
  const int B = c->dims.batch, n = c->dims.nx, m = c->dims.nu, N = c->dims.N;
  if (K && N > 0)
    GSLS_CUDA_CHECK(cudaMemcpyAsync(K, c->dev.K, sizeof(float) * (size_t)B * N * m * n, cudaMemcpyDeviceToDevice, st));
  if (k && N > 0)
    GSLS_CUDA_CHECK(cudaMemcpyAsync(k, c->dev.last_k, sizeof(double) * (size_t)B * N * m, cudaMemcpyDeviceToDevice, st));
  if (p)
    GSLS_CUDA_CHECK(cudaMemcpyAsync(p, c->dev.last_p, sizeof(double) * (size_t)B * (N + 1) * n, cudaMemcpyDeviceToDevice, st));
  if (P) {
    k_export_P<<<dim3(N + 1, B), 256, 0, st>>>(c->dev, P, nullptr);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  return GSLS_OK;
}

int admm_solve(Ctx* c, const gsls_qp_t* qp, const gsls_admm_settings_t* s, gsls_admm_state_t* state,
               gsls_admm_stats_t* stats, double* dx, double* du, cudaStream_t st) {
  const int B = c->dims.batch;
  if (s->sigma < 2 || s->max_iter < 1 || !(s->rho0 > 0) || !(s->tol_primal > 0) || !(s->tol_dual > 0)) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "invalid ADMM settings");
    return GSLS_ERR_ARG;
  }
  GSLS_CUDA_CHECK(cudaMemsetAsync(stats->iterations, 0, sizeof(int32_t) * B, st));
  GSLS_CUDA_CHECK(cudaMemsetAsync(stats->converged, 0, sizeof(int32_t) * B, st));
  GSLS_CUDA_CHECK(cudaMemsetAsync(stats->rho_changes, 0, sizeof(int32_t) * B, st));
  std::vector<int> builds(B, 0), list(B), status(B);
  for (int i = 0; i < B; ++i) list[i] = i;
  c->cache_valid = false;  // the ADMM rebuilds the cache at augmented costs
  while (!list.empty()) {
    const int cnt = (int)list.size();
    GSLS_CUDA_CHECK(cudaMemcpyAsync(c->d_inst_list, list.data(), sizeof(int) * cnt, cudaMemcpyHostToDevice, st));
    int rc = build_cache(c, qp, state->rho, c->d_inst_list, cnt, st);
    if (rc) return rc;
    for (int i : list) builds[i]++;
    ReplayArgs a{};
    a.qp = *qp;
    a.mode = MODE_ADMM;
    a.set = *s;
    a.state = *state;
    a.stats = *stats;
    a.status = c->d_status;
    a.dx = dx; a.du = du;
    a.list = c->d_inst_list;
    rc = launch_replay(c, a, cnt, st);
    if (rc) return rc;
    rc = check_errors(c, st, "admm");  // synchronizes
    if (rc) return rc;
    GSLS_CUDA_CHECK(cudaMemcpyAsync(status.data(), c->d_status, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
    GSLS_CUDA_CHECK(cudaStreamSynchronize(st));
    std::vector<int> next;
    for (int i : list)
      if (status[i] == ST_REBUILD) next.push_back(i);
    list.swap(next);
  }
  GSLS_CUDA_CHECK(cudaMemcpyAsync(stats->cache_builds, builds.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice, st));
  GSLS_CUDA_CHECK(cudaStreamSynchronize(st));
  return GSLS_OK;
}

}  // namespace gsls
