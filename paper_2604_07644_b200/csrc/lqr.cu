// LQR factorization ("cache build"): CVF leaves, CVF combine tree, gains,
// COT combine tree.  Matrix work only — every vector (p, b, k, dx, du) is
// produced by the replay kernel (admm.cu), so the full solve and the cached
// solve run the same vector code and agree bitwise (lqr.py:419-454 contract).
//
// Reference map:
//   k_leaf_init    _build_static / init_elements + ADMM augmentation
//                  (lqr.py:297-335, admm.py:100-110)
//   k_cvf_combine  _cvf_matrix_core + aux record (lqr.py:226-254)
//   k_gains        Gamma, K, Abar, COT leaves (lqr.py:398-404, :349-356)
//   k_cot_combine  cot_kernel + aux record (lqr.py:273-278)
#include <cstdio>
#include <cstring>
#include <mutex>

#include "ctx.h"
#include "prof.h"
#include "smallmat.cuh"
#include "gj.cuh"
#include "lowrank.cuh"

namespace gsls {

// ---------------------------------------------------------------------------
// error plumbing shared by all translation units

static std::mutex g_err_mu;
static gsls_error_t g_err{};

void set_last_error(const char* msg, const char* file, int line) {
  std::lock_guard<std::mutex> g(g_err_mu);
  g_err.code = GSLS_ERR_CUDA;
  g_err.instance = -1;
  snprintf(g_err.message, sizeof(g_err.message), "%s (%s:%d)", msg, file, line);
}

void set_error(int code, int inst, int where, int aux, int label, const char* msg) {
  std::lock_guard<std::mutex> g(g_err_mu);
  g_err.code = code;
  g_err.instance = inst;
  g_err.where = where;
  g_err.aux = aux;
  g_err.aux2 = label;
  snprintf(g_err.message, sizeof(g_err.message), "%s", msg);
}

int get_last_error(gsls_error_t* out) {
  std::lock_guard<std::mutex> g(g_err_mu);
  *out = g_err;
  return g_err.code;
}

void* dev_alloc(Ctx* c, size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  cudaMemset(p, 0, bytes);
  c->allocs.push_back(p);
  c->bytes += (int64_t)bytes;
  return p;
}

static const char* label_text(int label) {
  switch (label) {
    case GSLS_LABEL_R: return "R";
    case GSLS_LABEL_R_BPB: return "R + B'PB";
    case GSLS_LABEL_QU: return "Qu";
    case GSLS_LABEL_QU_BPB: return "Qu + B'PB";
    default: return "matrix";
  }
}

// Copies per-instance error slots to the host; raises the first one found.
int check_errors(Ctx* c, cudaStream_t st, const char* what) {
  const int B = c->dims.batch;
  std::vector<ErrSlot> h(B);
  GSLS_CUDA_CHECK(cudaMemcpyAsync(h.data(), c->dev.err, sizeof(ErrSlot) * B, cudaMemcpyDeviceToHost, st));
  GSLS_CUDA_CHECK(cudaStreamSynchronize(st));
  // A factored combine met an indefinite P (lowrank.cuh): switch that tree to dense
  // combines, clear those records and tell the caller to re-run the scan.
  bool lr[2] = {false, false};
  for (int i = 0; i < B; ++i) {
    if (h[i].key == 0) continue;
    const ErrInfo e = err_unpack(h[i].key);
    if (e.code != GSLS_ERR_LOWRANK) continue;
    lr[e.label == 1] = true;
    h[i].key = 0;
  }
  if (lr[0] || lr[1]) {
    if (lr[0]) {  // the LQR cache of those instances is not valid: every caller rebuilds
      c->lqr_dense = true;
      c->dev.cvf_ops = c->cvf_ops_v[1];
      c->dev.cvf_leaf = c->cvf_leaf_v[1];
      c->cache_valid = false;
      c->admm_prebuilt = false;
    }
    if (lr[1]) sls_use_dense(c);
    GSLS_CUDA_CHECK(cudaMemcpyAsync(c->dev.err, h.data(), sizeof(ErrSlot) * B, cudaMemcpyHostToDevice, st));
    GSLS_CUDA_CHECK(cudaStreamSynchronize(st));
    return GSLS_ERR_LOWRANK;
  }
  for (int i = 0; i < B; ++i) {
    if (h[i].key == 0) continue;
    const ErrInfo e = err_unpack(h[i].key);
    char msg[256];
    if (e.code == GSLS_ERR_SINGULAR_STAGE) {
      if (e.aux >= 0)
        snprintf(msg, sizeof msg, "singular %s block at (k=%d, j=%d)", label_text(e.label), e.where, e.aux);
      else
        snprintf(msg, sizeof msg, "singular %s at stage %d", label_text(e.label), e.where);
    } else if (e.code == GSLS_ERR_ILL_CONDITIONED) {
      snprintf(msg, sizeof msg, "ill-conditioned combine");
    } else if (e.code == GSLS_ERR_NONFINITE) {
      snprintf(msg, sizeof msg, "non-finite %s at stage %d",
               e.label == GSLS_LABEL_NONFINITE_CON ? "constraints" : "dynamics", e.where);
    } else {
      snprintf(msg, sizeof msg, "%s failed", what);
    }
    set_error(e.code, i, e.where, e.aux, e.label, msg);
    cudaMemsetAsync(c->dev.err, 0, sizeof(ErrSlot) * B, st);
    return e.code;
  }
  return GSLS_OK;
}

// ---------------------------------------------------------------------------
// kernels

__device__ inline int inst_of(const int* list) { return list ? list[blockIdx.y] : (int)blockIdx.y; }

// One bulk L2 prefetch of a contiguous operand read after the kernel's first phase.
__device__ inline void lqr_prefetch_l2(const void* p, size_t bytes) {
  const unsigned long long a = (unsigned long long)p & ~15ull;
  const unsigned long long e = ((unsigned long long)p + bytes + 15ull) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}

// CVF leaves (Eq. 29) with penalty augmentation rho (0 for a plain LQR).
// Computed in float64: the Schur complement Q^ - S^' R^-1 S^ cancels O(rho)
// terms; only the result is rounded to the float32 scan storage.
__global__ void __launch_bounds__(256) k_leaf_init(DevLqr L, gsls_qp_t qp, const double* rho_arr,
                                                   const int* list) {
  if (L.build_count && (int)blockIdx.y >= *L.build_count) return;
  const int inst = inst_of(list);
  const int k = blockIdx.x;
  const int n = L.n, m = L.m, c = L.c, nf = L.nf, N = L.N, ldg = L.ldg;
  const double rho = rho_arr ? rho_arr[inst] : 0.0;
  const size_t MS = (size_t)n * ldg;
  const size_t sbase = ((size_t)inst * L.cvf_nslots + k) * MS;
  float* Pd = L.Ps + sbase;
  float* Ad = L.As + sbase;
  float* ATd = L.ATs + sbase;
  float* Cd = L.Cs + sbase;
  if (k == N) {
    const float* QN = qp.QN + (size_t)inst * n * n;
    const float* CN = qp.CN + (size_t)inst * nf * n;
    for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) {
      const int i = L.fd_ldg.div(e), j = e - i * ldg;
      double v = 0.0;
      if (j < n) {
        double s = 0.0;
        for (int f = 0; f < nf; ++f) s = fma((double)CN[f * n + i], (double)CN[f * n + j], s);
        v = (double)QN[i * n + j] + rho * s;
      }
      Pd[e] = (float)v;
      Ad[e] = 0.f;
      ATd[e] = 0.f;
      Cd[e] = 0.f;
    }
    return;
  }
  extern __shared__ double smd[];
  double* Cst = smd;                 // c x n
  double* Dst = Cst + c * n;         // c x m
  const int ldb = m | 1;             // odd row stride: rows of B read across lanes hit distinct banks
  double* Bst = Dst + c * m;         // n x ldb
  double* Sh = Bst + n * ldb;        // m x n
  double* Rh = Sh + m * n;           // m x m
  double* Ri = Rh + m * m;           // m x m
  double* RS = Ri + m * m;           // m x n
  double* BR = RS + m * n;           // n x m
  double* wk = BR + n * m;           // spd work
  const size_t st = (size_t)inst * N + k;
  if (threadIdx.x == 0) {  // Q_k and A_k: read once per element by the P / A loop after the inverse
    lqr_prefetch_l2(qp.Q + st * n * n, (size_t)n * n * sizeof(float));
    lqr_prefetch_l2(qp.A + st * n * n, (size_t)n * n * sizeof(float));
  }
  const float* Cg = qp.C + st * c * n;
  const float* Dg = qp.D + st * c * m;
  const float* Bg = qp.B + st * n * m;
  for (int e = threadIdx.x; e < c * n; e += blockDim.x) Cst[e] = Cg[e];
  for (int e = threadIdx.x; e < c * m; e += blockDim.x) Dst[e] = Dg[e];
  for (int e = threadIdx.x; e < n * m; e += blockDim.x) {
    const int i = L.fd_m.div(e);
    Bst[i * ldb + (e - i * m)] = Bg[e];
  }
  __syncthreads();
  const float* Rg = qp.R + st * m * m;
  const float* Sg = qp.S ? qp.S + st * m * n : nullptr;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = L.fd_m.div(e), j = e - i * m;
    double s = 0.0;
    for (int r = 0; r < c; ++r) s = fma(Dst[r * m + i], Dst[r * m + j], s);
    Rh[e] = (double)Rg[e] + rho * s;
  }
  __syncthreads();
  // warp 0 inverts R-hat while warps 1.. form S-hat (independent of the inverse)
  if (threadIdx.x < 32) {
    if (warp_spd_inverse(Rh, m, Ri, m, wk) && threadIdx.x == 0)
      raise_err(L.err + inst, GSLS_ERR_SINGULAR_STAGE, k, -1, GSLS_LABEL_R);
  }
  for (int e = (int)threadIdx.x - 32; e >= 0 && e < m * n; e += (int)blockDim.x - 32) {
    const int i = L.fd_n.div(e), j = e - i * n;
    double s = 0.0;
    for (int r = 0; r < c; ++r) s = fma(Dst[r * m + i], Cst[r * n + j], s);
    Sh[e] = (Sg ? (double)Sg[e] : 0.0) + rho * s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int l = L.fd_n.div(e), j = e - l * n;
    double s = 0.0;
    for (int t = 0; t < m; ++t) s = fma(Ri[l * m + t], Sh[t * n + j], s);
    RS[e] = s;
  }
  for (int e = threadIdx.x; e < n * m; e += blockDim.x) {
    const int i = L.fd_m.div(e), l = e - i * m;
    double s = 0.0;
    for (int t = 0; t < m; ++t) s = fma(Bst[i * ldb + t], Ri[t * m + l], s);
    BR[e] = s;
  }
  __syncthreads();
  const float* Qg = qp.Q + st * n * n;
  const float* Ag = qp.A + st * n * n;
  // C-hat = B R-hat^-1 B' is stored as the factor B L^-T (R-hat = L L', L^-1 left in
  // the inverse's work area) when the scan plan carries it factored (lowrank.cuh)
  const bool cfac = L.cvf_leaf && (L.cvf_leaf[k] & 8);
  const double* Linv = wk + kMaxM * (kMaxM + 1);
  // rows i and i + nh per thread: the column-j operands (C, RS, B rows of j) are loaded once
  // for both (the loop is bound by shared-memory wavefronts); every element keeps its chains
  const int nh = (n + 1) >> 1;
  for (int e = threadIdx.x; e < nh * ldg; e += blockDim.x) {
    const int i0 = L.fd_ldg.div(e), j = e - i0 * ldg;
    const bool two = i0 + nh < n;
    const int i1 = two ? i0 + nh : i0;
    double p0 = 0.0, a0 = 0.0, c0 = 0.0, p1 = 0.0, a1 = 0.0, c1 = 0.0;
    if (cfac && j < m) {
      double f0 = 0.0, f1 = 0.0;
      for (int b = 0; b <= j; ++b) {
        const double li = Linv[j * (kMaxM + 1) + b];
        f0 = fma(Bst[i0 * ldb + b], li, f0);
        f1 = fma(Bst[i1 * ldb + b], li, f1);
      }
      c0 = f0;
      c1 = f1;
    }
    if (j < n) {
      double s0 = 0.0, s1 = 0.0;
      for (int r = 0; r < c; ++r) {
        const double cj = Cst[r * n + j];
        s0 = fma(Cst[r * n + i0], cj, s0);
        s1 = fma(Cst[r * n + i1], cj, s1);
      }
      double sr0 = 0.0, br0 = 0.0, sr1 = 0.0, br1 = 0.0;
      for (int l = 0; l < m; ++l) {
        const double rs = RS[l * n + j];
        sr0 = fma(Sh[l * n + i0], rs, sr0);
        br0 = fma(Bst[i0 * ldb + l], rs, br0);
        sr1 = fma(Sh[l * n + i1], rs, sr1);
        br1 = fma(Bst[i1 * ldb + l], rs, br1);
      }
      p0 = ((double)Qg[i0 * n + j] + rho * s0) - sr0;
      a0 = (double)Ag[i0 * n + j] - br0;
      p1 = ((double)Qg[i1 * n + j] + rho * s1) - sr1;
      a1 = (double)Ag[i1 * n + j] - br1;
      if (!cfac) {  // dense C-hat = B R-hat^-1 B' (a factored leaf carries B L^-T instead)
        double bb0 = 0.0, bb1 = 0.0;
        for (int l = 0; l < m; ++l) {
          const double bj = Bst[j * ldb + l];
          bb0 = fma(BR[i0 * m + l], bj, bb0);
          bb1 = fma(BR[i1 * m + l], bj, bb1);
        }
        c0 = bb0;
        c1 = bb1;
      }
    }
    Pd[i0 * ldg + j] = (float)p0;
    Ad[i0 * ldg + j] = (float)a0;
    if (j < n) ATd[j * ldg + i0] = (float)a0;
    Cd[i0 * ldg + j] = (float)c0;
    if (two) {
      Pd[i1 * ldg + j] = (float)p1;
      Ad[i1 * ldg + j] = (float)a1;
      if (j < n) ATd[j * ldg + i1] = (float)a1;
      Cd[i1 * ldg + j] = (float)c1;
    }
  }
  double* Rhat = L.Rhat + st * m * m;
  float* Shat = L.Shat + st * m * n;
  float* Rinv = L.Rinv + st * m * m;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) { Rhat[e] = Rh[e]; Rinv[e] = (float)Ri[e]; }
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) Shat[e] = (float)Sh[e];
  double* Shd = L.Shat64 + st * m * n;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) Shd[e] = Sh[e];

  // fused leaf operator of the ADMM iteration (ctx.h): with X1 = rho Rinv D',
  // om0 = Rinv r:  pv = (q - Sh' om0) + (rho C' - Sh' X1) w,  bv = (b - B om0) - B X1 w.
  double* X1 = wk + 2 * kMaxM * (kMaxM + 1) + 8;  // m x c
  double* om0 = X1 + m * c;                        // m
  const double* rg = qp.r + st * m;
  for (int e = threadIdx.x; e < m * c + m; e += blockDim.x) {
    if (e < m * c) {
      const int l = L.fd_c.div(e), r = e - l * c;
      double s = 0.0;
      for (int t = 0; t < m; ++t) s = fma(Ri[l * m + t], Dst[r * m + t], s);
      X1[e] = rho * s;
    } else {
      const int l = e - m * c;
      double s = 0.0;
      for (int t = 0; t < m; ++t) s = fma(Ri[l * m + t], rg[t], s);
      om0[l] = s;
    }
  }
  __syncthreads();
  const int ld2n = L.ld2n, ldn = L.ldn, ldc = L.ldc;
  float* X23 = L.X23 + st * (size_t)c * ld2n;
  for (int e = threadIdx.x; e < c * ld2n; e += blockDim.x) {
    const int r = L.fd_ld2n.div(e), i = e - r * ld2n;
    double v = 0.0;
    if (i < n) {
      double s = 0.0;
      for (int l = 0; l < m; ++l) s = fma(Sh[l * n + i], X1[l * c + r], s);
      v = rho * Cst[r * n + i] - s;
    } else if (i < 2 * n) {
      const int ii = i - n;
      double s = 0.0;
      for (int l = 0; l < m; ++l) s = fma(Bst[ii * ldb + l], X1[l * c + r], s);
      v = -s;
    }
    X23[e] = (float)v;
  }
  const double* qg = qp.q + st * n;
  const double* bg = qp.b + st * n;
  double* pb0 = L.pb0 + st * 2 * n;
  for (int i = threadIdx.x; i < 2 * n; i += blockDim.x) {
    double s = 0.0;
    if (i < n) {
      for (int l = 0; l < m; ++l) s = fma(Sh[l * n + i], om0[l], s);
      pb0[i] = qg[i] - s;
    } else {
      for (int l = 0; l < m; ++l) s = fma(Bst[(i - n) * ldb + l], om0[l], s);
      pb0[i] = bg[i - n] - s;
    }
  }
  float* Bcm = L.Bcm + st * (size_t)m * ldn;
  for (int e = threadIdx.x; e < m * ldn; e += blockDim.x) {
    const int j = L.fd_ldn.div(e), i = e - j * ldn;
    Bcm[e] = (i < n) ? (float)Bst[i * ldb + j] : 0.f;
  }
  float* Dcm = L.ZD + st * (size_t)(n + m) * ldc + (size_t)n * ldc;  // D columns of [Z D]
  for (int e = threadIdx.x; e < m * ldc; e += blockDim.x) {
    const int j = L.fd_ldc.div(e), i = e - j * ldc;
    Dcm[e] = (i < c) ? (float)Dst[i * m + j] : 0.f;
  }
}

// Matrix half of the CVF combine (Eq. 28) for one op per CTA; optionally
// records the replay operators column-major: Ups, X = Ups Pr, Psi, -Y with
// Y = Psi Cl, so the cached replay p = Ups (p_r + Pr b_l) + p_l,
// b = Psi (b_l - Cl p_r) + b_r (lqr.py:242-246) becomes
// p = p_l + [Ups X] [p_r; b_l], b = b_r + [Psi -Y] [b_l; p_r]: two n x 2n
// column-major operators (consecutive in the record), one round per tree layer.  Shared with
// the SLS grid scan (no record).
//
// P and C are symmetric in exact arithmetic (value-function Hessians and
// controllability Gramians, lqr.py:236-238), so Pr and Cl serve as their own
// transposes; A is kept in both orientations (As, ATs) so every operand
// arrives by a plain cp.async copy.  With Minv = (I + Pr Cl)^-1, the products
// Minv Pr and Minv' Cl are symmetric, so X' = Minv Pr Al = V (the product P
// needs anyway) and Y' = Minv' Cl Ar' = Minv' W2.  Six n x lds smem buffers:
//   b0 Pr -> W2 | b1 Cl -> Minv -> V | b2 M1 -> Minv^T | b3 Al | b4 Ar^T | b5 W1 -> Psi^T
// GSLS_COMBINE_TRACE: clock64 at the phase points of one CTA mid-grid (diagnostics only).
__device__ long long* g_comb_trace = nullptr;

// Factored combine (lowrank.cuh) of one op: C_l = F F' with F the earlier slot's
// factor (rank re = op.w bits 8-15), C_r the later slot's factor (rank rl, bits
// 16-23) or dense (rl = 255); bit 3: the output C is stored as the factor
// [U, F_r].  Same outputs and record layout as the dense path below.  Six
// ldg x lds buffers:
//   b0 Pr -> Pm | b1 F -> Fh -> X' | b2 W -> V -> Fr' | b3 Al | b4 Ar' -> Psi' | sb S -> U' -> V' -> T
// Returns false (block-uniform) when S has a pivot below 0.5 (P_r indefinite).
template <int NP>
__device__ __forceinline__ bool cvf_combine_factored(const CombineArgs& a, const int4 op, int inst, float* sm,
                                                     float* rec, long long* trc) {
#define FTRACE(i) do { if (trc) trc[i] = clock64(); } while (0)
  const int n = a.n, ldg = ldg_of(n), lds = gj_lds(NP, n);
  const int re = (op.w >> 8) & 0xFF, rl = (op.w >> 16) & 0xFF;
  const int R = round_up(re, 4);
  const size_t MS = (size_t)n * ldg;
  const size_t BSL = (size_t)ldg * lds;
  float* b0 = sm;
  float* b1 = b0 + BSL;
  float* b2 = b1 + BSL;
  float* b3 = b2 + BSL;
  float* b4 = b3 + BSL;
  float* sb = b4 + BSL;
  const long long ib = (long long)inst * a.inst_stride;
  const size_t oe = (size_t)op.y * MS, ol = (size_t)op.z * MS, od = (size_t)op.x * MS;
  const bool need_a = !(op.w & 1);                // A (A^T unless bit 2) live
  const bool need_c = !(op.w & 2);                // C live
  const bool need_psi = need_a;                   // (a recorded op with bit 0 is never read: no b half)
  const bool need_u = need_psi || need_c;
  const bool out_factor = (op.w & 8) != 0;
  const float* Cr = a.Cs + ib + ol;
  float* Cd = a.Cs + ib + od;
  cta_load_async(b0, lds, a.Ps + ib + ol, n);  // Pr
  cta_load_async(b1, lds, a.Cs + ib + oe, n);  // F (columns >= re stored as zero)
  cp_async_commit();
  cta_load_async(b3, lds, a.As + ib + oe, n);  // Al
  if (need_u) cta_load_async(b4, lds, a.ATs + ib + ol, n);  // Ar^T
  else cta_load_async(b4, lds, a.Ps + ib + oe, n);          // Pl (the P epilogue's addend)
  cp_async_commit();
  cp_async_wait<1>();
  __syncthreads();
  FTRACE(8);
  gemm_tn_mn(n, R, n, b0, lds, b1, lds, EpiS{b2, lds, n});  // W = Pr F
  __syncthreads();
  gemm_tn_mn(R, R, n, b1, lds, b2, lds, EpiSId{sb, lds, R});  // S = I + F' W
  __syncthreads();
  FTRACE(9);
  if (!chol_stack(sb, b1, b2, lds, R, n)) return false;  // b1 = Fh, b2 = V
  cp_async_wait<0>();
  __syncthreads();
  FTRACE(10);
  if (need_u) {
    gemm_tn_mn(R, n, n, b1, lds, b4, lds, EpiS{sb, lds, R});  // U' = Fh' Ar^T
    __syncthreads();
    if (need_psi)  // Psi' = Ar^T - V U' (in place), record slot 2
      gemm_nn_mn(n, n, R, b2, lds, sb, lds, EpiSub{b4, b4, lds, n, rec ? rec + 2 * MS : nullptr, ldg});
    if (rec && need_psi)  // -Y' = -Fh U', record slot 3
      gemm_nn_mn(n, n, R, b1, lds, sb, lds, EpiG{rec + 3 * MS, nullptr, ldg, n, nullptr, nullptr, 0, -1.f});
    if (need_c) {
      if (out_factor) {  // [U | F_r], zero beyond (ranks are multiples of 4: float4 columns)
        const int q = ldg >> 2;
        for (int e = threadIdx.x; e < n * q; e += blockDim.x) {
          const int j = (e / n) << 2, i = e - (e / n) * n;  // consecutive threads: consecutive rows
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (j < re) v = make_float4(sb[j * lds + i], sb[(j + 1) * lds + i], sb[(j + 2) * lds + i], sb[(j + 3) * lds + i]);
          else if (j < re + rl) v = *reinterpret_cast<const float4*>(Cr + (size_t)i * ldg + j - re);
          *reinterpret_cast<float4*>(Cd + (size_t)i * ldg + j) = v;
        }
      } else {  // U U' + C_r (dense C_r; a factored C_r is added at the end)
        gemm_tn_mn(n, n, R, sb, lds, sb, lds, EpiG{Cd, rl == 255 ? Cr : nullptr, ldg, n, nullptr, nullptr, 0, 1.f});
      }
    }
    __syncthreads();
  }
  FTRACE(11);
  for (int e = threadIdx.x; e < R * ldg; e += blockDim.x) {  // V' -> sb
    const int k = e / ldg, i = e - k * ldg;
    sb[k * lds + i] = i < n ? b2[i * lds + k] : 0.f;
  }
  __syncthreads();
  gemm_tn_mn(n, n, R, sb, lds, sb, lds, EpiSub{b0, b0, lds, n, nullptr, 0});  // Pm = Pr - V V'
  __syncthreads();
  if (rec) {
    gemm_tn_mn(R, n, n, b2, lds, b3, lds, EpiS{sb, lds, R});  // T = V' Al
    __syncthreads();
    if (need_u) cta_load_async(b2, lds, a.Ps + ib + oe, n);  // Pl (V is dead)
    cp_async_commit();
    gemm_nn_mn(n, n, R, b1, lds, sb, lds, EpiSub{nullptr, b3, lds, n, rec, ldg});  // Ups' = Al - Fh T, slot 0
    __syncthreads();
  } else if (need_u) {
    cta_load_async(b2, lds, a.Ps + ib + oe, n);  // Pl (V is dead)
    cp_async_commit();
  }
  const float* plb = need_u ? b2 : b4;
  FTRACE(12);
  // X' = Pm Al (record slot 1), then P = Al' X' + Pl
  gemm_tn_mn(n, n, n, b0, lds, b3, lds, EpiG{rec ? rec + MS : nullptr, nullptr, ldg, n, nullptr, b1, lds, 1.f});
  cp_async_wait<0>();
  __syncthreads();
  gemm_tn_mn(n, n, n, b3, lds, b1, lds, EpiG{a.Ps + ib + od, nullptr, ldg, n, nullptr, nullptr, lds, 1.f, plb});
  if (need_a)  // A = Psi Al (+ A^T)
    gemm_tn_mn(n, n, n, b4, lds, b3, lds,
               EpiG{a.As + ib + od, nullptr, ldg, n, (op.w & 4) ? nullptr : a.ATs + ib + od, nullptr, 0, 1.f});
  if (need_c && !out_factor && rl != 255) {  // C += F_r F_r'
    __syncthreads();  // b2 may hold Pl, read by the P epilogue above
    const int RL = round_up(rl, 4);
    for (int e = threadIdx.x; e < RL * ldg; e += blockDim.x) {
      const int k = e / ldg, i = e - k * ldg;
      b2[k * lds + i] = i < n ? Cr[(size_t)i * ldg + k] : 0.f;
    }
    __syncthreads();
    gemm_tn_mn(n, n, RL, b2, lds, b2, lds, EpiG{Cd, Cd, ldg, n, nullptr, nullptr, 0, 1.f});
  }
  __syncthreads();
  FTRACE(13);
#undef FTRACE
  return true;
}

template <int NP>
__global__ void __launch_bounds__(NP == 64 ? 288 : 416, NP == 64 ? 2 : 1) k_cvf_combine(CombineArgs a) {
  long long* trc = (g_comb_trace && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == gridDim.y / 2) ? g_comb_trace : nullptr;
#define CTRACE(i) do { if (trc) trc[i] = clock64(); } while (0)
  CTRACE(0);
  if (a.count && (int)blockIdx.y >= *a.count) return;
  const int inst = inst_of(a.list);
  const int4 op = a.ops[blockIdx.x];
  const int n = a.n, ldg = ldg_of(n), lds = gj_lds(NP, n);  // >= lds_of(n): the inverse's column tiles fit a row
  const size_t MS = (size_t)n * ldg;
  const size_t BS = (size_t)n * lds;
  extern __shared__ float sm[];
  if (((op.w >> 8) & 0xFF) != 0xFF) {  // earlier C carried as a factor
    float* recf = a.rec ? a.rec + (long long)inst * a.rec_inst_stride + (size_t)(a.op_base + blockIdx.x) * 4 * MS
                        : nullptr;
    const bool ok = cvf_combine_factored<NP>(a, op, inst, sm, recf, trc);
    if (!ok && threadIdx.x == 0)
      raise_err(a.err ? a.err + inst : nullptr, GSLS_ERR_LOWRANK, a.op_base + blockIdx.x, -1, a.label);
    CTRACE(5);
    return;
  }
  float* b0 = sm;
  float* b1 = b0 + BS;
  float* b2 = b1 + BS;
  float* b3 = b2 + BS;
  float* b4 = b3 + BS;
  float* b5 = b4 + BS;
  float* gjbuf = b5 + BS;
  const long long ib = (long long)inst * a.inst_stride;
  const size_t oe = (size_t)op.y * MS, ol = (size_t)op.z * MS, od = (size_t)op.x * MS;
  float* rec = a.rec ? a.rec + (long long)inst * a.rec_inst_stride + (size_t)(a.op_base + blockIdx.x) * 4 * MS
                     : nullptr;

  // fin: the output's A, A^T and C are all dead (plan .w bit 0): only P is formed, so
  // Ar^T, W2, Psi, A and C are skipped (4 of 8 GEMMs).  A recorded op with bit 0 is one
  // whose result no later op reads (recorded readers always need A^T), so its b half
  // is never replayed either (partition_unread_last): only Ups and X are recorded.
  const bool fin = (op.w & 1);
  cta_load_async(b0, lds, a.Ps + ib + ol, n);   // Pr (= Pr^T)
  cta_load_async(b1, lds, a.Cs + ib + oe, n);   // Cl (= Cl^T)
  cp_async_commit();
  cta_load_async(b3, lds, a.As + ib + oe, n);   // Al
  if (!fin) cta_load_async(b4, lds, a.ATs + ib + ol, n);  // Ar^T
  cp_async_commit();
  cp_async_wait<1>();
  __syncthreads();
  CTRACE(1);
  gemm_tn(n, b0, b1, lds, EpiSmem{b2, lds, n, true});   // M1 = I + Pr Cl
  cp_async_wait<0>();
  __syncthreads();
  CTRACE(2);
  gemm_tn(n, b0, b3, lds, EpiSmem{b5, lds, n, false});  // W1 = Pr Al
  __syncthreads();
  // C dead (plan .w bit 1): W2 only feeds C (and the -Y record)
  const bool need_w2 = !fin && (rec != nullptr || !(op.w & 2));
  if (need_w2) gemm_tn(n, b1, b4, lds, EpiSmem{b0, lds, n, false});  // W2 = Cl Ar^T (over Pr)
  __syncthreads();
  CTRACE(3);
  // Minv = M1^{-1} -> b1 (row-major, over Cl), Minv^T -> b2 (over M1, read first)
  // work: b1 (Cl is dead); row threads on 4 x (NP/16) (row, column) tiles
  const bool ok = gj_inverse_lookahead44<NP>(b2, b1, b1, b2, lds, n, gjbuf, a.rel_tol);
  if (!ok && threadIdx.x == 0)
    raise_err(a.err ? a.err + inst : nullptr, GSLS_ERR_ILL_CONDITIONED, a.op_base + blockIdx.x);
  CTRACE(4);
  if (rec) {
    gemm_tn(n, b1, b3, lds, EpiGlobal{rec + 0 * MS, nullptr, ldg, n, nullptr});  // Ups^T = Minv^T Al
    if (!fin) gemm_tn(n, b1, b0, lds, EpiGlobalNeg{rec + 3 * MS, ldg, n});  // -Y^T = -Minv^T W2
    __syncthreads();
  }
  gemm_tn(n, b2, b5, lds, EpiSmem{b1, lds, n, false});  // V = Minv W1 = X^T (over Minv)
  __syncthreads();
  if (rec) cta_store(rec + 1 * MS, b1, lds, n);          // X record
  gemm_tn(n, b3, b1, lds, EpiGlobal{a.Ps + ib + od, a.Ps + ib + oe, ldg, n, nullptr});  // P = Al^T V + Pl
  if (fin) {
    CTRACE(5);
    return;
  }
  gemm_tn(n, b2, b4, lds, EpiSmem{b5, lds, n, false});  // Psi^T = Minv Ar^T (over W1)
  __syncthreads();
  if (rec) cta_store(rec + 2 * MS, b5, lds, n);          // Psi record
  gemm_tn(n, b5, b3, lds, EpiGlobal{a.As + ib + od, nullptr, ldg, n, (op.w & 4) ? nullptr : a.ATs + ib + od});  // A = Psi Al (+ A^T)
  if (!(op.w & 2)) gemm_tn(n, b5, b0, lds, EpiGlobal{a.Cs + ib + od, a.Cs + ib + ol, ldg, n, nullptr});  // C = Psi W2 + Cr
  __syncthreads();
  CTRACE(5);
#undef CTRACE
}

size_t combine_smem_bytes(int n) {
  const int NP = n <= 64 ? 64 : 80;
  const size_t dense = 6 * (size_t)n * gj_lds(NP, n) + gjl_scratch_words(NP);
  const size_t factored = 6 * (size_t)ldg_of(n) * gj_lds(NP, n);  // cvf_combine_factored
  return std::max(dense, factored) * sizeof(float);
}

int combine_threads(int n) {  // k_cvf_combine: 4*NP row threads + the inverse's panel warp, >= GEMM tiles
  if (n <= 64) return 288;
  return 416;
}

int matmul_threads(int n) {
  const int T = ldg_of(n) / 4;
  int t = ((T * T + 31) / 32) * 32;
  if (t < 128) t = 128;
  if (t > 512) t = 512;
  return t;
}


// Gains, closed loop and COT leaves per stage (lqr.py:398-404, :349-356), in float64.
__global__ void __launch_bounds__(256) k_gains(DevLqr L, gsls_qp_t qp, const double* rho_arr, const int* list) {
  if (L.build_count && (int)blockIdx.y >= *L.build_count) return;
  const int inst = inst_of(list);
  const int k = blockIdx.x;
  const int n = L.n, m = L.m, N = L.N, ldg = L.ldg, c = L.c;
  const size_t MS = (size_t)n * ldg;
  const double rho = rho_arr ? rho_arr[inst] : 0.0;
  extern __shared__ double smd[];
  double* Bst = smd;             // n x m
  double* BtP = Bst + n * m;     // m x n
  double* H = BtP + m * n;       // m x m
  double* Gm = H + m * m;        // m x n
  double* Ga = Gm + m * n;       // m x m
  double* Ks = Ga + m * m;       // m x n
  double* wk = Ks + m * n;
  const int ldd = m | 1;  // D's row stride (odd: the Z = C + D K loop reads D by column across lanes)
  // n x ldg floats, 16-byte aligned; holds P+ (16-byte async copies) until Abar replaces it
  float* Abar = reinterpret_cast<float*>(wk + ((2 * kMaxM * (kMaxM + 1) + 8 + L.c * ldd + m + 1) & ~1));
  const size_t st = (size_t)inst * N + k;
  const float* Pn = L.Ps + ((size_t)inst * L.cvf_nslots + L.cvf_out[k + 1]) * MS;
  const float* Bg = qp.B + st * n * m;
  if (threadIdx.x == 0) lqr_prefetch_l2(qp.A + st * n * n, (size_t)n * n * sizeof(float));  // read by G and A + B K
  float* Pns = Abar;
  for (int e = threadIdx.x; e < (n * ldg) >> 2; e += blockDim.x) cp_async16(Pns + 4 * e, Pn + 4 * e);
  cp_async_commit();
  for (int e = threadIdx.x; e < n * m; e += blockDim.x) Bst[e] = Bg[e];
  cp_async_wait<0>();
  __syncthreads();
  const int mh = (m + 1) >> 1;
  for (int e = threadIdx.x; e < mh * n; e += blockDim.x) {  // B' P+, rows l and l + mh (one P+ load for both)
    const int l = L.fd_n.div(e), j = e - l * n;
    const bool two = l + mh < m;
    const int l1 = two ? l + mh : l;
    double s0 = 0.0, s1 = 0.0;
    for (int i = 0; i < n; ++i) {
      const double pv = (double)Pns[i * ldg + j];
      s0 = fma(Bst[i * m + l], pv, s0);
      s1 = fma(Bst[i * m + l1], pv, s1);
    }
    BtP[l * n + j] = s0;
    if (two) BtP[l1 * n + j] = s1;
  }
  __syncthreads();
  const float* Ag = qp.A + st * n * n;
  const double* Rhat = L.Rhat + st * m * m;
  const double* Shat = L.Shat64 + st * m * n;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int l = L.fd_m.div(e), t = e - l * m;
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fma(BtP[l * n + j], Bst[j * m + t], s);
    H[e] = Rhat[e] + s;
  }
  __syncthreads();
  // warps 1.. form G = Shat + B' P+ A while warp 0 inverts H (independent)
  for (int e = (int)threadIdx.x - 32; e >= 0 && e < m * n; e += (int)blockDim.x - 32) {
    const int l = L.fd_n.div(e), j = e - l * n;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = fma(BtP[l * n + i], (double)Ag[i * n + j], s);
    Gm[e] = Shat[e] + s;
  }
  if (threadIdx.x < 32) {
    if (warp_spd_inverse(H, m, Ga, m, wk) && threadIdx.x == 0)
      raise_err(L.err + inst, GSLS_ERR_SINGULAR_STAGE, k, -1, GSLS_LABEL_R_BPB);
  }
  __syncthreads();
  float* Kg = L.K + st * m * n;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int l = L.fd_n.div(e), j = e - l * n;
    double s = 0.0;
    for (int t = 0; t < m; ++t) s = fma(Ga[l * m + t], Gm[t * n + j], s);
    Ks[e] = -s;
    Kg[e] = (float)(-s);
  }
  float* Gg = L.Gamma + st * m * m;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) Gg[e] = (float)Ga[e];
  const double* bg = qp.b + st * n;
  double* cv = L.cvec + st * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fma((double)Pn[i * ldg + j], bg[j], s);
    cv[i] = s;
  }
  __syncthreads();
  // closed loop Abar = A + B K -> COT leaf k (leaf 0 carries A = 0, lqr.py:354)
  float* Ad = L.cotA + ((size_t)inst * L.cot_nslots + k) * MS;
  float* ATd = L.cotAT + ((size_t)inst * L.cot_nslots + k) * MS;
  const int nh = (n + 1) >> 1;
  for (int e = threadIdx.x; e < nh * ldg; e += blockDim.x) {  // rows i and i + nh (one K load for both)
    const int i = L.fd_ldg.div(e), j = e - i * ldg;
    const bool two = i + nh < n;
    const int i1 = two ? i + nh : i;
    double v0 = 0.0, v1 = 0.0;
    if (j < n) {
      double s0 = 0.0, s1 = 0.0;
      for (int l = 0; l < m; ++l) {
        const double kv = Ks[l * n + j];
        s0 = fma(Bst[i * m + l], kv, s0);
        s1 = fma(Bst[i1 * m + l], kv, s1);
      }
      v0 = (double)Ag[i * n + j] + s0;
      v1 = (double)Ag[i1 * n + j] + s1;
    }
    Abar[i * ldg + j] = (float)v0;
    Ad[i * ldg + j] = (k == 0) ? 0.f : (float)v0;
    if (j < n) ATd[j * ldg + i] = (k == 0) ? 0.f : (float)v0;
    if (two) {
      Abar[i1 * ldg + j] = (float)v1;
      Ad[i1 * ldg + j] = (k == 0) ? 0.f : (float)v1;
      if (j < n) ATd[j * ldg + i1] = (k == 0) ? 0.f : (float)v1;
    }
  }
  // fused feedforward / constraint operators (ctx.h):
  //   kf = kk0 + X5 p+ + X4 w with X5 = -Gamma B', X4 = -rho Gamma D', kk0 = -Gamma (B' cvec + r)
  //   G  = Z dx + D kf with Z = C + D K
  {
    double* Dst = wk + 2 * kMaxM * (kMaxM + 1) + 8;  // c x ldd (Abar follows tk)
    double* tk = Dst + c * ldd;                       // m
    const float* Dg = qp.D + st * c * m;
    for (int e = threadIdx.x; e < c * m; e += blockDim.x) {
      const int r = L.fd_m.div(e);
      Dst[r * ldd + (e - r * m)] = Dg[e];
    }
    __syncthreads();
    const double* rg = qp.r + st * m;
    for (int l = threadIdx.x; l < m; l += blockDim.x) {
      double s = rg[l];
      for (int i = 0; i < n; ++i) s = fma(Bst[i * m + l], cv[i], s);
      tk[l] = s;
    }
    __syncthreads();
    const int ldm = L.ldm, ldc = L.ldc;
    float* X5 = L.XK + st * (size_t)(n + c) * ldm;  // [X5 X4]
    for (int e = threadIdx.x; e < n * ldm; e += blockDim.x) {
      const int i = L.fd_ldm.div(e), l = e - i * ldm;
      double s = 0.0;
      if (l < m)
        for (int t = 0; t < m; ++t) s = fma(Ga[l * m + t], Bst[i * m + t], s);
      X5[e] = (float)(-s);
    }
    float* X4 = X5 + (size_t)n * ldm;
    for (int e = threadIdx.x; e < c * ldm; e += blockDim.x) {
      const int r = L.fd_ldm.div(e), l = e - r * ldm;
      double s = 0.0;
      if (l < m)
        for (int t = 0; t < m; ++t) s = fma(Ga[l * m + t], Dst[r * ldd + t], s);
      X4[e] = (float)(-rho * s);
    }
    double* kk0 = L.kk0 + st * m;
    for (int l = threadIdx.x; l < m; l += blockDim.x) {
      double s = 0.0;
      for (int t = 0; t < m; ++t) s = fma(Ga[l * m + t], tk[t], s);
      kk0[l] = -s;
    }
    const float* Cg = qp.C + st * c * n;
    float* Zcm = L.ZD + st * (size_t)(n + m) * ldc;
    for (int e = threadIdx.x; e < n * ldc; e += blockDim.x) {
      const int i = L.fd_ldc.div(e), r = e - i * ldc;
      double v = 0.0;
      if (r < c) {
        double s = (double)Cg[r * n + i];
        for (int l = 0; l < m; ++l) s = fma(Dst[r * ldd + l], Ks[l * n + i], s);
        v = s;
      }
      Zcm[e] = (float)v;
    }
  }
  if (k == 0) {
    __syncthreads();
    const double* dx0 = qp.dx0 + (size_t)inst * n;
    double* v0 = L.v0 + (size_t)inst * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s = fma((double)Abar[i * ldg + j], dx0[j], s);
      v0[i] = s;
    }
  }
}

// COT combine: A = A_later A_earlier (+ transpose); records A_later column-major.
__global__ void __launch_bounds__(512) k_cot_combine(DevLqr L, const int4* ops, int op_base, const int* list) {
  if (L.build_count && (int)blockIdx.y >= *L.build_count) return;
  const int inst = inst_of(list);
  const int4 op = ops[blockIdx.x];
  const int n = L.n, ldg = L.ldg, lds = lds_of(n);
  const size_t MS = (size_t)n * ldg;
  extern __shared__ float sm[];
  float* Art = sm;
  float* Ae = Art + (size_t)n * lds;
  const size_t ib = (size_t)inst * L.cot_nslots * MS;
  cta_load_async(Art, lds, L.cotAT + ib + (size_t)op.z * MS, n);
  cta_load_async(Ae, lds, L.cotA + ib + (size_t)op.y * MS, n);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  float* rec = L.cot_rec + ((size_t)inst * L.cot_nops + op_base + blockIdx.x) * MS;
  cta_store(rec, Art, lds, n);
  gemm_tn(n, Art, Ae, lds, EpiGlobal{L.cotA + ib + (size_t)op.x * MS, nullptr, ldg, n, L.cotAT + ib + (size_t)op.x * MS});
}

// ---------------------------------------------------------------------------
// host driver

static size_t leaf_smem_bytes(int n, int m, int c) {  // B at row stride m | 1
  return (size_t)(c * n + c * m + n * (m | 1) + m * n + 2 * m * m + m * n + n * m + 2 * kMaxM * (kMaxM + 1) + 8 + m * c + m) *
         sizeof(double);
}
static size_t gains_smem_bytes(int n, int m, int c) {  // D at row stride m | 1
  return (size_t)(n * m + m * n + m * m + m * n + m * m + m * n + 2 * kMaxM * (kMaxM + 1) + 8 + c * (m | 1) + m + 1) *
             sizeof(double) +
         (size_t)n * ldg_of(n) * sizeof(float);
}

static int set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) {
    GSLS_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  }
  return GSLS_OK;
}

int launch_combine(const CombineArgs& a, int nops, int count, cudaStream_t st) {
  if (nops == 0 || count == 0) return GSLS_OK;
  size_t sb = combine_smem_bytes(a.n);
  if (getenv("GSLS_COMBINE_1CTA")) sb = 200 * 1024;  // diagnostics: one CTA per SM
  static long long* trace = nullptr;
  const bool tracing = getenv("GSLS_COMBINE_TRACE") != nullptr;
  if (tracing && !trace) {
    GSLS_CUDA_CHECK(cudaMalloc(&trace, 16 * sizeof(long long)));
    GSLS_CUDA_CHECK(cudaMemset(trace, 0, 16 * sizeof(long long)));
    GSLS_CUDA_CHECK(cudaMemcpyToSymbol(g_comb_trace, &trace, sizeof(trace)));
  }
  if (tracing) GSLS_CUDA_CHECK(cudaMemsetAsync(trace, 0, 16 * sizeof(long long), st));
  if (a.n <= 64) {
    int rc = set_smem((const void*)k_cvf_combine<64>, sb);
    if (rc) return rc;
    k_cvf_combine<64><<<dim3(nops, count), combine_threads(a.n), sb, st>>>(a);
  } else {
    int rc = set_smem((const void*)k_cvf_combine<80>, sb);
    if (rc) return rc;
    k_cvf_combine<80><<<dim3(nops, count), combine_threads(a.n), sb, st>>>(a);
  }
  GSLS_CUDA_CHECK(cudaGetLastError());
  if (tracing) {
    long long h[16];
    GSLS_CUDA_CHECK(cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st));
    GSLS_CUDA_CHECK(cudaStreamSynchronize(st));
    if (h[13] > 0)
      fprintf(stderr, "combine n=%d ops=%d count=%d rec=%d factored cycles: load %lld W,S %lld chol %lld U,Psi,Y,C %lld Pm(,T,Ups) %lld X,P,A %lld total %lld\n",
              a.n, nops, count, a.rec != nullptr, h[8] - h[0], h[9] - h[8], h[10] - h[9], h[11] - h[10], h[12] - h[11],
              h[13] - h[12], h[13] - h[0]);
    else
      fprintf(stderr, "combine n=%d ops=%d count=%d rec=%d cycles: load %lld gemm1 %lld gemm2+3 %lld gj %lld rest %lld total %lld\n",
              a.n, nops, count, a.rec != nullptr, h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4], h[5] - h[0]);
  }
  return GSLS_OK;
}

int build_cache(Ctx* c, const gsls_qp_t* qp, const double* d_rho, const int* d_list, int count, cudaStream_t st) {
  const gsls_dims_t& d = c->dims;
  DevLqr& L = c->dev;
  if (count == 0) return GSLS_OK;
  const int n = d.nx, N = d.N;
  // leaves
  {
    const size_t sb = leaf_smem_bytes(n, d.nu, d.nc);
    int rc = set_smem((const void*)k_leaf_init, sb);
    if (rc) return rc;
    ProfScope ps(P_LEAF, st, (double)(N + 1) * count);
    k_leaf_init<<<dim3(N + 1, count), 256, sb, st>>>(L, *qp, d_rho, d_list);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  // CVF tree
  const size_t MS = mat_elems(n);
  for (int l = 0; l < c->cvf.layers; ++l) {
    const int o0 = c->cvf_layer_off[l], o1 = c->cvf_layer_off[l + 1];
    CombineArgs a{n, L.cvf_ops + o0, o0, L.Ps, L.As, L.Cs, L.ATs, (long long)L.cvf_nslots * (long long)MS,
                  L.cvf_rec, (long long)L.cvf_nops * 4 * (long long)MS, d_list, L.err, 1e-10f, 0, L.build_count};
    if (o1 == o0) continue;
    ProfScope ps(P_CVF_LQR, st, (double)(o1 - o0) * count);
    int rc = launch_combine(a, o1 - o0, count, st);
    if (rc) return rc;
  }
  if (N == 0) return GSLS_OK;
  // gains / COT leaves
  {
    const size_t sb = gains_smem_bytes(n, d.nu, d.nc);
    int rc = set_smem((const void*)k_gains, sb);
    if (rc) return rc;
    ProfScope ps(P_GAINS, st, (double)N * count);
    k_gains<<<dim3(N, count), 256, sb, st>>>(L, *qp, d_rho, d_list);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  // COT tree
  {
    const size_t sb = 2 * (size_t)n * lds_of(n) * sizeof(float);
    int rc = set_smem((const void*)k_cot_combine, sb);
    if (rc) return rc;
    for (int l = 0; l < c->cot.layers; ++l) {
      const int o0 = c->cot_layer_off[l], o1 = c->cot_layer_off[l + 1];
      if (o1 == o0) continue;
      ProfScope ps(P_COT, st, (double)(o1 - o0) * count);
      k_cot_combine<<<dim3(o1 - o0, count), matmul_threads(n), sb, st>>>(L, L.cot_ops + o0, o0, d_list);
      GSLS_CUDA_CHECK(cudaGetLastError());
    }
  }
  return GSLS_OK;
}

// ---------------------------------------------------------------------------
// context

int factor_rmax(int n, int tree) {
  // Default: the SLS tree only.  The factored forms M1^-1 P_r = P_r - V V' and
  // Ups' = A_l - Fh V' A_l subtract nearly equal terms where P_r C_l is large, which the
  // ADMM penalty produces in the LQR tree; the recorded operators then drive hundreds of
  // ADMM iterations: on cfg-B (12D quadrotor, N = 100, 500-1000 iterations per QP) the
  // factored LQR tree moves inner iteration counts by up to 22 against the reference
  // (the dense tree: <= 1, tests/test_gpu_configs.py).  The SLS costs keep P_r C_l = O(1):
  // there the factored tree matches the oracle as closely as the dense one
  // (tools/probe/sls_factored_shapes.py, tools/probe/tau_sensitivity.py).
  // GSLS_LOWRANK: "0" none, "1" / "all" both trees, "lqr" the LQR tree only.
  bool on = tree == 1;
  if (const char* e = getenv("GSLS_LOWRANK")) {
    if (e[0] == '0') on = false;
    else if (e[0] == '1' || e[0] == 'a') on = true;
    else if (e[0] == 'l') on = tree == 0;
    else if (e[0] == 's') on = tree == 1;
  }
  return on ? (n / 4) * 4 : 0;  // the output factor [U, F_r] must fit the slot's n x ldg storage
}

int upload_plan(Ctx* c, const ScanPlan& p, const int4** ops, const int** out, const int** loff, int kind,
                const int** leaf_dead, const std::vector<int>* leaf_rank, int rmax) {
  std::vector<int4> h(p.ops.size() ? p.ops.size() : 1);
  // Dead-output flags in .w, from the last layer back (kind: PLAN_CVF / PLAN_CVF_REC /
  // PLAN_OTHER).  For a CVF combine (dst <- earlier (x) later) a reader needs, of its
  // earlier operand, C, A and P always; of its later operand, P always, A^T when the
  // reader forms Psi (its own A, A^T or C is live, or it is recorded) and C when the
  // reader forms its own C.
  //   bit 0: CVF: the output's A, A^T and C are all dead (only P may be read);
  //          other plans: the slot is never read again.
  //   bit 1: CVF: the output's C is dead.
  //   bit 2: CVF: the output's A^T is dead (no transposed copy).
  const int ns = std::max(p.nslots, 1);
  std::vector<char> rd(ns, 0), nA(ns, 0), nAT(ns, 0), nC(ns, 0);
  const bool cvf = kind != PLAN_OTHER, rec = kind == PLAN_CVF_REC;
  for (int l = (int)p.layer_off.size() - 2; l >= 0; --l) {
    for (int o = p.layer_off[l]; o < p.layer_off[l + 1]; ++o) {
      const ScanOp& q = p.ops[o];
      int w = 0;
      if (q.dst >= 0) {
        if (!cvf) w = rd[q.dst] ? 0 : 1;
        else w = ((nA[q.dst] || nAT[q.dst] || nC[q.dst]) ? 0 : 1) | (nC[q.dst] ? 0 : 2) | (nAT[q.dst] ? 0 : 4);
      }
      h[o] = make_int4(q.dst, q.earlier, q.later, w);
    }
    for (int o = p.layer_off[l]; o < p.layer_off[l + 1]; ++o) {
      const ScanOp& q = p.ops[o];
      const bool psi = rec || !(h[o].w & 1), ownc = !(h[o].w & 2);
      if (q.earlier >= 0) rd[q.earlier] = nA[q.earlier] = nC[q.earlier] = 1;
      if (q.later >= 0) {
        rd[q.later] = 1;
        if (psi) nAT[q.later] = 1;
        if (ownc) nC[q.later] = 1;
      }
    }
  }
  // C representation (CVF plans; lowrank.cuh): every slot's C is either a factor F F'
  // (F: n x rank, rank <= rmax) or dense.  Leaves have the ranks given (m; 0 for the
  // terminal element); a combine's C has rank <= rank C_earlier + rank C_later, so its
  // output is a factor while both operands are and the sum stays <= rmax.  A combine
  // whose earlier C is dense takes the dense path, which adds C_later as a dense matrix
  // when it forms its own C: such a later slot is forced dense (its producer then writes
  // the dense C), iterated to a fixed point.
  //   .w bits 8-15: rank of the earlier operand's C factor (255: dense -> dense path)
  //   .w bits 16-23: rank of the later operand's C factor (255: dense)
  //   .w bit 3: the output C is stored as a factor
  // Leaf flag bit 3: the leaf's C is stored as a factor.
  std::vector<int> rep(ns, -1);
  if (cvf && leaf_rank) {
    std::vector<char> forced(ns, 0);
    for (int iter = 0; iter < ns + 1; ++iter) {
      for (int i = 0; i < p.length && i < ns; ++i) rep[i] = forced[i] ? -1 : (*leaf_rank)[i];
      for (const ScanOp& q : p.ops) {
        const int re = rep[q.earlier], rl = rep[q.later];
        rep[q.dst] = (forced[q.dst] || re < 0 || rl < 0 || re + rl > rmax) ? -1 : re + rl;
      }
      bool changed = false;
      for (size_t o = 0; o < p.ops.size(); ++o) {
        const ScanOp& q = p.ops[o];
        if (rep[q.earlier] < 0 && !(h[o].w & 2) && rep[q.later] >= 0 && !forced[q.later]) {
          forced[q.later] = 1;
          changed = true;
        }
      }
      if (!changed) break;
    }
  }
  if (cvf)
    for (size_t o = 0; o < p.ops.size(); ++o) {
      const ScanOp& q = p.ops[o];
      const int re = rep[q.earlier], rl = rep[q.later];
      h[o].w |= ((re < 0 ? 255 : re) << 8) | ((rl < 0 ? 255 : rl) << 16) | (rep[q.dst] >= 0 ? 8 : 0);
    }
  if (cvf && getenv("GSLS_PLAN_VERBOSE")) {  // per layer: factored ops (rank histogram), dense ops, P-only ops
    for (int l = 0; l + 1 < (int)p.layer_off.size(); ++l) {
      int nf = 0, nd = 0, fin = 0, rsum = 0;
      for (int o = p.layer_off[l]; o < p.layer_off[l + 1]; ++o) {
        const int re = (h[o].w >> 8) & 0xFF;
        if (re == 255) ++nd; else { ++nf; rsum += re; }
        fin += h[o].w & 1;
      }
      fprintf(stderr, "plan%s layer %d: %d factored (mean rank %.1f), %d dense, %d P-only\n", rec ? " rec" : "", l, nf,
              nf ? (double)rsum / nf : 0.0, nd, fin);
    }
  }
  if (leaf_dead) {  // per leaf slot (< p.length): bit 0 A dead, bit 1 A^T dead, bit 2 C dead, bit 3 C factored
    std::vector<int> lf(std::max(p.length, 1), 0);
    for (int i = 0; i < p.length && i < ns; ++i)
      lf[i] = (nA[i] ? 0 : 1) | (nAT[i] ? 0 : 2) | (nC[i] ? 0 : 4) | (rep[i] >= 0 ? 8 : 0);
    int* dlf = (int*)dev_alloc(c, lf.size() * sizeof(int));
    if (!dlf) return GSLS_ERR_CUDA;
    GSLS_CUDA_CHECK(cudaMemcpy(dlf, lf.data(), lf.size() * sizeof(int), cudaMemcpyHostToDevice));
    *leaf_dead = dlf;
  }
  int4* dops = (int4*)dev_alloc(c, h.size() * sizeof(int4));
  int* dout = (int*)dev_alloc(c, (p.out.size() + 1) * sizeof(int));
  int* dl = (int*)dev_alloc(c, (p.layer_off.size() + 1) * sizeof(int));
  if (!dops || !dout || !dl) return GSLS_ERR_CUDA;
  GSLS_CUDA_CHECK(cudaMemcpy(dops, h.data(), h.size() * sizeof(int4), cudaMemcpyHostToDevice));
  if (!p.out.empty()) GSLS_CUDA_CHECK(cudaMemcpy(dout, p.out.data(), p.out.size() * sizeof(int), cudaMemcpyHostToDevice));
  if (!p.layer_off.empty())
    GSLS_CUDA_CHECK(cudaMemcpy(dl, p.layer_off.data(), p.layer_off.size() * sizeof(int), cudaMemcpyHostToDevice));
  *ops = dops;
  *out = dout;
  *loff = dl;
  return GSLS_OK;
}

int ctx_create(const gsls_dims_t* dims, Ctx** out) {
  const gsls_dims_t d = *dims;
  if (d.nx < 1 || d.nu < 0 || d.nc < 0 || d.nf < 0 || d.N < 0 || d.batch < 1) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "invalid dimensions");
    return GSLS_ERR_ARG;
  }
  if (d.nx > kMaxN || d.nu > kMaxM || (d.N > 0 && d.nu < 1)) {
    set_error(GSLS_ERR_TOO_LARGE, -1, 0, 0, 0, "dimensions exceed compiled limits (nx<=80, 1<=nu<=24)");
    return GSLS_ERR_TOO_LARGE;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error(GSLS_ERR_NO_DEVICE, -1, 0, 0, 0, "no CUDA device");
    return GSLS_ERR_NO_DEVICE;
  }
  Ctx* c = new Ctx();
  c->dims = d;
  c->ldg = ldg_of(d.nx);
  c->mtot = d.N * d.nc + d.nf;
  c->cvf = make_scan_plan(d.N + 1, true);
  const std::vector<int> cvf_blive = partition_unread_last(c->cvf);
  c->cot = d.N > 0 ? make_scan_plan(d.N, false) : ScanPlan{};
  c->cvf_layer_off = c->cvf.layer_off;
  c->cot_layer_off = c->cot.layer_off;
  if (c->cot_layer_off.empty()) c->cot_layer_off.push_back(0);
  for (int l = 0; l < c->cvf.layers; ++l)
    c->cvf_max_layer = std::max(c->cvf_max_layer, c->cvf_layer_off[l + 1] - c->cvf_layer_off[l]);
  for (int l = 0; l < c->cot.layers; ++l)
    c->cot_max_layer = std::max(c->cot_max_layer, c->cot_layer_off[l + 1] - c->cot_layer_off[l]);

  DevLqr& L = c->dev;
  L.n = d.nx; L.m = d.nu; L.c = d.nc; L.nf = d.nf; L.N = d.N; L.ldg = c->ldg; L.mtot = c->mtot;
  // leaf C ranks: B R^-1 B' (m) at the stages, 0 at the terminal element (lqr.py:306-320)
  std::vector<int> leaf_rank(d.N + 1, round_up(d.nu, 4));  // factor ranks carried as multiples of 4
  leaf_rank[d.N] = 0;
  const int rmax = factor_rmax(d.nx, 0);
  int rc = upload_plan(c, c->cvf, &c->cvf_ops_v[1], &L.cvf_out, &L.cvf_loff, PLAN_CVF_REC, &c->cvf_leaf_v[1]);
  if (!rc)
    rc = upload_plan(c, c->cvf, &c->cvf_ops_v[0], &L.cvf_out, &L.cvf_loff, PLAN_CVF_REC, &c->cvf_leaf_v[0],
                     rmax > 0 ? &leaf_rank : nullptr, rmax);
  c->lqr_dense = false;
  L.cvf_ops = c->cvf_ops_v[0];
  L.cvf_leaf = c->cvf_leaf_v[0];
  if (!rc && d.N > 0) rc = upload_plan(c, c->cot, &L.cot_ops, &L.cot_out, &L.cot_loff, PLAN_OTHER);
  if (rc) { delete c; return rc; }
  L.cvf_nphys = compress_slots(c->cvf, c->cvf_phys);
  L.cot_nphys = d.N > 0 ? compress_slots(c->cot, c->cot_phys) : 0;
  {
    int* dp = (int*)dev_alloc(c, (c->cvf_phys.size() + c->cot_phys.size() + 1) * sizeof(int));
    if (!dp) { delete c; return GSLS_ERR_CUDA; }
    GSLS_CUDA_CHECK(cudaMemcpy(dp, c->cvf_phys.data(), c->cvf_phys.size() * sizeof(int), cudaMemcpyHostToDevice));
    if (!c->cot_phys.empty())
      GSLS_CUDA_CHECK(cudaMemcpy(dp + c->cvf_phys.size(), c->cot_phys.data(), c->cot_phys.size() * sizeof(int),
                                 cudaMemcpyHostToDevice));
    L.cvf_phys = dp;
    L.cot_phys = dp + c->cvf_phys.size();
  }
  {
    int* db = (int*)dev_alloc(c, (cvf_blive.size() + 1) * sizeof(int));
    if (!db) { delete c; return GSLS_ERR_CUDA; }
    if (!cvf_blive.empty())
      GSLS_CUDA_CHECK(cudaMemcpy(db, cvf_blive.data(), cvf_blive.size() * sizeof(int), cudaMemcpyHostToDevice));
    L.cvf_blive = db;
  }
  L.cvf_nslots = c->cvf.nslots;
  L.cvf_nops = (int)c->cvf.ops.size();
  L.cvf_layers = c->cvf.layers;
  L.cot_nslots = c->cot.nslots;
  L.cot_nops = (int)c->cot.ops.size();
  L.cot_layers = c->cot.layers;
  const size_t B = d.batch, MS = mat_elems(d.nx), n = d.nx, m = d.nu, N = d.N;
  L.Ps = (float*)dev_alloc(c, B * L.cvf_nslots * MS * 4);
  L.As = (float*)dev_alloc(c, B * L.cvf_nslots * MS * 4);
  L.Cs = (float*)dev_alloc(c, B * L.cvf_nslots * MS * 4);
  L.ATs = (float*)dev_alloc(c, B * L.cvf_nslots * MS * 4);
  L.cvf_rec = (float*)dev_alloc(c, B * L.cvf_nops * 4 * MS * 4);
  L.cotA = (float*)dev_alloc(c, B * L.cot_nslots * MS * 4);
  L.cotAT = (float*)dev_alloc(c, B * L.cot_nslots * MS * 4);
  L.cot_rec = (float*)dev_alloc(c, B * L.cot_nops * MS * 4);
  L.Rhat = (double*)dev_alloc(c, B * N * m * m * 8);
  L.Shat = (float*)dev_alloc(c, B * N * m * n * 4);
  L.Shat64 = (double*)dev_alloc(c, B * N * m * n * 8);
  L.Rinv = (float*)dev_alloc(c, B * N * m * m * 4);
  L.Gamma = (float*)dev_alloc(c, B * N * m * m * 4);
  L.K = (float*)dev_alloc(c, B * N * m * n * 4);
  L.cvec = (double*)dev_alloc(c, B * N * n * 8);
  L.v0 = (double*)dev_alloc(c, B * n * 8);
  L.last_k = (double*)dev_alloc(c, B * N * m * 8);
  L.last_p = (double*)dev_alloc(c, B * (N + 1) * n * 8);
  L.err = (ErrSlot*)dev_alloc(c, B * sizeof(ErrSlot));
  const size_t cc = d.nc;
  L.ldm = ldg_of(d.nu); L.ldn = ldg_of(d.nx); L.ldc = ldg_of(std::max(1, d.nc)); L.ld2n = ldg_of(2 * d.nx);
  L.fd_ldg.init(ldg_of(d.nx)); L.fd_m.init(d.nu); L.fd_n.init(d.nx); L.fd_c.init(std::max(1, d.nc));
  L.fd_ldm.init(L.ldm); L.fd_ldn.init(L.ldn); L.fd_ldc.init(L.ldc); L.fd_ld2n.init(L.ld2n);
  L.X23 = (float*)dev_alloc(c, std::max<size_t>(1, B * N * cc * L.ld2n) * 4);
  L.pb0 = (double*)dev_alloc(c, std::max<size_t>(1, B * N * 2 * n) * 8);
  L.XK = (float*)dev_alloc(c, std::max<size_t>(1, B * N * (n + cc) * L.ldm) * 4);
  L.kk0 = (double*)dev_alloc(c, std::max<size_t>(1, B * N * m) * 8);
  L.Bcm = (float*)dev_alloc(c, std::max<size_t>(1, B * N * m * L.ldn) * 4);
  L.ZD = (float*)dev_alloc(c, std::max<size_t>(1, B * N * (n + m) * L.ldc) * 4);
  c->d_inst_all = (int*)dev_alloc(c, B * sizeof(int));
  c->d_inst_list = (int*)dev_alloc(c, B * sizeof(int));
  c->d_build_list = (int*)dev_alloc(c, B * sizeof(int));
  c->d_status = (int32_t*)dev_alloc(c, B * sizeof(int32_t));
  c->d_counts = (int*)dev_alloc(c, 4 * sizeof(int));
  cudaStreamCreateWithFlags(&c->body_stream, cudaStreamNonBlocking);
  c->scratch_floats = replay_smem_floats(c);  // doubles
  if (c->scratch_floats * 8 > kReplaySmemMax) c->d_scratch = (double*)dev_alloc(c, B * c->scratch_floats * 8);
  bool fail = !L.Ps || !L.As || !L.Cs || !L.ATs || !L.cotAT || !L.cvf_rec || !L.cotA || !L.cot_rec || !L.Rhat || !L.Shat || !L.Shat64 || !L.Rinv ||
              !L.Gamma || !L.K || !L.cvec || !L.v0 || !L.last_k || !L.last_p || !L.err || !L.X23 || !L.pb0 || !L.XK || !L.kk0 ||
              !L.Bcm || !L.ZD || !c->d_inst_all || !c->d_inst_list || !c->d_build_list || !c->d_status || !c->d_counts ||
              (c->scratch_floats * 8 > kReplaySmemMax && !c->d_scratch);
  if (fail) {
    for (void* p : c->allocs) cudaFree(p);
    delete c;
    set_error(GSLS_ERR_CUDA, -1, 0, 0, 0, "device allocation failed");
    return GSLS_ERR_CUDA;
  }
  std::vector<int> all(B);
  for (size_t i = 0; i < B; ++i) all[i] = (int)i;
  GSLS_CUDA_CHECK(cudaMemcpy(c->d_inst_all, all.data(), B * sizeof(int), cudaMemcpyHostToDevice));
  c->gen_host.assign(B, -1);
  *out = c;
  return GSLS_OK;
}

void ctx_destroy(Ctx* c) {
  if (!c) return;
  if (c->side) cudaStreamDestroy(c->side);
  if (c->body_stream) cudaStreamDestroy(c->body_stream);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->step_side) cudaStreamDestroy(c->step_side);
  if (c->step_fork) cudaEventDestroy(c->step_fork);
  if (c->step_join) cudaEventDestroy(c->step_join);
  if (c->sls) sls_destroy(c);
  for (void* p : c->allocs) cudaFree(p);
  delete c;
}

}  // namespace gsls
