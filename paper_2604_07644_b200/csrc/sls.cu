// SLS disturbance-feedback synthesis and tube tightening on the device.
//
// The reference scans a full (position x injection-time) grid with neutral
// elements outside each column's range (sls.py:245-285).  Here every column j
// gets the SAME balanced tree (scan.py:141-234) with its neutral positions
// resolved symbolically (plan.h): combines with a neutral element are exact
// no-ops in the reference, so eliding them changes no value while cutting the
// work from T(N+1)*N combines to ~N(N-1).  Scan values live in
// a triangular cell layout: cell(k, j), k in [j+1, N], one n x ldg block each.
//
// Reference map:
//   k_sls_assemble  assemble_costs            sls.py:176-200
//   k_sls_leaf      synthesize grid leaves    sls.py:245-279
//   (CVF tree)      _sls_cvf_kernel           sls.py:203-207, :281-285  (k_cvf_combine, no record)
//   k_sls_gains     G, K grid, closed loop    sls.py:287-302
//   k_matprod       _matprod_kernel           sls.py:217-218, :303-307
//   k_sls_phi       Phi^u = K Phi^x, rows     sls.py:310-318, :336, :340
//   k_sls_tighten   tighten                   sls.py:329-341
//   k_sls_duals     compute_duals             sls.py:150-173
#include <algorithm>
#include <cmath>
#include <vector>

#include "ctx.h"
#include "smallmat.cuh"

namespace gsls {

int check_errors(Ctx* c, cudaStream_t st, const char* what);
void set_error(int code, int inst, int where, int aux, int label, const char* msg);
__host__ __device__ inline int cell_of(int N, int k, int j) { return j * N - j * (j - 1) / 2 + (k - j - 1); }

// merge per-column plans into one layered plan with remapped slots
static ScanPlan merge_columns(int N, bool cvf) {
  const int ncell = N * (N + 1) / 2;
  ScanPlan out;
  const int len = cvf ? N + 1 : N;
  out.layers = scan_depth(len);
  std::vector<std::vector<ScanOp>> per_layer(out.layers);
  out.out.assign(ncell, -1);
  int next = ncell;
  for (int j = 0; j < N; ++j) {
    std::vector<char> neutral(len, 0);
    for (int p = 0; p < len; ++p) neutral[p] = cvf ? (p <= j) : (p < j);
    ScanPlan pj = make_scan_plan(len, cvf, neutral, 0);
    const int base = next;
    auto remap = [&](int s) -> int {
      if (s < 0) return -1;
      if (s < len) return cvf ? cell_of(N, s, j) : cell_of(N, s + 1, j);  // leaf position
      return base + (s - len);
    };
    next += pj.nslots - len;
    for (int l = 0; l < pj.layers; ++l)
      for (int o = pj.layer_off[l]; o < pj.layer_off[l + 1]; ++o)
        per_layer[l].push_back({remap(pj.ops[o].dst), remap(pj.ops[o].earlier), remap(pj.ops[o].later)});
    for (int k = j + 1; k <= N; ++k) out.out[cell_of(N, k, j)] = remap(pj.out[cvf ? k : k - 1]);
  }
  for (int l = 0; l < out.layers; ++l) {
    out.layer_off.push_back((int)out.ops.size());
    for (auto& o : per_layer[l]) out.ops.push_back(o);
  }
  out.layer_off.push_back((int)out.ops.size());
  out.length = ncell;
  out.nslots = next;
  return out;
}

struct DevSls {
  int n, m, c, nf, N, ldg, ncell, cmax;
  const int2* cell_kj;
  const int4* cvf_ops;
  const int* cvf_out;
  const int* cvf_loff;
  int cvf_nslots, cvf_nops, cvf_layers;
  const int4* mp_ops;
  const int* mp_out;
  const int* mp_loff;
  int mp_nslots, mp_nops, mp_layers;
  float *Ps, *As, *Cs, *Ms;
  float *Qx, *Qu, *Qux, *Kc, *Phiu;
  double* rn;
  ErrSlot* err;
  int have_response;
};

struct SlsState {
  ScanPlan cvf, mp;
  DevSls dev{};
  bool ready = false;
};

static SlsState* sls_of(Ctx* c) { return reinterpret_cast<SlsState*>(c->sls); }

void sls_destroy(Ctx* c) { delete sls_of(c); c->sls = nullptr; }

static int sls_init(Ctx* c) {
  if (c->sls) return GSLS_OK;
  const gsls_dims_t& d = c->dims;
  if (d.N < 1) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "SLS needs N >= 1");
    return GSLS_ERR_ARG;
  }
  SlsState* s = new SlsState();
  c->sls = s;
  DevSls& S = s->dev;
  const int N = d.N, n = d.nx, m = d.nu;
  S.n = n; S.m = m; S.c = d.nc; S.nf = d.nf; S.N = N; S.ldg = ldg_of(n);
  S.ncell = N * (N + 1) / 2;
  S.cmax = std::max(1, std::max(d.nc, d.nf));
  s->cvf = merge_columns(N, true);
  s->mp = merge_columns(N, false);
  int rc = upload_plan(c, s->cvf, &S.cvf_ops, &S.cvf_out, &S.cvf_loff);
  if (!rc) rc = upload_plan(c, s->mp, &S.mp_ops, &S.mp_out, &S.mp_loff);
  if (rc) return rc;
  S.cvf_nslots = s->cvf.nslots; S.cvf_nops = (int)s->cvf.ops.size(); S.cvf_layers = s->cvf.layers;
  S.mp_nslots = s->mp.nslots; S.mp_nops = (int)s->mp.ops.size(); S.mp_layers = s->mp.layers;
  std::vector<int2> kj(S.ncell);
  for (int j = 0; j < N; ++j)
    for (int k = j + 1; k <= N; ++k) kj[cell_of(N, k, j)] = make_int2(k, j);
  int2* dkj = (int2*)dev_alloc(c, sizeof(int2) * S.ncell);
  if (!dkj) return GSLS_ERR_CUDA;
  GSLS_CUDA_CHECK(cudaMemcpy(dkj, kj.data(), sizeof(int2) * S.ncell, cudaMemcpyHostToDevice));
  S.cell_kj = dkj;
  const size_t B = d.batch, MS = mat_elems(n);
  S.Ps = (float*)dev_alloc(c, B * S.cvf_nslots * MS * 4);
  S.As = (float*)dev_alloc(c, B * S.cvf_nslots * MS * 4);
  S.Cs = (float*)dev_alloc(c, B * S.cvf_nslots * MS * 4);
  S.Ms = (float*)dev_alloc(c, B * S.mp_nslots * MS * 4);
  S.Qx = (float*)dev_alloc(c, B * S.ncell * MS * 4);
  S.Qu = (float*)dev_alloc(c, B * S.ncell * m * m * 4);
  S.Qux = (float*)dev_alloc(c, B * S.ncell * m * n * 4);
  S.Kc = (float*)dev_alloc(c, B * S.ncell * m * n * 4);
  S.Phiu = (float*)dev_alloc(c, B * S.ncell * m * n * 4);
  S.rn = (double*)dev_alloc(c, B * S.ncell * S.cmax * 8);
  S.err = c->dev.err;
  if (!S.Ps || !S.As || !S.Cs || !S.Ms || !S.Qx || !S.Qu || !S.Qux || !S.Kc || !S.Phiu || !S.rn) {
    set_error(GSLS_ERR_CUDA, -1, 0, 0, 0, "SLS workspace allocation failed");
    return GSLS_ERR_CUDA;
  }
  s->ready = true;
  return GSLS_OK;
}

// ---------------------------------------------------------------------------
// kernels

// [C D]' diag(tau) [C D] + blkdiag(Qbar, Rbar) per cell; terminal cells (k = N)
// get CN' diag(tau_N) CN + QbarN.  Weights are per instance (stride wst, 0 = shared).
__global__ void __launch_bounds__(256) k_sls_assemble(DevSls S, gsls_qp_t qp, const double* tau,
                                                      const double* tau_term, const float* Qbar, const float* Rbar,
                                                      const float* QbarN, long long wst) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int2 kj = S.cell_kj[cell];
  const int k = kj.x, j = kj.y;
  const int n = S.n, m = S.m, c = S.c, nf = S.nf, N = S.N, ldg = S.ldg;
  const size_t MS = (size_t)n * ldg;
  float* Qx = S.Qx + ((size_t)inst * S.ncell + cell) * MS;
  extern __shared__ float sm[];
  float* t = sm;  // c or nf
  if (k == N) {
    const float* CN = qp.CN + (size_t)inst * nf * n;
    const float* QbN = QbarN + (size_t)inst * wst * n * n;
    for (int f = threadIdx.x; f < nf; f += blockDim.x)
      t[f] = tau_term ? (float)tau_term[((size_t)inst * N + j) * nf + f] : 0.f;
    __syncthreads();
    for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) {
      const int i = e / ldg, jj = e - i * ldg;
      float v = 0.f;
      if (jj < n) {
        float s = 0.f;
        for (int f = 0; f < nf; ++f) s = fmaf(CN[f * n + i] * t[f], CN[f * n + jj], s);
        v = s + QbN[i * n + jj];
      }
      Qx[e] = v;
    }
    return;
  }
  const size_t st = (size_t)inst * N + k;
  const float* Ck = qp.C + st * c * n;
  const float* Dk = qp.D + st * c * m;
  for (int r = threadIdx.x; r < c; r += blockDim.x)
    t[r] = tau ? (float)tau[((size_t)inst * S.ncell + cell) * c + r] : 0.f;
  __syncthreads();
  const float* Qb = Qbar + (size_t)inst * wst * n * n;
  const float* Rb = Rbar + (size_t)inst * wst * m * m;
  for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) {
    const int i = e / ldg, jj = e - i * ldg;
    float v = 0.f;
    if (jj < n) {
      float s = 0.f;
      for (int r = 0; r < c; ++r) s = fmaf(Ck[r * n + i] * t[r], Ck[r * n + jj], s);
      v = s + Qb[i * n + jj];
    }
    Qx[e] = v;
  }
  float* Qu = S.Qu + ((size_t)inst * S.ncell + cell) * m * m;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int a = e / m, b = e - a * m;
    float s = 0.f;
    for (int r = 0; r < c; ++r) s = fmaf(Dk[r * m + a] * t[r], Dk[r * m + b], s);
    Qu[e] = s + Rb[e];
  }
  float* Qux = S.Qux + ((size_t)inst * S.ncell + cell) * m * n;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int a = e / n, i = e - a * n;
    float s = 0.f;
    for (int r = 0; r < c; ++r) s = fmaf(Dk[r * m + a] * t[r], Ck[r * n + i], s);
    Qux[e] = s;
  }
}

// Grid leaves: Qu^-1, P = Qx - Qux' Qu^-1 Qux, A = A_k - B_k Qu^-1 Qux, C = B_k Qu^-1 B_k'.
__global__ void __launch_bounds__(256) k_sls_leaf(DevSls S, gsls_qp_t qp) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int2 kj = S.cell_kj[cell];
  const int k = kj.x, j = kj.y;
  const int n = S.n, m = S.m, N = S.N, ldg = S.ldg;
  const size_t MS = (size_t)n * ldg;
  const int slot = cell;  // leaves occupy slots [0, ncell)
  float* Pd = S.Ps + ((size_t)inst * S.cvf_nslots + slot) * MS;
  float* Ad = S.As + ((size_t)inst * S.cvf_nslots + slot) * MS;
  float* Cd = S.Cs + ((size_t)inst * S.cvf_nslots + slot) * MS;
  const float* Qx = S.Qx + ((size_t)inst * S.ncell + cell) * MS;
  if (k == N) {  // terminal element (Qx_term, 0, 0)
    for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) { Pd[e] = Qx[e]; Ad[e] = 0.f; Cd[e] = 0.f; }
    return;
  }
  extern __shared__ float sm[];
  float* Qu = sm;             // m x m
  float* Qi = Qu + m * m;     // m x m
  float* Qux = Qi + m * m;    // m x n
  float* QQ = Qux + m * n;    // m x n
  float* Bk = QQ + m * n;     // n x m
  float* BQ = Bk + n * m;     // n x m
  float* wk = BQ + n * m;
  const size_t cb = (size_t)inst * S.ncell + cell;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) Qu[e] = S.Qu[cb * m * m + e];
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) Qux[e] = S.Qux[cb * m * n + e];
  const size_t st = (size_t)inst * N + k;
  for (int e = threadIdx.x; e < n * m; e += blockDim.x) Bk[e] = qp.B[st * n * m + e];
  __syncthreads();
  if (threadIdx.x < 32) {
    if (warp_spd_inverse(Qu, m, Qi, m, wk) && threadIdx.x == 0)
      raise_err(S.err + inst, GSLS_ERR_SINGULAR_STAGE, k, j, GSLS_LABEL_QU);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int a = e / n, i = e - a * n;
    float s = 0.f;
    for (int b = 0; b < m; ++b) s = fmaf(Qi[a * m + b], Qux[b * n + i], s);
    QQ[e] = s;
  }
  for (int e = threadIdx.x; e < n * m; e += blockDim.x) {
    const int i = e / m, a = e - i * m;
    float s = 0.f;
    for (int b = 0; b < m; ++b) s = fmaf(Bk[i * m + b], Qi[b * m + a], s);
    BQ[e] = s;
  }
  __syncthreads();
  const float* Ak = qp.A + st * n * n;
  for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) {
    const int i = e / ldg, jj = e - i * ldg;
    float p = 0.f, a = 0.f, cc = 0.f;
    if (jj < n) {
      float s1 = 0.f, s2 = 0.f, s3 = 0.f;
      for (int l = 0; l < m; ++l) {
        s1 = fmaf(Qux[l * n + i], QQ[l * n + jj], s1);
        s2 = fmaf(Bk[i * m + l], QQ[l * n + jj], s2);
        s3 = fmaf(BQ[i * m + l], Bk[jj * m + l], s3);
      }
      p = Qx[i * ldg + jj] - s1;
      a = Ak[i * n + jj] - s2;
      cc = s3;
    }
    Pd[e] = p;
    Ad[e] = a;
    Cd[e] = cc;
  }
}

// Gains on cell (k, j), k <= N-1, from P+ = P(k+1, j); closed loop -> product
// leaf of position k.  Cell (N, j) writes E_j into the leaf of position j.
__global__ void __launch_bounds__(256) k_sls_gains(DevSls S, gsls_qp_t qp, const float* E) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int2 kj = S.cell_kj[cell];
  const int k = kj.x, j = kj.y;
  const int n = S.n, m = S.m, N = S.N, ldg = S.ldg;
  const size_t MS = (size_t)n * ldg;
  float* Mbase = S.Ms + (size_t)inst * S.mp_nslots * MS;
  if (k == N) {
    float* Ml = Mbase + (size_t)cell_of(N, j + 1, j) * MS;
    const float* Ej = E + ((size_t)inst * N + j) * n * n;
    for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) {
      const int i = e / ldg, jj = e - i * ldg;
      Ml[e] = (jj < n) ? Ej[i * n + jj] : 0.f;
    }
    return;
  }
  extern __shared__ float sm[];
  float* Pn = sm;               // n x ldg
  float* Bst = Pn + n * ldg;    // n x m
  float* BtP = Bst + n * m;     // m x n
  float* H = BtP + m * n;       // m x m
  float* Gm = H + m * m;        // m x n
  float* Ga = Gm + m * m;       // m x m
  float* Ks = Ga + m * m;       // m x n
  float* wk = Ks + m * n;
  const float* Pg = S.Ps + ((size_t)inst * S.cvf_nslots + S.cvf_out[cell_of(N, k + 1, j)]) * MS;
  for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) Pn[e] = Pg[e];
  const size_t st = (size_t)inst * N + k;
  for (int e = threadIdx.x; e < n * m; e += blockDim.x) Bst[e] = qp.B[st * n * m + e];
  __syncthreads();
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int l = e / n, jj = e - l * n;
    float s = 0.f;
    for (int i = 0; i < n; ++i) s = fmaf(Bst[i * m + l], Pn[i * ldg + jj], s);
    BtP[e] = s;
  }
  __syncthreads();
  const float* Ak = qp.A + st * n * n;
  const size_t cb = (size_t)inst * S.ncell + cell;
  const float* Qu = S.Qu + cb * m * m;
  const float* Qux = S.Qux + cb * m * n;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int l = e / m, t = e - l * m;
    float s = 0.f;
    for (int i = 0; i < n; ++i) s = fmaf(BtP[l * n + i], Bst[i * m + t], s);
    H[e] = Qu[e] + s;
  }
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int l = e / n, jj = e - l * n;
    float s = 0.f;
    for (int i = 0; i < n; ++i) s = fmaf(BtP[l * n + i], Ak[i * n + jj], s);
    Gm[e] = Qux[e] + s;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    if (warp_spd_inverse(H, m, Ga, m, wk) && threadIdx.x == 0)
      raise_err(S.err + inst, GSLS_ERR_SINGULAR_STAGE, k, j, GSLS_LABEL_QU_BPB);
  }
  __syncthreads();
  float* Kg = S.Kc + cb * m * n;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int l = e / n, jj = e - l * n;
    float s = 0.f;
    for (int t = 0; t < m; ++t) s = fmaf(Ga[l * m + t], Gm[t * n + jj], s);
    Ks[e] = -s;
    Kg[e] = -s;
  }
  __syncthreads();
  float* Ml = Mbase + (size_t)cell_of(N, k + 1, j) * MS;  // product leaf of position k
  for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) {
    const int i = e / ldg, jj = e - i * ldg;
    float v = 0.f;
    if (jj < n) {
      float s = 0.f;
      for (int l = 0; l < m; ++l) s = fmaf(Bst[i * m + l], Ks[l * n + jj], s);
      v = Ak[i * n + jj] + s;
    }
    Ml[e] = v;
  }
}

// Matrix-product combine: M = M_later M_earlier (sls.py:217-218).
__global__ void __launch_bounds__(512) k_matprod(float* Ms, long long inst_stride, int n, const int4* ops) {
  const int inst = blockIdx.y;
  const int4 op = ops[blockIdx.x];
  const int ldg = ldg_of(n), lds = lds_of(n);
  const size_t MS = (size_t)n * ldg;
  extern __shared__ float sm[];
  float* Lt = sm;
  float* Er = Lt + (size_t)n * lds;
  float* base = Ms + (size_t)inst * inst_stride;
  cta_load_t(Lt, lds, base + (size_t)op.z * MS, ldg, n);
  cta_load(Er, lds, base + (size_t)op.y * MS, ldg, n, n);
  __syncthreads();
  gemm_tn(n, Lt, Er, lds, EpiGlobal{base + (size_t)op.x * MS, nullptr, ldg});
}

// Phi^u = K Phi^x and the constraint-row norms of C Phi^x + D Phi^u (terminal: CN Phi^x).
__global__ void __launch_bounds__(256) k_sls_phi(DevSls S, gsls_qp_t qp) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int2 kj = S.cell_kj[cell];
  const int k = kj.x;
  const int n = S.n, m = S.m, c = S.c, nf = S.nf, N = S.N, ldg = S.ldg;
  const size_t MS = (size_t)n * ldg;
  extern __shared__ float sm[];
  float* Px = sm;            // n x ldg
  float* Pu = Px + n * ldg;  // m x n
  const float* Pg = S.Ms + ((size_t)inst * S.mp_nslots + S.mp_out[cell]) * MS;
  for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) Px[e] = Pg[e];
  __syncthreads();
  const size_t cb = (size_t)inst * S.ncell + cell;
  double* rn = S.rn + cb * S.cmax;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (k == N) {
    const float* CN = qp.CN + (size_t)inst * nf * n;
    for (int f = warp; f < nf; f += nw) {
      double ss = 0.0;
      for (int i = lane; i < n; i += 32) {
        float s = 0.f;
        for (int l = 0; l < n; ++l) s = fmaf(CN[f * n + l], Px[l * ldg + i], s);
        ss += (double)s * (double)s;
      }
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) rn[f] = sqrt(ss);
    }
    return;
  }
  const float* Kg = S.Kc + cb * m * n;
  float* Pug = S.Phiu + cb * m * n;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int a = e / n, i = e - a * n;
    float s = 0.f;
    for (int l = 0; l < n; ++l) s = fmaf(Kg[a * n + l], Px[l * ldg + i], s);
    Pu[e] = s;
    Pug[e] = s;
  }
  __syncthreads();
  const size_t st = (size_t)inst * N + k;
  const float* Ck = qp.C + st * c * n;
  const float* Dk = qp.D + st * c * m;
  for (int r = warp; r < c; r += nw) {
    double ss = 0.0;
    for (int i = lane; i < n; i += 32) {
      float s1 = 0.f, s2 = 0.f;
      for (int l = 0; l < n; ++l) s1 = fmaf(Ck[r * n + l], Px[l * ldg + i], s1);
      for (int a = 0; a < m; ++a) s2 = fmaf(Dk[r * m + a], Pu[a * n + i], s2);
      const double v = (double)(s1 + s2);
      ss += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) rn[r] = sqrt(ss);
  }
}

// h_k = sum_{j<k} rownorm(k, j) (k >= 1; h_0 = 0); hf = sum_j rownorm(N, j).
__global__ void k_sls_tighten(DevSls S, double* h, double* hf) {
  const int inst = blockIdx.x;
  const int c = S.c, nf = S.nf, N = S.N;
  const double* rn = S.rn + (size_t)inst * S.ncell * S.cmax;
  for (int e = threadIdx.x; e < N * c; e += blockDim.x) {
    const int k = e / c, r = e - k * c;
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += rn[(size_t)cell_of(N, k, j) * S.cmax + r];
    h[(size_t)inst * N * c + e] = s;
  }
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < N; ++j) s += rn[(size_t)cell_of(N, N, j) * S.cmax + f];
    hf[(size_t)inst * nf + f] = s;
  }
}

// tau = max(lam, 0) / sqrt(beta + eps), beta = rownorm^2 (0 without a response).
__global__ void k_sls_duals(DevSls S, const double* lam_s, const double* lam_t, double eps, double* tau,
                            double* tau_term, double* beta, double* beta_term) {
  const int inst = blockIdx.x;
  const int c = S.c, nf = S.nf, N = S.N;
  const double* rn = S.rn + (size_t)inst * S.ncell * S.cmax;
  for (int e = threadIdx.x; e < S.ncell * c; e += blockDim.x) {
    const int cell = e / c, r = e - cell * c;
    const int2 kj = S.cell_kj[cell];
    if (kj.x >= N) continue;
    const double v = S.have_response ? rn[(size_t)cell * S.cmax + r] : 0.0;
    const double b = v * v;
    const double l = fmax(lam_s[((size_t)inst * N + kj.x) * c + r], 0.0);
    const size_t o = ((size_t)inst * S.ncell + cell) * c + r;
    tau[o] = l / sqrt(b + eps);
    if (beta) beta[o] = b;
  }
  for (int e = threadIdx.x; e < N * nf; e += blockDim.x) {
    const int j = e / nf, f = e - j * nf;
    const double v = S.have_response ? rn[(size_t)cell_of(N, N, j) * S.cmax + f] : 0.0;
    const double b = v * v;
    const double l = fmax(lam_t[(size_t)inst * nf + f], 0.0);
    tau_term[(size_t)inst * N * nf + e] = l / sqrt(b + eps);
    if (beta_term) beta_term[(size_t)inst * N * nf + e] = b;
  }
}

__global__ void k_sls_export(DevSls S, float* phix, float* phiu, float* gains) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int n = S.n, m = S.m, ldg = S.ldg, N = S.N;
  const int k = S.cell_kj[cell].x;
  const size_t cb = (size_t)inst * S.ncell + cell;
  if (phix) {
    const float* src = S.Ms + ((size_t)inst * S.mp_nslots + S.mp_out[cell]) * n * ldg;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) phix[cb * n * n + e] = src[(e / n) * ldg + e % n];
  }
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    if (phiu) phiu[cb * m * n + e] = (k < N) ? S.Phiu[cb * m * n + e] : 0.f;
    if (gains) gains[cb * m * n + e] = (k < N) ? S.Kc[cb * m * n + e] : 0.f;
  }
}

// ---------------------------------------------------------------------------
// host entry points

static int smem_attr(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024)
    GSLS_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return GSLS_OK;
}

int sls_assemble(Ctx* c, const gsls_qp_t* qp, const double* tau, const double* tau_term, const float* Qbar,
                 const float* Rbar, const float* QbarN, int weights_per_instance, cudaStream_t st) {
  int rc = sls_init(c);
  if (rc) return rc;
  DevSls& S = sls_of(c)->dev;
  const size_t sb = (size_t)S.cmax * sizeof(float) + 16;
  k_sls_assemble<<<dim3(S.ncell, c->dims.batch), 256, sb, st>>>(S, *qp, tau, tau_term, Qbar, Rbar, QbarN,
                                                                  weights_per_instance ? 1 : 0);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

// Explicit costs (cell layout, unpadded): Qx (B,ncell,n,n) with Qx_term on k = N
// cells, Qu (B,ncell,m,m), Qux (B,ncell,m,n).
__global__ void k_sls_set_costs(DevSls S, const float* Qx, const float* Qu, const float* Qux) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int n = S.n, m = S.m, ldg = S.ldg;
  const size_t cb = (size_t)inst * S.ncell + cell;
  for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) {
    const int i = e / ldg, j = e - i * ldg;
    S.Qx[cb * n * ldg + e] = (j < n) ? Qx[cb * n * n + i * n + j] : 0.f;
  }
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) S.Qu[cb * m * m + e] = Qu[cb * m * m + e];
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) S.Qux[cb * m * n + e] = Qux[cb * m * n + e];
}

int sls_set_costs(Ctx* c, const float* Qx, const float* Qu, const float* Qux, cudaStream_t st) {
  int rc = sls_init(c);
  if (rc) return rc;
  DevSls& S = sls_of(c)->dev;
  k_sls_set_costs<<<dim3(S.ncell, c->dims.batch), 256, 0, st>>>(S, Qx, Qu, Qux);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

int sls_synthesize(Ctx* c, const gsls_qp_t* qp, const float* E, cudaStream_t st, bool check) {
  int rc = sls_init(c);
  if (rc) return rc;
  SlsState* s = sls_of(c);
  DevSls& S = s->dev;
  const int B = c->dims.batch, n = S.n, m = S.m, ldg = S.ldg;
  const size_t MS = mat_elems(n);
  const size_t wk = 2 * kMaxM * (kMaxM + 1) + 8;
  {
    const size_t sb = (2 * m * m + 2 * m * n + 2 * n * m + wk) * sizeof(float);
    if ((rc = smem_attr((const void*)k_sls_leaf, sb))) return rc;
    k_sls_leaf<<<dim3(S.ncell, B), 256, sb, st>>>(S, *qp);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  for (int l = 0; l < s->cvf.layers; ++l) {
    const int o0 = s->cvf.layer_off[l], o1 = s->cvf.layer_off[l + 1];
    CombineArgs a{n, S.cvf_ops + o0, o0, S.Ps, S.As, S.Cs, (long long)S.cvf_nslots * (long long)MS, nullptr, 0,
                  nullptr, S.err, 1e-10f};
    if ((rc = launch_combine(a, o1 - o0, B, st))) return rc;
  }
  {
    const size_t sb = ((size_t)n * ldg + n * m + 3 * m * n + 2 * m * m + wk) * sizeof(float);
    if ((rc = smem_attr((const void*)k_sls_gains, sb))) return rc;
    k_sls_gains<<<dim3(S.ncell, B), 256, sb, st>>>(S, *qp, E);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  {
    const size_t sb = 2 * (size_t)n * lds_of(n) * sizeof(float);
    if ((rc = smem_attr((const void*)k_matprod, sb))) return rc;
    for (int l = 0; l < s->mp.layers; ++l) {
      const int o0 = s->mp.layer_off[l], o1 = s->mp.layer_off[l + 1];
      if (o1 == o0) continue;
      k_matprod<<<dim3(o1 - o0, B), combine_threads(n), sb, st>>>(S.Ms, (long long)S.mp_nslots * (long long)MS, n,
                                                                  S.mp_ops + o0);
      GSLS_CUDA_CHECK(cudaGetLastError());
    }
  }
  {
    const size_t sb = ((size_t)n * ldg + m * n) * sizeof(float);
    if ((rc = smem_attr((const void*)k_sls_phi, sb))) return rc;
    k_sls_phi<<<dim3(S.ncell, B), 256, sb, st>>>(S, *qp);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  S.have_response = 1;
  return check ? check_errors(c, st, "sls.synthesize") : GSLS_OK;
}

int sls_tighten(Ctx* c, double* h, double* hf, cudaStream_t st) {
  SlsState* s = sls_of(c);
  if (!s || !s->dev.have_response) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "no SLS response in context");
    return GSLS_ERR_ARG;
  }
  k_sls_tighten<<<c->dims.batch, 256, 0, st>>>(s->dev, h, hf);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

int sls_duals(Ctx* c, const double* lam_s, const double* lam_t, double eps, int use_response, double* tau,
              double* tau_term, double* beta, double* beta_term, cudaStream_t st) {
  int rc = sls_init(c);
  if (rc) return rc;
  DevSls S = sls_of(c)->dev;
  S.have_response = use_response && S.have_response;
  k_sls_duals<<<c->dims.batch, 256, 0, st>>>(S, lam_s, lam_t, eps, tau, tau_term, beta, beta_term);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

int sls_export(Ctx* c, float* phix, float* phiu, float* gains, cudaStream_t st) {
  SlsState* s = sls_of(c);
  if (!s || !s->dev.have_response) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "no SLS response in context");
    return GSLS_ERR_ARG;
  }
  k_sls_export<<<dim3(s->dev.ncell, c->dims.batch), 256, 0, st>>>(s->dev, phix, phiu, gains);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

int sls_ncell(int N) { return N * (N + 1) / 2; }

}  // namespace gsls
