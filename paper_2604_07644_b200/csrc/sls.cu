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
#include "prof.h"
#include "smallmat.cuh"

namespace gsls {

int check_errors(Ctx* c, cudaStream_t st, const char* what);
void set_error(int code, int inst, int where, int aux, int label, const char* msg);
__host__ __device__ inline int cell_of(int N, int k, int j) { return j * N - j * (j - 1) / 2 + (k - j - 1); }

// merge the per-column plans of columns [j0, j1) into one layered plan with remapped
// slots; leaves sit at the shard-local cell index cell(k, j) - cell(j0 + 1, j0)
static ScanPlan merge_columns(int N, bool cvf, int j0 = 0, int j1 = -1) {
  if (j1 < 0) j1 = N;
  const int cell0 = cell_of(N, j0 + 1, j0);
  const int ncell = cell_of(N, j1 + 1, j1) - cell0;
  ScanPlan out;
  const int len = cvf ? N + 1 : N;
  out.layers = scan_depth(len);
  std::vector<std::vector<ScanOp>> per_layer(out.layers);
  out.out.assign(ncell, -1);
  int next = ncell;
  for (int j = j0; j < j1; ++j) {
    std::vector<char> neutral(len, 0);
    for (int p = 0; p < len; ++p) neutral[p] = cvf ? (p <= j) : (p < j);
    ScanPlan pj = make_scan_plan(len, cvf, neutral, 0);
    const int base = next;
    auto remap = [&](int s) -> int {
      if (s < 0) return -1;
      if (s < len) return (cvf ? cell_of(N, s, j) : cell_of(N, s + 1, j)) - cell0;  // leaf position
      return base + (s - len);
    };
    next += pj.nslots - len;
    for (int l = 0; l < pj.layers; ++l)
      for (int o = pj.layer_off[l]; o < pj.layer_off[l + 1]; ++o)
        per_layer[l].push_back({remap(pj.ops[o].dst), remap(pj.ops[o].earlier), remap(pj.ops[o].later)});
    for (int k = j + 1; k <= N; ++k) out.out[cell_of(N, k, j) - cell0] = remap(pj.out[cvf ? k : k - 1]);
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
  FastDiv fd_ldg, fd_q4, fd_m, fd_n;  // ldg (= np), ldg / 4, m, n: the cell kernels' loop indices
  int j0, j1, cell0;  // column shard [j0, j1); ncell counts its cells, which start at global cell0
  const int2* cell_kj;
  const int* leaf_dead;  // per cell: bit 0 A, bit 1 A^T, bit 2 C of its CVF leaf never read
  const int4* cvf_ops;
  const int* cvf_out;
  const int* cvf_loff;
  int cvf_nslots, cvf_nops, cvf_layers;
  const int4* mp_ops;
  const int* mp_out;
  const int* mp_loff;
  int mp_nslots, mp_nops, mp_layers;
  float *Ps, *As, *Cs, *ATs, *Ms, *MsT;
  double *Qx, *Qu, *Qux;  // cost blocks (float64: the leaf Schur complement cancels O(tau) terms)
  double *Qi, *QL;        // per cell: Qu^-1 and L^-1 (Qu = L L') from k_sls_qu_inverse (m x m each)
  float *Kc, *Phiu;
  double* rn;
  ErrSlot* err;
  int have_response;
};

struct SlsState {
  ScanPlan cvf, mp;
  DevSls dev{};
  bool ready = false;
  // CVF plan variants (lowrank.cuh): [0] factored combines where C has low rank, [1] dense
  const int4* cvf_ops_v[2] = {nullptr, nullptr};
  const int* leaf_v[2] = {nullptr, nullptr};
  bool dense = false;
  double* cost_cells = nullptr;  // sls_cost: per (instance, cell) terms
};

static SlsState* sls_of(Ctx* c) { return reinterpret_cast<SlsState*>(c->sls); }

void sls_destroy(Ctx* c) { delete sls_of(c); c->sls = nullptr; }

void sls_use_dense(Ctx* c) {
  SlsState* s = sls_of(c);
  if (!s) return;
  s->dense = true;
  s->dev.cvf_ops = s->cvf_ops_v[1];
  s->dev.leaf_dead = s->leaf_v[1];
}

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
  S.fd_ldg.init(S.ldg);
  S.fd_q4.init(S.ldg / 4);
  S.fd_m.init(m);
  S.fd_n.init(n);
  S.j0 = c->sls_j0;
  S.j1 = c->sls_j1 < 0 ? N : c->sls_j1;
  S.cell0 = cell_of(N, S.j0 + 1, S.j0);
  S.ncell = cell_of(N, S.j1 + 1, S.j1) - S.cell0;
  S.cmax = std::max(1, std::max(d.nc, d.nf));
  s->cvf = merge_columns(N, true, S.j0, S.j1);
  s->mp = merge_columns(N, false, S.j0, S.j1);
  std::vector<int2> kj(S.ncell);
  for (int j = S.j0; j < S.j1; ++j)
    for (int k = j + 1; k <= N; ++k) kj[cell_of(N, k, j) - S.cell0] = make_int2(k, j);
  // leaf C ranks: B Qu^-1 B' (m) on the stage cells, 0 on the terminal cells (sls.py:262-278)
  std::vector<int> leaf_rank(S.ncell);
  for (int i = 0; i < S.ncell; ++i) leaf_rank[i] = kj[i].x == N ? 0 : round_up(m, 4);  // multiples of 4
  const int rmax = factor_rmax(n, 1);
  int rc = upload_plan(c, s->cvf, &s->cvf_ops_v[1], &S.cvf_out, &S.cvf_loff, PLAN_CVF, &s->leaf_v[1]);
  if (!rc)
    rc = upload_plan(c, s->cvf, &s->cvf_ops_v[0], &S.cvf_out, &S.cvf_loff, PLAN_CVF, &s->leaf_v[0],
                     rmax > 0 ? &leaf_rank : nullptr, rmax);
  if (!rc) rc = upload_plan(c, s->mp, &S.mp_ops, &S.mp_out, &S.mp_loff, PLAN_OTHER);
  if (rc) return rc;
  s->dense = false;
  S.cvf_ops = s->cvf_ops_v[0];
  S.leaf_dead = s->leaf_v[0];
  S.cvf_nslots = s->cvf.nslots; S.cvf_nops = (int)s->cvf.ops.size(); S.cvf_layers = s->cvf.layers;
  S.mp_nslots = s->mp.nslots; S.mp_nops = (int)s->mp.ops.size(); S.mp_layers = s->mp.layers;
  int2* dkj = (int2*)dev_alloc(c, sizeof(int2) * S.ncell);
  if (!dkj) return GSLS_ERR_CUDA;
  GSLS_CUDA_CHECK(cudaMemcpy(dkj, kj.data(), sizeof(int2) * S.ncell, cudaMemcpyHostToDevice));
  S.cell_kj = dkj;
  const size_t B = d.batch, MS = mat_elems(n);
  S.Ps = (float*)dev_alloc(c, B * S.cvf_nslots * MS * 4);
  S.As = (float*)dev_alloc(c, B * S.cvf_nslots * MS * 4);
  S.Cs = (float*)dev_alloc(c, B * S.cvf_nslots * MS * 4);
  S.ATs = (float*)dev_alloc(c, B * S.cvf_nslots * MS * 4);
  S.Ms = (float*)dev_alloc(c, B * S.mp_nslots * MS * 4);
  S.MsT = (float*)dev_alloc(c, B * S.mp_nslots * MS * 4);
  S.Qx = (double*)dev_alloc(c, B * S.ncell * n * n * 8);
  S.Qu = (double*)dev_alloc(c, B * S.ncell * m * m * 8);
  S.Qux = (double*)dev_alloc(c, B * S.ncell * m * n * 8);
  S.Qi = (double*)dev_alloc(c, B * S.ncell * m * m * 8);
  S.QL = (double*)dev_alloc(c, B * S.ncell * m * m * 8);
  S.Kc = (float*)dev_alloc(c, B * S.ncell * m * n * 4);
  S.Phiu = (float*)dev_alloc(c, B * S.ncell * m * n * 4);
  S.rn = (double*)dev_alloc(c, B * S.ncell * S.cmax * 8);
  S.err = c->dev.err;
  if (!S.Ps || !S.As || !S.Cs || !S.ATs || !S.Ms || !S.MsT || !S.Qx || !S.Qu || !S.Qux || !S.Qi || !S.QL || !S.Kc || !S.Phiu || !S.rn) {
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
// float64 throughout; Qx is stored unpadded n x n.  Rows with tau = 0 (inactive
// constraints) contribute nothing and are skipped.
__global__ void __launch_bounds__(256) k_sls_assemble(DevSls S, gsls_qp_t qp, const double* tau,
                                                      const double* tau_term, const float* Qbar, const float* Rbar,
                                                      const float* QbarN, long long wst) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int2 kj = S.cell_kj[cell];
  const int k = kj.x, j = kj.y;
  const int n = S.n, m = S.m, c = S.c, nf = S.nf, N = S.N;
  const size_t cb = (size_t)inst * S.ncell + cell;
  double* Qx = S.Qx + cb * n * n;
  const bool term = (k == N);
  const int rows = term ? nf : c;
  extern __shared__ double smd[];
  double* Cw = smd;                 // active rows: tau_r * C_r      (rows x n)
  double* Cr = Cw + rows * n;       // active rows: C_r              (rows x n)
  double* Dw = Cr + rows * n;       // tau_r * D_r                   (rows x m)
  double* Dr = Dw + rows * m;       // D_r
  int* act = reinterpret_cast<int*>(Dr + rows * m);
  __shared__ int s_nact;
  const float* Cg = term ? qp.CN + (size_t)inst * nf * n : qp.C + ((size_t)inst * N + k) * c * n;
  const float* Dg = term ? nullptr : qp.D + ((size_t)inst * N + k) * c * m;
  const double* tg = term ? (tau_term ? tau_term + ((size_t)inst * N + j) * nf : nullptr)
                          : (tau ? tau + cb * c : nullptr);
  if (threadIdx.x == 0) {
    int na = 0;
    if (tg)
      for (int r = 0; r < rows; ++r)
        if (tg[r] != 0.0) act[na++] = r;
    s_nact = na;
  }
  __syncthreads();
  const int na = s_nact;
  for (int e = threadIdx.x; e < na * n; e += blockDim.x) {
    const int a = S.fd_n.div(e), i = e - a * n, r = act[a];
    const double v = Cg[r * n + i];
    Cr[e] = v;
    Cw[e] = tg[r] * v;
  }
  if (!term)
    for (int e = threadIdx.x; e < na * m; e += blockDim.x) {
      const int a = S.fd_m.div(e), i = e - a * m, r = act[a];
      const double v = Dg[r * m + i];
      Dr[e] = v;
      Dw[e] = tg[r] * v;
    }
  __syncthreads();
  const float* Qb = term ? QbarN + (size_t)inst * wst * n * n : Qbar + (size_t)inst * wst * n * n;
  // 1x4 tiles over columns c, c + q4, c + 2 q4, c + 3 q4: a warp stores whole runs of a Qx
  // row (4 adjacent columns per lane wrote one 8-byte word per 32-byte sector per store)
  const int q4 = (n + 3) >> 2;
  for (int e = threadIdx.x; e < n * q4; e += blockDim.x) {
    const int i = S.fd_q4.div(e), c0 = e - i * q4;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int a = 0; a < na; ++a) {
      const double w = Cw[a * n + i];
      const double* cr = Cr + a * n + c0;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (c0 + t * q4 < n) acc[t] = fma(w, cr[t * q4], acc[t]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int jj = c0 + t * q4;
      if (jj < n) Qx[i * n + jj] = acc[t] + (double)Qb[i * n + jj];
    }
  }
  if (term) return;
  const float* Rb = Rbar + (size_t)inst * wst * m * m;
  double* Qu = S.Qu + cb * m * m;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int a = S.fd_m.div(e), b2 = e - a * m;
    double s = 0.0;
    for (int r = 0; r < na; ++r) s = fma(Dw[r * m + a], Dr[r * m + b2], s);
    Qu[e] = s + (double)Rb[e];
  }
  double* Qux = S.Qux + cb * m * n;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int a = S.fd_n.div(e), i = e - a * n;
    double s = 0.0;
    for (int r = 0; r < na; ++r) s = fma(Dw[r * m + a], Cr[r * n + i], s);
    Qux[e] = s;
  }
}

// Grid leaves (float64 algebra, float32 result): Qu^-1, P = Qx - Qux' Qu^-1 Qux,
// A = A_k - B_k Qu^-1 Qux, C = B_k Qu^-1 B_k'.  1x4 output tiles.
// L2 prefetch of a contiguous operand that a kernel reads only after its first phase
// (one bulk request from one thread; the range is widened to 16-byte alignment).
__device__ inline void prefetch_l2(const void* p, size_t bytes) {
  const unsigned long long a = (unsigned long long)p & ~15ull;
  const unsigned long long e = ((unsigned long long)p + bytes + 15ull) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}

// The leaves' m x m SPD inverses (sls.py:258-261 via lqr.spd_inverse, lqr.py:185-220), one
// warp per cell and eight cells per CTA, ahead of k_sls_leaf: inside the leaf kernel the
// one-warp inverse held the other seven warps at a barrier (40 % of its stall samples).
// Writes Qu^-1 and L^-1 (Qu = L L', the factor the factored tree uses) per cell.
__global__ void __launch_bounds__(256) k_sls_qu_inverse(DevSls S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cell = blockIdx.x * 8 + warp, inst = blockIdx.y;
  const int m = S.m;
  const int ld = m + 1, xoff = m * ld;  // the inverse's workspace: L, X = L^-1 (ld m + 1)
  extern __shared__ double smq[];
  double* Qu = smq + warp * (m * m + 2 * xoff + 8);
  double* wk = Qu + m * m;
  const bool live = cell < S.ncell && S.cell_kj[cell].x < S.N;  // terminal cells have no inverse
  if (!live) return;  // warp-uniform
  const size_t cb = (size_t)inst * S.ncell + cell;
  for (int e = lane; e < m * m; e += 32) Qu[e] = S.Qu[cb * m * m + e];
  __syncwarp();
  double* Qi = S.Qi + cb * m * m;
  if (warp_spd_inverse(Qu, m, Qi, m, wk, ld, xoff) && lane == 0) {
    const int2 kj = S.cell_kj[cell];
    raise_err(S.err + inst, GSLS_ERR_SINGULAR_STAGE, kj.x, kj.y, GSLS_LABEL_QU);
  }
  __syncwarp();
  double* QL = S.QL + cb * m * m;
  for (int e = lane; e < m * m; e += 32) {
    const int a = e / m, b = e - a * m;
    QL[e] = (b <= a) ? wk[xoff + a * ld + b] : 0.0;
  }
}

// 4 CTAs per SM (<= 64 registers): 40 % of the warps' time is the wait for the one-warp
// inverse, so the extra resident CTA pays (21.3 vs 23.2 ms at B = 1024; 5 CTAs spill)
__global__ void __launch_bounds__(256, 4) k_sls_leaf(DevSls S, gsls_qp_t qp) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int2 kj = S.cell_kj[cell];
  const int k = kj.x, j = kj.y;
  const int n = S.n, m = S.m, N = S.N, ldg = S.ldg;
  const size_t MS = (size_t)n * ldg;
  const int slot = cell;  // leaves occupy slots [0, ncell)
  float* Pd = S.Ps + ((size_t)inst * S.cvf_nslots + slot) * MS;
  float* Ad = S.As + ((size_t)inst * S.cvf_nslots + slot) * MS;
  float* ATd = S.ATs + ((size_t)inst * S.cvf_nslots + slot) * MS;
  float* Cd = S.Cs + ((size_t)inst * S.cvf_nslots + slot) * MS;
  const size_t cb = (size_t)inst * S.ncell + cell;
  const double* Qx = S.Qx + cb * n * n;
  if (k == N) {  // terminal element (Qx_term, 0, 0)
    for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) {
      const int i = S.fd_ldg.div(e), jj = e - i * ldg;
      Pd[e] = (jj < n) ? (float)Qx[i * n + jj] : 0.f;
      Ad[e] = 0.f;
      ATd[e] = 0.f;
      Cd[e] = 0.f;
    }
    return;
  }
  const size_t st = (size_t)inst * N + k;
  if (threadIdx.x == 0) {  // the epilogue's operands, read after the inverse and the products
    prefetch_l2(Qx, (size_t)n * n * sizeof(double));
    prefetch_l2(qp.A + st * n * n, (size_t)n * n * sizeof(float));
  }
  extern __shared__ double smd[];
  const int np = ldg;                // row length of the n-vectors below (padded, zero tail)
  double* Qu = smd;                  // m x m
  double* Qi = Qu + m * m;           // m x m
  double* Qux = Qi + m * m;          // m x np
  double* QQ = Qux + m * np;         // m x np   Qu^-1 Qux
  double* BT = QQ + m * np;          // m x np   B_k^T
  double* BQT = BT + m * np;         // m x ldq  (B_k Qu^-1)^T
  const int ldq = np + 1;            // odd: the factored epilogue reads BQT by column (16 rows a warp)
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {  // Qu^-1 and L^-1 from k_sls_qu_inverse
    Qi[e] = S.Qi[cb * m * m + e];
    Qu[e] = S.QL[cb * m * m + e];  // (the Qu buffer holds L^-1 here)
  }
  const float* Bg = qp.B + st * n * m;
  for (int e = threadIdx.x; e < m * np; e += blockDim.x) {
    const int l = S.fd_ldg.div(e), i = e - l * np;
    Qux[e] = (i < n) ? S.Qux[cb * m * n + l * n + i] : 0.0;
    BT[e] = (i < n) ? (double)Bg[i * m + l] : 0.0;
  }
  __syncthreads();
  const int dead = S.leaf_dead[cell];  // parts of this leaf no combine reads (scan-plan analysis)
  // C = B Qu^-1 B' is stored as the factor F = B L^-T (Qu = L L', L^-1 left in the
  // inverse's work area) when the plan carries it factored (lowrank.cuh): BQT then
  // holds F' = L^-1 B' instead of (B Qu^-1)'
  const bool cfac = (dead & 8) != 0;
  const double* Linv = Qu;  // m x m, row-major (ld m)
  for (int e = threadIdx.x; e < m * np; e += blockDim.x) {
    const int a = S.fd_ldg.div(e), i = e - a * np;
    double s1 = 0.0, s2 = 0.0;
    for (int b2 = 0; b2 < m; ++b2) {
      const double qi = Qi[b2 * m + a];  // Qi symmetric in exact arithmetic; use Qi^T consistently
      s1 = fma(qi, Qux[b2 * np + i], s1);
      if (!cfac) s2 = fma(qi, BT[b2 * np + i], s2);
    }
    if (cfac)
      for (int b2 = 0; b2 <= a; ++b2) s2 = fma(Linv[a * m + b2], BT[b2 * np + i], s2);
    QQ[e] = s1;
    BQT[a * ldq + i] = s2;
  }
  __syncthreads();
  const float* Ak = qp.A + st * n * n;
  // 1x4 tiles over columns c, c + q4, c + 2 q4, c + 3 q4: a warp's lanes read consecutive
  // doubles of a row (the 4-wide column tiles put lanes 32 bytes apart: 2x the shared
  // wavefronts, the kernel being shared-memory bound)
  const int q4 = np >> 2;
  auto epilogue = [&](int i, int jj, double p, double a, double cc) {
    const bool in = jj < n;
    const float po = in ? (float)(Qx[i * n + jj] - p) : 0.f;
    const float ao = in ? (float)((double)Ak[i * n + jj] - a) : 0.f;
    const float co = cfac ? (jj < m ? (float)BQT[jj * ldq + i] : 0.f) : (in ? (float)cc : 0.f);
    if (in && !(dead & 2)) ATd[(size_t)jj * ldg + i] = ao;
    Pd[(size_t)i * ldg + jj] = po;
    if (!(dead & 1)) Ad[(size_t)i * ldg + jj] = ao;
    if (!(dead & 4)) Cd[(size_t)i * ldg + jj] = co;
  };
  if (cfac) {  // C comes from BQT directly: 2x4 tiles (rows i, i + nh), one QQ row load feeds both
    const int nh = (n + 1) >> 1;
    for (int e = threadIdx.x; e < nh * q4; e += blockDim.x) {
      const int i = S.fd_q4.div(e), c0 = e - i * q4;
      const bool two = i + nh < n;
      const int i1 = two ? i + nh : i;
      double p0[4] = {0.0, 0.0, 0.0, 0.0}, a0[4] = {0.0, 0.0, 0.0, 0.0};
      double p1[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
      for (int l = 0; l < m; ++l) {
        const double qx0 = Qux[l * np + i], bt0 = BT[l * np + i];
        const double qx1 = Qux[l * np + i1], bt1 = BT[l * np + i1];
        const double* qr = QQ + l * np + c0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const double qq = qr[t * q4];
          p0[t] = fma(qx0, qq, p0[t]);
          a0[t] = fma(bt0, qq, a0[t]);
          p1[t] = fma(qx1, qq, p1[t]);
          a1[t] = fma(bt1, qq, a1[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        epilogue(i, c0 + t * q4, p0[t], a0[t], 0.0);
        if (two) epilogue(i1, c0 + t * q4, p1[t], a1[t], 0.0);
      }
    }
    return;
  }
  for (int e = threadIdx.x; e < n * q4; e += blockDim.x) {
    const int i = S.fd_q4.div(e), c0 = e - i * q4;
    double p4[4] = {0.0, 0.0, 0.0, 0.0}, a4[4] = {0.0, 0.0, 0.0, 0.0}, c4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int l = 0; l < m; ++l) {
      const double qx = Qux[l * np + i], bt = BT[l * np + i], bq = BQT[l * ldq + i];
      const double* qr = QQ + l * np + c0;
      const double* br = BT + l * np + c0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double qq = qr[t * q4];
        p4[t] = fma(qx, qq, p4[t]);
        a4[t] = fma(bt, qq, a4[t]);
        c4[t] = fma(bq, br[t * q4], c4[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) epilogue(i, c0 + t * q4, p4[t], a4[t], c4[t]);
  }
}

// Gains on cell (k, j), k <= N-1, from P+ = P(k+1, j); closed loop -> product
// leaf of position k (float64 algebra, 1x4 tiles).  Cell (N, j) writes E_j into
// the leaf of position j.
__global__ void __launch_bounds__(256, 4) k_sls_gains(DevSls S, gsls_qp_t qp, const float* E) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int2 kj = S.cell_kj[cell];
  const int k = kj.x, j = kj.y;
  const int n = S.n, m = S.m, N = S.N, ldg = S.ldg;
  const size_t MS = (size_t)n * ldg;
  float* Mbase = S.Ms + (size_t)inst * S.mp_nslots * MS;
  float* MTbase = S.MsT + (size_t)inst * S.mp_nslots * MS;
  if (k == N) {
    float* Ml = Mbase + (size_t)(cell_of(N, j + 1, j) - S.cell0) * MS;
    float* MTl = MTbase + (size_t)(cell_of(N, j + 1, j) - S.cell0) * MS;
    const float* Ej = E + ((size_t)inst * N + j) * n * n;
    for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) {
      const int i = S.fd_ldg.div(e), jj = e - i * ldg;
      Ml[e] = (jj < n) ? Ej[i * n + jj] : 0.f;
      MTl[e] = (jj < n) ? Ej[jj * n + i] : 0.f;
    }
    return;
  }
  extern __shared__ double smd[];
  // B' and B'P+ rows at an odd stride: H = (B'P+) B reads 12 rows of B' and 3 of B'P+
  // per warp, all in one bank at an even stride
  const int np = ldg, lds = lds_of(n), ldb = np + 1;
  // shared memory for 4 CTAs per SM (56.7 KB at 61/12): K overwrites B'P+ (dead once G is
  // formed) and the inverse's workspace is sized for m
  double* BT = smd;              // m x ldb  B_k^T
  double* BtP = BT + m * ldb;    // m x ldb  B' P+, then K
  double* Gm = BtP + m * ldb;    // m x np
  double* Ks = BtP;
  double* H = Gm + m * np;       // m x m
  double* Ga = H + m * m;        // m x m
  double* wk = Ga + m * m;       // 2 m (m + 1) (+ 8): the inverse's L and X
  float* Pn = reinterpret_cast<float*>(wk + 2 * m * (m + 1) + 8);  // n x lds
  float* Ak = Pn + n * lds;                                                // n x lds
  const float* Pg = S.Ps + ((size_t)inst * S.cvf_nslots + S.cvf_out[cell_of(N, k + 1, j) - S.cell0]) * MS;
  if (threadIdx.x == 0) {  // Qu, Qux: read after the B' P+ product
    const size_t cbp = (size_t)inst * S.ncell + cell;
    prefetch_l2(S.Qu + cbp * m * m, (size_t)m * m * sizeof(double));
    prefetch_l2(S.Qux + cbp * m * n, (size_t)m * n * sizeof(double));
  }
  cta_load_async(Pn, lds, Pg, n);
  const size_t st = (size_t)inst * N + k;
  const float* Bg = qp.B + st * n * m;
  const float* Ag = qp.A + st * n * n;
  for (int e = threadIdx.x; e < n * np; e += blockDim.x) {  // A_k: 4-byte async copies (rows of n floats)
    const int i = S.fd_ldg.div(e), jj = e - i * np;
    if (jj < n) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(Ak + i * lds + jj);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(Ag + i * n + jj) : "memory");
    } else {
      Ak[i * lds + jj] = 0.f;
    }
  }
  cp_async_commit();
  for (int e = threadIdx.x; e < m * np; e += blockDim.x) {
    const int l = S.fd_ldg.div(e), i = e - l * np;
    BT[l * ldb + i] = (i < n) ? (double)Bg[i * m + l] : 0.0;
  }
  cp_async_wait<0>();
  __syncthreads();
  // The products below are register-blocked two or four rows deep: the kernel is bound by
  // shared-memory wavefronts, and a row of the right operand loaded once feeds every row of
  // the tile.  Each element keeps its own ascending fma chain.
  const int q4 = np >> 2, mh = (m + 1) >> 1;
  for (int e = threadIdx.x; e < mh * q4; e += blockDim.x) {  // B' P+ (2x4 tiles: rows l, l + mh)
    const int l = S.fd_q4.div(e), j0 = (e - l * q4) << 2;
    const int l1 = l + mh < m ? l + mh : l;
    double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < n; ++i) {
      const double b0 = BT[l * ldb + i], b1 = BT[l1 * ldb + i];
      const float4 pv = *reinterpret_cast<const float4*>(Pn + i * lds + j0);
      const double p4[4] = {(double)pv.x, (double)pv.y, (double)pv.z, (double)pv.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a0[t] = fma(b0, p4[t], a0[t]);
        a1[t] = fma(b1, p4[t], a1[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      BtP[l * ldb + j0 + t] = a0[t];
      BtP[l1 * ldb + j0 + t] = (l1 != l) ? a1[t] : a0[t];
    }
  }
  __syncthreads();
  const size_t cb = (size_t)inst * S.ncell + cell;
  const double* Qu = S.Qu + cb * m * m;
  const double* Qux = S.Qux + cb * m * n;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int l = S.fd_m.div(e), t = e - l * m;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = fma(BtP[l * ldb + i], BT[t * ldb + i], s);
    H[e] = Qu[e] + s;
  }
  __syncthreads();
  // warp 0 inverts H while warps 1.. form G = Qux + B' P+ A (independent of the inverse)
  if (threadIdx.x < 32) {
    if (warp_spd_inverse(H, m, Ga, m, wk, m + 1, m * (m + 1)) && threadIdx.x == 0)
      raise_err(S.err + inst, GSLS_ERR_SINGULAR_STAGE, k, j, GSLS_LABEL_QU_BPB);
  }
  for (int e = (int)threadIdx.x - 32; e >= 0 && e < mh * q4; e += (int)blockDim.x - 32) {  // 2x4 tiles
    const int l = S.fd_q4.div(e), j0 = (e - l * q4) << 2;
    const int l1 = l + mh < m ? l + mh : l;
    double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < n; ++i) {
      const double b0 = BtP[l * ldb + i], b1 = BtP[l1 * ldb + i];
      const float4 av = *reinterpret_cast<const float4*>(Ak + i * lds + j0);
      const double v4[4] = {(double)av.x, (double)av.y, (double)av.z, (double)av.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a0[t] = fma(b0, v4[t], a0[t]);
        a1[t] = fma(b1, v4[t], a1[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int jj = j0 + t;
      Gm[l * np + jj] = (jj < n) ? Qux[l * n + jj] + a0[t] : 0.0;
      if (l1 != l) Gm[l1 * np + jj] = (jj < n) ? Qux[l1 * n + jj] + a1[t] : 0.0;
    }
  }
  __syncthreads();
  float* Kg = S.Kc + cb * m * n;
  const int mq = (m + 3) >> 2;
  for (int e = threadIdx.x; e < mq * np; e += blockDim.x) {  // K = -H^-1 G, rows l + r mq (r < 4)
    const int l = S.fd_ldg.div(e), jj = e - l * np;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int t = 0; t < m; ++t) {
      const double g = Gm[t * np + jj];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (l + r * mq < m) s[r] = fma(Ga[(l + r * mq) * m + t], g, s[r]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int lr = l + r * mq;
      if (lr < m) {
        Ks[lr * ldb + jj] = -s[r];
        if (jj < n) Kg[lr * n + jj] = (float)(-s[r]);
      }
    }
  }
  __syncthreads();
  float* Ml = Mbase + (size_t)(cell_of(N, k + 1, j) - S.cell0) * MS;  // product leaf of position k
  float* MTl = MTbase + (size_t)(cell_of(N, k + 1, j) - S.cell0) * MS;
  // A + B K, 1x4 tiles over columns c, c + q4, c + 2 q4, c + 3 q4 (lanes on consecutive
  // doubles of a K row; 4-wide column tiles put them 32 bytes apart)
  // rows i and i + nh of each 2x4 tile
  const int nh = (n + 1) >> 1;
  for (int e = threadIdx.x; e < nh * q4; e += blockDim.x) {
    const int i = S.fd_q4.div(e), c0 = e - i * q4;
    const bool two = i + nh < n;
    const int i1 = two ? i + nh : i;
    double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
    for (int l = 0; l < m; ++l) {
      const double b0 = BT[l * ldb + i], b1 = BT[l * ldb + i1];
      const double* kr = Ks + l * ldb + c0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double kv = kr[t * q4];
        a0[t] = fma(b0, kv, a0[t]);
        a1[t] = fma(b1, kv, a1[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int jj = c0 + t * q4;
      const float o0 = (jj < n) ? (float)((double)Ak[i * lds + jj] + a0[t]) : 0.f;
      if (jj < n) Pn[jj * lds + i] = o0;  // transpose staged in smem (P+ is dead here)
      Ml[(size_t)i * ldg + jj] = o0;
      if (two) {
        const float o1 = (jj < n) ? (float)((double)Ak[i1 * lds + jj] + a1[t]) : 0.f;
        if (jj < n) Pn[jj * lds + i1] = o1;
        Ml[(size_t)i1 * ldg + jj] = o1;
      }
    }
  }
  __syncthreads();
  // M^T rows: coalesced 16-byte stores instead of one scattered store per element
  for (int e = threadIdx.x; e < n * q4; e += blockDim.x) {
    const int jj = S.fd_q4.div(e), i0 = (e - jj * q4) << 2;
    const float4 p = *reinterpret_cast<const float4*>(Pn + jj * lds + i0);
    const float v[4] = {p.x, i0 + 1 < n ? p.y : 0.f, i0 + 2 < n ? p.z : 0.f, i0 + 3 < n ? p.w : 0.f};
    *reinterpret_cast<float4*>(MTl + (size_t)jj * ldg + i0) = make_float4(i0 < n ? v[0] : 0.f, v[1], v[2], v[3]);
  }
}

// k_matprod threads: one per 8 x 4 tile of the padded product (gemm_tn84), >= 2 warps.
static int matprod_threads(int n) {
  const int np = ldg_of(n), tiles = ((np + 7) / 8) * (np / 4);
  return std::max(64, std::min(512, (tiles + 31) / 32 * 32));
}

// Matrix-product combine: M = M_later M_earlier (sls.py:217-218), both orientations.
__global__ void __launch_bounds__(512) k_matprod(float* Ms, float* MsT, long long inst_stride, int n, const int4* ops) {
  const int inst = blockIdx.y;
  const int4 op = ops[blockIdx.x];
  const int ldg = ldg_of(n), lds = lds_of(n);
  const size_t MS = (size_t)n * ldg;
  extern __shared__ float sm[];
  float* Lt = sm;
  float* Er = Lt + (size_t)n * lds;
  float* base = Ms + (size_t)inst * inst_stride;
  float* baseT = MsT + (size_t)inst * inst_stride;
  cta_load_async(Lt, lds, baseT + (size_t)op.z * MS, n);
  cta_load_async(Er, lds, base + (size_t)op.y * MS, n);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  // plan .w = 1: no later product reads this slot, so its transposed copy is dead
  gemm_tn84(n, Lt, Er, lds, EpiGlobal{base + (size_t)op.x * MS, nullptr, ldg, n, (op.w & 1) ? nullptr : baseT + (size_t)op.x * MS});
}

// Phi^u_{k,j} = K_{k,j} Phi^x_{k,j} (sls.py:310-318).
__global__ void __launch_bounds__(256) k_sls_phiu(DevSls S) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int k = S.cell_kj[cell].x;
  if (k >= S.N) return;
  const int n = S.n, m = S.m, ldg = S.ldg;
  const size_t MS = (size_t)n * ldg;
  extern __shared__ float sm[];
  float* Px = sm;
  const float* Pg = S.Ms + ((size_t)inst * S.mp_nslots + S.mp_out[cell]) * MS;
  const size_t cb = (size_t)inst * S.ncell + cell;
  const float* Kg = S.Kc + cb * m * n;
  float* Pug = S.Phiu + cb * m * n;
  float* Ks = Px + n * ldg;  // K staged in smem (m x n)
  // 16-byte async copies of the contiguous blocks (K's per-cell blocks are 16-byte aligned
  // when m n is a multiple of 4; otherwise plain loads)
  for (int e = threadIdx.x; e < (n * ldg) >> 2; e += blockDim.x) cp_async16(Px + 4 * e, Pg + 4 * e);
  if (((m * n) & 3) == 0)
    for (int e = threadIdx.x; e < (m * n) >> 2; e += blockDim.x) cp_async16(Ks + 4 * e, Kg + 4 * e);
  else
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) Ks[e] = Kg[e];
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  // Phi^u = K Phi^x: thread task = (rows a and a + mh, columns c, c + q4, c + 2 q4, c + 3 q4):
  // two broadcast K values and four consecutive-lane Phi^x loads per l, and whole warp runs
  // of a Phi^u row per store (each element keeps its ascending fma chain)
  const int q4 = ldg >> 2, mh = (m + 1) >> 1;
  for (int t = threadIdx.x; t < mh * q4; t += blockDim.x) {
    const int a = t / q4, c0 = t - a * q4;
    const bool two = a + mh < m;
    const int a1 = two ? a + mh : a;
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
    for (int l = 0; l < n; ++l) {
      const float k0 = Ks[a * n + l], k1 = Ks[a1 * n + l];
      const float* pr = Px + l * ldg + c0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float p = pr[q * q4];
        s0[q] = fmaf(k0, p, s0[q]);
        s1[q] = fmaf(k1, p, s1[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = c0 + q * q4;
      if (i < n) {
        Pug[a * n + i] = s0[q];
        if (two) Pug[a1 * n + i] = s1[q];
      }
    }
  }
}

// Row norms of C_k Phi^x + D_k Phi^u (terminal cells: CN Phi^x), sls.py:146-147, :167, :336, :340.
__global__ void __launch_bounds__(256, 5) k_sls_rownorm(DevSls S, gsls_qp_t qp) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int k = S.cell_kj[cell].x;
  const int n = S.n, m = S.m, c = S.c, nf = S.nf, N = S.N, ldg = S.ldg;
  const size_t MS = (size_t)n * ldg;
  extern __shared__ float sm[];
  float* Px = sm;            // n x ldg
  float* Pu = Px + n * ldg;  // m x ldg (zero beyond n: 16-byte row loads)
  const float* Pg = S.Ms + ((size_t)inst * S.mp_nslots + S.mp_out[cell]) * MS;
  const size_t cb = (size_t)inst * S.ncell + cell;
  for (int e = threadIdx.x; e < (n * ldg) >> 2; e += blockDim.x) cp_async16(Px + 4 * e, Pg + 4 * e);
  cp_async_commit();
  if (k < N)
    for (int e = threadIdx.x; e < m * ldg; e += blockDim.x) {
      const int a = S.fd_ldg.div(e), i = e - a * ldg;
      Pu[e] = i < n ? S.Phiu[cb * m * n + a * n + i] : 0.f;
    }
  cp_async_wait<0>();
  __syncthreads();
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
  const size_t st = (size_t)inst * N + k;
  const float* Ck = qp.C + st * c * n;
  const float* Dk = qp.D + st * c * m;
  // C_k, D_k staged in smem; thread task = (rows r and r + ch, 4 columns): 8 independent
  // FMA chains per l from two broadcast C values and one 16-byte Phi^x row load (the
  // kernel is bound by shared-memory wavefronts)
  float* Cs = Pu + m * ldg;        // c x n
  float* Ds = Cs + c * n;          // c x m
  const int poff = (n * ldg + m * ldg + c * n + c * m + 1) & ~1;      // 8-byte aligned
  double* part = reinterpret_cast<double*>(sm + poff);              // c x q4 partial sums of squares
  for (int e = threadIdx.x; e < c * n; e += blockDim.x) Cs[e] = Ck[e];
  for (int e = threadIdx.x; e < c * m; e += blockDim.x) Ds[e] = Dk[e];
  __syncthreads();
  const int q4 = ldg >> 2, ch = (c + 1) >> 1;
  for (int t = threadIdx.x; t < ch * q4; t += blockDim.x) {
    const int r = t / q4, i0 = (t - r * q4) << 2;
    const bool two = r + ch < c;
    const int r1 = two ? r + ch : r;
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, u0[4] = {0.f, 0.f, 0.f, 0.f};
    float s1[4] = {0.f, 0.f, 0.f, 0.f}, u1[4] = {0.f, 0.f, 0.f, 0.f};
    for (int l = 0; l < n; ++l) {
      const float c0 = Cs[r * n + l], c1 = Cs[r1 * n + l];
      const float4 p = *reinterpret_cast<const float4*>(Px + l * ldg + i0);
      const float pv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        s0[q] = fmaf(c0, pv[q], s0[q]);
        s1[q] = fmaf(c1, pv[q], s1[q]);
      }
    }
    for (int a = 0; a < m; ++a) {
      const float d0 = Ds[r * m + a], d1 = Ds[r1 * m + a];
      const float4 p = *reinterpret_cast<const float4*>(Pu + a * ldg + i0);
      const float pv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        u0[q] = fmaf(d0, pv[q], u0[q]);
        u1[q] = fmaf(d1, pv[q], u1[q]);
      }
    }
    double ss0 = 0.0, ss1 = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + q < n) {
        const double v0 = (double)(s0[q] + u0[q]), v1 = (double)(s1[q] + u1[q]);
        ss0 += v0 * v0;
        ss1 += v1 * v1;
      }
    part[r * q4 + (i0 >> 2)] = ss0;
    if (two) part[r1 * q4 + (i0 >> 2)] = ss1;
  }
  __syncthreads();
  for (int r = warp; r < c; r += nw) {
    double ss = 0.0;
    for (int q = lane; q < q4; q += 32) ss += part[r * q4 + q];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) rn[r] = sqrt(ss);
  }
}

// Response import (cell layout, unpadded) for responses built elsewhere.
__global__ void k_sls_import(DevSls S, const float* phix, const float* phiu) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int n = S.n, m = S.m, ldg = S.ldg;
  const size_t cb = (size_t)inst * S.ncell + cell;
  float* dst = S.Ms + ((size_t)inst * S.mp_nslots + S.mp_out[cell]) * n * ldg;
  for (int e = threadIdx.x; e < n * ldg; e += blockDim.x) {
    const int i = e / ldg, j = e - i * ldg;
    dst[e] = (j < n) ? phix[cb * n * n + i * n + j] : 0.f;
  }
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) S.Phiu[cb * m * n + e] = phiu[cb * m * n + e];
}

// h_k = sum_{j<k} rownorm(k, j) (k >= 1; h_0 = 0); hf = sum_j rownorm(N, j).
__global__ void k_sls_tighten(DevSls S, double* h, double* hf) {
  const int inst = blockIdx.x;
  const int c = S.c, nf = S.nf, N = S.N;
  const double* rn = S.rn + (size_t)inst * S.ncell * S.cmax;
  for (int e = threadIdx.x; e < N * c; e += blockDim.x) {
    const int k = e / c, r = e - k * c;
    double s = 0.0;
    for (int j = S.j0; j < min(k, S.j1); ++j) s += rn[(size_t)(cell_of(N, k, j) - S.cell0) * S.cmax + r];
    h[(size_t)inst * N * c + e] = s;
  }
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    double s = 0.0;
    for (int j = S.j0; j < S.j1; ++j) s += rn[(size_t)(cell_of(N, N, j) - S.cell0) * S.cmax + f];
    hf[(size_t)inst * nf + f] = s;
  }
}

// tau = max(lam, 0) / sqrt(beta + eps), beta = rownorm^2 (0 without a response).
// lam is the stacked ADMM multiplier (B, N*nc + nf) (admm.py:82-88).
__global__ void k_sls_duals(DevSls S, const double* lam, double eps, double* tau, double* tau_term, double* beta,
                            double* beta_term) {
  const int inst = blockIdx.x;
  const int c = S.c, nf = S.nf, N = S.N;
  const double* lam_s = lam + (size_t)inst * (N * c + nf);
  const double* lam_t = lam_s + (size_t)N * c;
  const double* rn = S.rn + (size_t)inst * S.ncell * S.cmax;
  for (int e = threadIdx.x; e < S.ncell * c; e += blockDim.x) {
    const int cell = e / c, r = e - cell * c;
    const int2 kj = S.cell_kj[cell];
    if (kj.x >= N) continue;
    const double v = S.have_response ? rn[(size_t)cell * S.cmax + r] : 0.0;
    const double b = v * v;
    const double l = fmax(lam_s[(size_t)kj.x * c + r], 0.0);
    const size_t o = ((size_t)inst * S.ncell + cell) * c + r;
    tau[o] = l / sqrt(b + eps);
    if (beta) beta[o] = b;
  }
  for (int e = threadIdx.x; e < N * nf; e += blockDim.x) {
    const int j = e / nf, f = e - j * nf;
    if (j < S.j0 || j >= S.j1) continue;  // terminal cells of other shards' columns
    const double v = S.have_response ? rn[(size_t)(cell_of(N, N, j) - S.cell0) * S.cmax + f] : 0.0;
    const double b = v * v;
    const double l = fmax(lam_t[f], 0.0);
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
  const size_t rows = (size_t)S.cmax;
  const size_t sb = (rows * (2 * S.n + 2 * S.m)) * sizeof(double) + rows * sizeof(int) + 16;
  int rc2 = smem_attr((const void*)k_sls_assemble, sb);
  if (rc2) return rc2;
  ProfScope ps(P_SLS_ASSEMBLE, st, (double)S.ncell * c->dims.batch);
  k_sls_assemble<<<dim3(S.ncell, c->dims.batch), 256, sb, st>>>(S, *qp, tau, tau_term, Qbar, Rbar, QbarN,
                                                                  weights_per_instance ? 1 : 0);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

// Explicit costs (cell layout, unpadded): Qx (B,ncell,n,n) with Qx_term on k = N
// cells, Qu (B,ncell,m,m), Qux (B,ncell,m,n).
__global__ void k_sls_set_costs(DevSls S, const double* Qx, const double* Qu, const double* Qux) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int n = S.n, m = S.m;
  const size_t cb = (size_t)inst * S.ncell + cell;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) S.Qx[cb * n * n + e] = Qx[cb * n * n + e];
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) S.Qu[cb * m * m + e] = Qu[cb * m * m + e];
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) S.Qux[cb * m * n + e] = Qux[cb * m * n + e];
}

int sls_set_costs(Ctx* c, const double* Qx, const double* Qu, const double* Qux, cudaStream_t st) {
  int rc = sls_init(c);
  if (rc) return rc;
  DevSls& S = sls_of(c)->dev;
  k_sls_set_costs<<<dim3(S.ncell, c->dims.batch), 256, 0, st>>>(S, Qx, Qu, Qux);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

static int sls_synthesize_once(Ctx* c, const gsls_qp_t* qp, const float* E, cudaStream_t st);

// A factored combine that met an indefinite P (GSLS_ERR_LOWRANK) switches the tree to
// dense combines; the synthesis is then re-run once.
int sls_synthesize(Ctx* c, const gsls_qp_t* qp, const float* E, cudaStream_t st, bool check) {
  int rc = sls_synthesize_once(c, qp, E, st);
  if (rc || !check) return rc;
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  GSLS_CUDA_CHECK(cudaStreamIsCapturing(st, &cst));
  if (cst != cudaStreamCaptureStatusNone) return GSLS_OK;  // captured step: errors are read after the graph
  rc = check_errors(c, st, "sls.synthesize");
  if (rc == GSLS_ERR_LOWRANK) {
    rc = sls_synthesize_once(c, qp, E, st);
    if (!rc) rc = check_errors(c, st, "sls.synthesize");
  }
  return rc;
}

static int sls_synthesize_once(Ctx* c, const gsls_qp_t* qp, const float* E, cudaStream_t st) {
  int rc = sls_init(c);
  if (rc) return rc;
  SlsState* s = sls_of(c);
  DevSls& S = s->dev;
  const int B = c->dims.batch, n = S.n, m = S.m, ldg = S.ldg;
  const size_t MS = mat_elems(n);
  const size_t wk = 2 * kMaxM * (kMaxM + 1) + 8;
  {
    const size_t sbq = 8 * (size_t)(m * m + 2 * m * (m + 1) + 8) * sizeof(double);
    const size_t sb = (2 * m * m + 4 * (size_t)m * ldg + m) * sizeof(double);  // + BQT's odd stride
    if ((rc = smem_attr((const void*)k_sls_leaf, sb))) return rc;
    if ((rc = smem_attr((const void*)k_sls_qu_inverse, sbq))) return rc;
    ProfScope ps(P_SLS_LEAF, st, (double)S.ncell * B);
    k_sls_qu_inverse<<<dim3((S.ncell + 7) / 8, B), 256, sbq, st>>>(S);
    k_sls_leaf<<<dim3(S.ncell, B), 256, sb, st>>>(S, *qp);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  for (int l = 0; l < s->cvf.layers; ++l) {
    const int o0 = s->cvf.layer_off[l], o1 = s->cvf.layer_off[l + 1];
    CombineArgs a{n, S.cvf_ops + o0, o0, S.Ps, S.As, S.Cs, S.ATs, (long long)S.cvf_nslots * (long long)MS, nullptr, 0,
                  nullptr, S.err, 1e-10f, 1};
    if (o1 == o0) continue;
    ProfScope ps(P_SLS_CVF, st, (double)(o1 - o0) * B);
    if ((rc = launch_combine(a, o1 - o0, B, st))) return rc;
  }
  {
    const size_t sb = (3 * (size_t)m * ldg + 2 * m + 2 * m * m + 2 * m * (m + 1) + 8) * sizeof(double) +
                      2 * (size_t)n * lds_of(n) * sizeof(float);
    if ((rc = smem_attr((const void*)k_sls_gains, sb))) return rc;
    ProfScope ps(P_SLS_GAINS, st, (double)S.ncell * B);
    k_sls_gains<<<dim3(S.ncell, B), 256, sb, st>>>(S, *qp, E);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  {
    const size_t sb = 2 * (size_t)n * lds_of(n) * sizeof(float);
    if ((rc = smem_attr((const void*)k_matprod, sb))) return rc;
    for (int l = 0; l < s->mp.layers; ++l) {
      const int o0 = s->mp.layer_off[l], o1 = s->mp.layer_off[l + 1];
      if (o1 == o0) continue;
      ProfScope ps(P_SLS_MATPROD, st, (double)(o1 - o0) * B);
      k_matprod<<<dim3(o1 - o0, B), matprod_threads(n), sb, st>>>(S.Ms, S.MsT, (long long)S.mp_nslots * (long long)MS, n,
                                                                  S.mp_ops + o0);
      GSLS_CUDA_CHECK(cudaGetLastError());
    }
  }
  {
    const size_t sb = ((size_t)n * ldg + (size_t)m * n) * sizeof(float);
    if ((rc = smem_attr((const void*)k_sls_phiu, sb))) return rc;
    ProfScope ps(P_SLS_PHIU, st, (double)S.ncell * B);
    k_sls_phiu<<<dim3(S.ncell, B), 256, sb, st>>>(S);
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  S.have_response = 1;
  return GSLS_OK;
}

static int sls_rownorms(Ctx* c, const gsls_qp_t* qp, cudaStream_t st) {
  DevSls& S = sls_of(c)->dev;
  const size_t sb = (((size_t)S.n * S.ldg + S.m * S.ldg + (size_t)S.c * S.n + S.c * S.m + 1) & ~(size_t)1) * sizeof(float) +
                    (size_t)S.c * (S.ldg / 4) * sizeof(double);
  int rc = smem_attr((const void*)k_sls_rownorm, sb);
  if (rc) return rc;
  ProfScope ps(P_SLS_ROWNORM, st, (double)S.ncell * c->dims.batch);
  k_sls_rownorm<<<dim3(S.ncell, c->dims.batch), 256, sb, st>>>(S, *qp);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

int sls_import(Ctx* c, const float* phix, const float* phiu, cudaStream_t st) {
  int rc = sls_init(c);
  if (rc) return rc;
  DevSls& S = sls_of(c)->dev;
  k_sls_import<<<dim3(S.ncell, c->dims.batch), 256, 0, st>>>(S, phix, phiu);
  GSLS_CUDA_CHECK(cudaGetLastError());
  S.have_response = 1;
  return GSLS_OK;
}

int sls_tighten(Ctx* c, const gsls_qp_t* qp, double* h, double* hf, cudaStream_t st) {
  SlsState* s = sls_of(c);
  if (!s || !s->dev.have_response) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "no SLS response in context");
    return GSLS_ERR_ARG;
  }
  int rc = sls_rownorms(c, qp, st);
  if (rc) return rc;
  ProfScope ps(P_SLS_SMALL, st, (double)c->dims.batch);
  k_sls_tighten<<<c->dims.batch, 256, 0, st>>>(s->dev, h, hf);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

int sls_duals(Ctx* c, const gsls_qp_t* qp, const double* lam, double eps, int use_response, int reuse_rownorms,
              double* tau, double* tau_term, double* beta, double* beta_term, cudaStream_t st) {
  int rc = sls_init(c);
  if (rc) return rc;
  DevSls S = sls_of(c)->dev;
  S.have_response = use_response && S.have_response;
  if (S.have_response && !reuse_rownorms && (rc = sls_rownorms(c, qp, st))) return rc;
  ProfScope ps(P_SLS_SMALL, st, (double)c->dims.batch);
  k_sls_duals<<<c->dims.batch, 256, 0, st>>>(S, lam, eps, tau, tau_term, beta, beta_term);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

// sls.sls_cost (sls.py:344-358): sum over the response's cells of ||L' Phi||_F^2 with
// W = L L' the cell's weight (Qbar for Phi^x_{k,j}, k < N; QbarN at k = N; Rbar for
// Phi^u), i.e. tr(Phi' W Phi).  One CTA per (cell, instance) writes the cell's term in
// float64 (Phi read from the synthesis storage); a second pass sums each instance's
// cells in cell order (deterministic).
__global__ void __launch_bounds__(256) k_sls_cost_cells(DevSls S, const double* Qbar, const double* Rbar,
                                                        const double* QbarN, double* cells) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int n = S.n, m = S.m, ldg = S.ldg, N = S.N;
  const int k = S.cell_kj[cell].x;
  const size_t cb = (size_t)inst * S.ncell + cell;
  extern __shared__ double smc[];
  double* W = smc;            // n x n
  double* F = W + n * n;      // n x n   Phi^x (then Phi^u rows in the first m rows)
  double* red = F + n * n;    // 32
  const float* px = S.Ms + ((size_t)inst * S.mp_nslots + S.mp_out[cell]) * n * ldg;
  const double* Wx = (k < N) ? Qbar : QbarN;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    W[e] = Wx[e];
    F[e] = (double)px[(e / n) * ldg + e % n];
  }
  __syncthreads();
  double acc = 0.0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {  // (a, c): Phi[a][c] (W Phi)[a][c]
    const int a = e / n, cc = e - a * n;
    double t = 0.0;
    for (int b = 0; b < n; ++b) t = fma(W[a * n + b], F[b * n + cc], t);
    acc = fma(F[e], t, acc);
  }
  if (k < N) {  // Phi^u_{k,j} (m x n) with Rbar
    __syncthreads();
    const float* pu = S.Phiu + cb * m * n;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) W[e] = Rbar[e];
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) F[e] = (double)pu[e];
    __syncthreads();
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
      const int a = e / n, cc = e - a * n;
      double t = 0.0;
      for (int b = 0; b < m; ++b) t = fma(W[a * m + b], F[b * n + cc], t);
      acc = fma(F[e], t, acc);
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sum += red[w];
    cells[cb] = sum;
  }
}

__global__ void k_sls_cost_sum(const double* cells, int ncell, int B, double* cost) {
  const int inst = blockIdx.x * blockDim.x + threadIdx.x;
  if (inst >= B) return;
  double s = 0.0;
  for (int i = 0; i < ncell; ++i) s += cells[(size_t)inst * ncell + i];
  cost[inst] = s;
}

int sls_cost(Ctx* c, const double* Qbar, const double* Rbar, const double* QbarN, double* cost, cudaStream_t st) {
  int rc = sls_init(c);
  if (rc) return rc;
  SlsState* s = sls_of(c);
  DevSls& S = s->dev;
  const int B = c->dims.batch;
  if (!s->cost_cells) {
    s->cost_cells = (double*)dev_alloc(c, (size_t)B * S.ncell * sizeof(double));
    if (!s->cost_cells) return GSLS_ERR_CUDA;
  }
  const size_t sb = (2 * (size_t)S.n * S.n + 32) * sizeof(double);
  if ((rc = smem_attr((const void*)k_sls_cost_cells, sb))) return rc;
  k_sls_cost_cells<<<dim3(S.ncell, B), 256, sb, st>>>(S, Qbar, Rbar, QbarN, s->cost_cells);
  GSLS_CUDA_CHECK(cudaGetLastError());
  k_sls_cost_sum<<<(B + 127) / 128, 128, 0, st>>>(s->cost_cells, S.ncell, B, cost);
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

__global__ void k_sls_export_costs(DevSls S, double* Qx, double* Qu, double* Qux) {
  const int cell = blockIdx.x, inst = blockIdx.y;
  const int n = S.n, m = S.m;
  const size_t cb = (size_t)inst * S.ncell + cell;
  if (Qx)
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) Qx[cb * n * n + e] = S.Qx[cb * n * n + e];
  if (Qu)
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) Qu[cb * m * m + e] = S.Qu[cb * m * m + e];
  if (Qux)
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) Qux[cb * m * n + e] = S.Qux[cb * m * n + e];
}

int sls_export_costs(Ctx* c, double* Qx, double* Qu, double* Qux, cudaStream_t st) {
  int rc = sls_init(c);
  if (rc) return rc;
  DevSls& S = sls_of(c)->dev;
  k_sls_export_costs<<<dim3(S.ncell, c->dims.batch), 256, 0, st>>>(S, Qx, Qu, Qux);
  GSLS_CUDA_CHECK(cudaGetLastError());
  return GSLS_OK;
}

int sls_ncell(int N) { return N * (N + 1) / 2; }

int sls_set_columns(Ctx* c, int j0, int j1) {
  const int N = c->dims.N;
  if (j1 < 0) j1 = N;
  if (j0 < 0 || j1 > N || j0 >= j1) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "SLS column range must satisfy 0 <= j0 < j1 <= N");
    return GSLS_ERR_ARG;
  }
  if (c->sls && (c->sls_j0 != j0 || (c->sls_j1 < 0 ? N : c->sls_j1) != j1)) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "SLS column range must be set before the first SLS call");
    return GSLS_ERR_ARG;
  }
  c->sls_j0 = j0;
  c->sls_j1 = j1;
  return GSLS_OK;
}

int sls_plan(int N, int cvf, int max_ops, int* ops, int* layer_off, int* out, int* n_ops, int* n_layers,
             int* n_slots) {
  ScanPlan p = merge_columns(N, cvf != 0);
  *n_ops = (int)p.ops.size();
  *n_layers = p.layers;
  *n_slots = p.nslots;
  if ((int)p.ops.size() > max_ops) return GSLS_OK;
  for (size_t i = 0; i < p.ops.size(); ++i) {
    ops[3 * i] = p.ops[i].dst;
    ops[3 * i + 1] = p.ops[i].earlier;
    ops[3 * i + 2] = p.ops[i].later;
  }
  for (int l = 0; l <= p.layers; ++l) layer_off[l] = p.layer_off[l];
  for (size_t i = 0; i < p.out.size(); ++i) out[i] = p.out[i];
  return GSLS_OK;
}

}  // namespace gsls
