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
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <type_traits>
#include <vector>

#include <cooperative_groups.h>

#include "ctx.h"
#include "prof.h"
#include "cluster.cuh"

namespace gsls {

int check_errors(Ctx* c, cudaStream_t st, const char* what);
void set_error(int code, int inst, int where, int aux, int label, const char* msg);

// Whole-GPU replay of ONE large instance (vectors too large for shared memory, e.g.
// cfg-E: 75D, N = 2047): the instance's vectors live once in global memory (L2) and
// every CTA of a cooperative grid owns a share of each phase, exactly as the ranks
// of a cluster do; puts are plain global stores and phases end with a grid barrier.
struct GridCl {
  unsigned rank, cs;
  __device__ void put(double* p, double v) const { *p = v; }
  __device__ void put_mask(double* p, double v, unsigned) const { *p = v; }
  __device__ void sync() const { cooperative_groups::this_grid().sync(); }
};

enum { MODE_LQR = 0, MODE_ADMM = 1 };
enum { ST_DONE = 0, ST_REBUILD = 1, ST_CONTINUE = 2, ST_BUILD_ERR = 3 };  // per-instance exit status of a replay launch

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
  unsigned long long* trace;  // GSLS_REPLAY_TRACE: phase timestamps of the first iteration (rank 0)
  int prefetch;               // k_replay: bulk-prefetch the next tree layer's records into L2
  int cap;                    // ADMM: pause (ST_CONTINUE) an undecided instance at this iteration (0: none)
  const int* count;           // device-side instance count (graph-captured loop); nullptr: grid-sized
};

constexpr int kReplayThreads = 512;
constexpr int kMaxCluster = 16;

// Replay vectors (all float64).
struct VecLayout {
  int pv, bv, cb, t1, t2, z, lam, y, w, rhat, om, kf, du, red, part, redall, masks, plan, total;
};

__host__ __device__ inline VecLayout vec_layout(int n, int m, int N, int mtot, int s_cvf, int s_cot, int max_layer,
                                                int nops_cvf, int nops_cot, int lay_cvf, int lay_cot) {
  VecLayout v;
  int o = 0;
  auto take = [&](int sz) { int r = o; o += (sz + 1) & ~1; return r; };
  v.pv = take(s_cvf * n);
  v.bv = take(s_cvf * n);
  v.cb = take(s_cot * n);
  v.t1 = take(0);  // (unused since the one-round CVF replay)
  v.t2 = take(0);
  v.z = take(mtot);
  v.lam = take(mtot);
  v.y = take(mtot);
  v.w = take(mtot);  // y - z
  v.rhat = take(N * m);
  v.om = take(N * m);  // also the feedforward inner vector
  v.kf = take(N * m);
  v.du = take(N * m);
  v.red = take(64);
  v.part = take(kReplayThreads);     // split-K partial sums (kReplayThreads / 32 warps x 32 rows)
  v.redall = take(2 * kMaxCluster);  // per-rank partial maxima of the residuals
  v.masks = take((s_cvf + s_cot + 1) / 2 + 1);  // consumer-rank masks per slot (uint32)
  v.plan = take(2 * (nops_cvf + nops_cot) + (2 * lay_cvf + lay_cot + 2 + 2 * N + 2) / 2 + 2);  // scan plan copy
  v.total = o;
  return v;
}

size_t replay_smem_floats(const Ctx* c) {
  const int ml = std::max(1, std::max(c->cvf_max_layer, c->cot_max_layer));
  return (size_t)vec_layout(c->dims.nx, c->dims.nu, c->dims.N, c->mtot, c->cvf.nslots, c->cot.nslots, ml,
                           (int)c->cvf.ops.size(), (int)c->cot.ops.size(), c->cvf.layers, c->cot.layers).total;
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

// Partial column-major matvec over k in [k0, k1) for one 32-row block: lanes
// with g == 0 return the sums of rows 32rb + 4rq .. +3 (see warp_cm_matvec).
__device__ inline void warp_cm_partial(const float* __restrict__ Mcm, int ldg, int rb, const double* x, int k0,
                                       int k1, double (&acc)[4]) {
  const int lane = threadIdx.x & 31;
  const int rq = lane & 7, g = lane >> 3;
  const int row0 = rb * 32 + 4 * rq;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (row0 < ldg) {
    const float* p = Mcm + row0;
#pragma unroll 8
    for (int k = k0 + g; k < k1; k += 4) {
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
  acc[0] = a0; acc[1] = a1; acc[2] = a2; acc[3] = a3;
}

// f32 -> f64 widening off the conversion pipe (F2F.F64.F32 issues at 16 / clk / SM on
// B200, tools/micro/cvt.cu): shifting the f32 exponent+mantissa down 3 bits into an f64
// gives exactly f * 2^-896 for every finite f, denormals included.  Accumulate in that
// scale and multiply the sum by 2^896; products stay normal unless |M x| < 2^-126.
__device__ __forceinline__ double widen_scaled(uint32_t u) {
  const uint32_t hi = ((u >> 3) & 0x0FFFFFFFu) | (u & 0x80000000u);
  return __hiloint2double((int)hi, (int)(u << 29));
}
constexpr double kWidenUnscale = 0x1p896;

// L2 prefetch of a contiguous byte range (the next tree layer's recorded operators),
// issued by one thread in <= 1 MB bulk requests; addresses widened to 16-byte alignment.
__device__ inline void prefetch_l2_range(const void* p, size_t bytes) {
  unsigned long long a = (unsigned long long)p & ~15ull;
  const unsigned long long e = ((unsigned long long)p + bytes + 15ull) & ~15ull;
  while (a < e) {
    const unsigned long long len = (e - a) < (1ull << 20) ? (e - a) : (1ull << 20);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)len) : "memory");
    a += len;
  }
}

// Stage operator product for one (4*RQ)-row block: acc = M x (+ M2 x2), both
// column-major with leading dimension ld (rows padded with zeros).  Lane
// (rq, g): rows 4rq..4rq+3 of the block as one 16-byte load per column, k =
// g, g + 32/RQ, ...  Lanes with g == 0 return the sums.
template <int RQ>
__device__ inline void warp_stage_mv(const float* __restrict__ M, int ld, int rb, const double* x, int klen,
                                     const float* __restrict__ M2, const double* x2, int klen2, double (&acc)[4]) {
  constexpr int KG = 32 / RQ;
  const int lane = threadIdx.x & 31;
  const int rq = lane % RQ, g = lane / RQ;
  const int row0 = rb * 4 * RQ + 4 * rq;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (row0 < ld) {
#pragma unroll 4
    for (int k = g; k < klen; k += KG) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(M + (size_t)k * ld + row0));
      const double xk = x[k];
      a0 = fma((double)v.x, xk, a0);
      a1 = fma((double)v.y, xk, a1);
      a2 = fma((double)v.z, xk, a2);
      a3 = fma((double)v.w, xk, a3);
    }
    if (M2) {
#pragma unroll 4
      for (int k = g; k < klen2; k += KG) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(M2 + (size_t)k * ld + row0));
        const double xk = x2[k];
        a0 = fma((double)v.x, xk, a0);
        a1 = fma((double)v.y, xk, a1);
        a2 = fma((double)v.z, xk, a2);
        a3 = fma((double)v.w, xk, a3);
      }
    }
  }
#pragma unroll
  for (int o = RQ; o < 32; o <<= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    a3 += __shfl_xor_sync(0xffffffffu, a3, o);
  }
  acc[0] = a0; acc[1] = a1; acc[2] = a2; acc[3] = a3;
}

// 64-row variant: lane (rq, g) = (lane & 15, lane >> 4) covers rows 64rb + 4rq .. +3, k = g, g + 2, ...;
// 16 lanes of equal g read one full 256-byte column segment per k (better DRAM locality
// for the batched replay, where the recorded operators stream from HBM).
__device__ inline void warp_cm_partial64(const float* __restrict__ Mcm, int ldg, int rb, const double* x, int k0,
                                         int k1, double (&acc)[4]) {
  const int lane = threadIdx.x & 31;
  const int rq = lane & 15, g = lane >> 4;
  const int row0 = rb * 64 + 4 * rq;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (row0 < ldg) {
    const float* p = Mcm + row0;
#pragma unroll 8
    for (int k = k0 + g; k < k1; k += 2) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p + (size_t)k * ldg));
      const double xk = x[k];
      a0 = fma((double)v.x, xk, a0);
      a1 = fma((double)v.y, xk, a1);
      a2 = fma((double)v.z, xk, a2);
      a3 = fma((double)v.w, xk, a3);
    }
  }
  a0 += __shfl_xor_sync(0xffffffffu, a0, 16);
  a1 += __shfl_xor_sync(0xffffffffu, a1, 16);
  a2 += __shfl_xor_sync(0xffffffffu, a2, 16);
  a3 += __shfl_xor_sync(0xffffffffu, a3, 16);
  acc[0] = a0; acc[1] = a1; acc[2] = a2; acc[3] = a3;
}

// acc = M x (+ sgn2 M2 x2) over k in [k0, k1) for one 32-row block.
__device__ inline void warp_cm_partial2(const float* __restrict__ M, const double* x, const float* __restrict__ M2,
                                        const double* x2, double sgn2, int ldg, int rb, int k0, int k1,
                                        double (&acc)[4]) {
  if (!M2) {
    warp_cm_partial64(M, ldg, rb, x, k0, k1, acc);
    return;
  }
  // both operators in one loop: twice the loads in flight per lane
  const int lane = threadIdx.x & 31;
  const int rq = lane & 15, g = lane >> 4;
  const int row0 = rb * 64 + 4 * rq;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
  if (row0 < ldg) {
    const float* p = M + row0;
    const float* q = M2 + row0;
#pragma unroll 4
    for (int k = k0 + g; k < k1; k += 2) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p + (size_t)k * ldg));
      const float4 u = __ldg(reinterpret_cast<const float4*>(q + (size_t)k * ldg));
      const double xk = x[k], yk = x2[k];
      a0 = fma((double)v.x, xk, a0);
      a1 = fma((double)v.y, xk, a1);
      a2 = fma((double)v.z, xk, a2);
      a3 = fma((double)v.w, xk, a3);
      b0 = fma((double)u.x, yk, b0);
      b1 = fma((double)u.y, yk, b1);
      b2 = fma((double)u.z, yk, b2);
      b3 = fma((double)u.w, yk, b3);
    }
  }
  a0 = fma(sgn2, b0, a0);
  a1 = fma(sgn2, b1, a1);
  a2 = fma(sgn2, b2, a2);
  a3 = fma(sgn2, b3, a3);
  a0 += __shfl_xor_sync(0xffffffffu, a0, 16);
  a1 += __shfl_xor_sync(0xffffffffu, a1, 16);
  a2 += __shfl_xor_sync(0xffffffffu, a2, 16);
  a3 += __shfl_xor_sync(0xffffffffu, a3, 16);
  acc[0] = a0; acc[1] = a1; acc[2] = a2; acc[3] = a3;
}

// One matvec of a replay round: y = add + sgn * M x (M column-major, fp32).
struct MvTask {
  const float* M;
  const double* x;
  const double* add;
  double sgn;
  double* y;
  unsigned mask;     // ranks (besides this one) whose replica of y consumes the result
  const float* M2;   // optional second operator: y = add + sgn * (M x + sgn2 * M2 x2)
  const double* x2;
  double sgn2;
};

// Runs `ntask` independent matvecs (descriptors from desc(i)) with the CTA's
// warps, splitting the k range over up to 4 warps when there are fewer
// (task, row block) pairs than warps.  Partial sums are combined in a fixed
// order, so the result does not depend on timing.  Ends with __syncthreads
// (outputs are complete in this CTA; remote replicas need the caller's
// cluster barrier).
__device__ inline unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <class Comm, class Desc>
__device__ void mv_round(int ntask, int n, int ldg, double* part, const Comm& cl, Desc desc,
                         unsigned long long* dbg = nullptr) {
  auto D = [&](int j) { if (dbg && threadIdx.x == 0) dbg[j] = clock64(); };
  D(0);
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, nwarp = nthr >> 5, lane = tid & 31;
  const int RB = (n + 63) >> 6;  // 64-row blocks
  const int base = ntask * RB;
  int KS = 1;
  while (KS < 4 && base * KS * 2 <= nwarp / 2) KS <<= 1;  // partials: base * KS * 64 <= 512
  if (KS == 1) {
    for (int t = warp; t < base; t += nwarp) {
      const int ti = t / RB, rb = t - ti * RB;
      const MvTask d = desc(ti);
      double acc[4];
      warp_cm_partial2(d.M, d.x, d.M2, d.x2, d.sgn2, ldg, rb, 0, n, acc);
      if ((lane >> 4) == 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int row = rb * 64 + 4 * (lane & 15) + r;
          if (row < n) {
            const double v = d.add[row] + d.sgn * acc[r];
            cl.put_mask(d.y + row, v, d.mask);
          }
        }
      }
    }
    __syncthreads();
    return;
  }
  const int kc = ((n + KS - 1) / KS + 1) & ~1;  // slice length, even (keeps the 2-way lane interleave)
  for (int t = warp; t < base * KS; t += nwarp) {
    const int tb = t / KS, ks = t - tb * KS;
    const int ti = tb / RB, rb = tb - ti * RB;
    const MvTask d = desc(ti);
    if (t == 0) D(1);
    double acc[4];
    const int k0 = ks * kc;
    warp_cm_partial2(d.M, d.x, d.M2, d.x2, d.sgn2, ldg, rb, k0, min(n, k0 + kc), acc);
    if (t == 0) D(2);
    if ((lane >> 4) == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) part[(tb * KS + ks) * 64 + 4 * (lane & 15) + r] = acc[r];
    }
  }
  __syncthreads();
  D(3);
  for (int e = tid; e < base * 64; e += nthr) {
    const int tb = e >> 6, ro = e & 63;
    const int ti = tb / RB, rb = tb - ti * RB;
    const int row = rb * 64 + ro;
    if (row >= n) continue;
    double s = 0.0;
    for (int ks = 0; ks < KS; ++ks) s += part[(tb * KS + ks) * 64 + ro];
    const MvTask d = desc(ti);
    const double v = d.add[row] + d.sgn * s;
    cl.put_mask(d.y + row, v, d.mask);
  }
  D(4);
  __syncthreads();
}

// Cooperative dot products: G lanes per output, outputs spread over the whole
// cluster (gt / gs = cluster-wide thread index / stride).  out(e, s) is called
// by the group's first lane with s = sum_t term(e, t), t < len.
template <int G, class Term, class Out>
__device__ inline void gdot(int total, int len, int gt, int gs, Term term, Out out) {
  const int lane = threadIdx.x & 31, lg = lane & (G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  for (int e = gt / G; e < total; e += gs / G) {
    double s = 0.0;
#pragma unroll 16
    for (int t = lg; t < len; t += G) s += term(e, t);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(gmask, s, o);
    if (lg == 0) out(e, s);
  }
}

// Single CTA per instance (large batches): one thread per output keeps more
// independent work in flight per warp; clusters: G lanes per output.
template <int G, class Term, class Out>
__device__ inline void gdotc(int cs, int total, int len, int gt, int gs, Term term, Out out) {
  if (cs == 1) gdot<1>(total, len, gt, gs, term, out);
  else gdot<G>(total, len, gt, gs, term, out);
}

// GRID: one instance over a cooperative grid (GridCl, rank = blockIdx.x); otherwise one
// instance per cluster (Cl, rank = cluster rank), blockIdx.y = instance.
template <bool GRID>
__global__ void __launch_bounds__(kReplayThreads, 1) k_replay(ReplayArgs a) {
  using Comm = typename std::conditional<GRID, GridCl, Cl>::type;
  const DevLqr& L = a.L;
  if (!GRID && a.count && (int)blockIdx.y >= *a.count) return;
  const int inst = a.list ? a.list[blockIdx.y] : (int)blockIdx.y;
  if (a.mode == MODE_ADMM && L.err[inst].key != 0) {  // its (re)build raised: the host driver decides
    if ((GRID ? blockIdx.x : cluster_rank()) == 0 && threadIdx.x == 0) a.status[inst] = ST_BUILD_ERR;
    return;
  }
  const int n = L.n, m = L.m, c = L.c, nf = L.nf, N = L.N, ldg = L.ldg, mtot = L.mtot;
  const size_t MS = (size_t)n * ldg;
  const int tid = threadIdx.x, nthr = blockDim.x;
  Comm cl;
  cl.rank = GRID ? blockIdx.x : cluster_rank();
  cl.cs = GRID ? gridDim.x : cluster_size();
  const int rank = (int)cl.rank, cs = (int)cl.cs;
  const int gt = rank * nthr + tid, gs = cs * nthr;  // cluster- (grid-) wide thread index / stride
  const VecLayout V = vec_layout(n, m, N, mtot, L.cvf_nslots, L.cot_nslots, a.max_layer, L.cvf_nops, L.cot_nops,
                                 L.cvf_layers, L.cot_layers);
  extern __shared__ double smem[];
  double* vs = a.gscratch ? a.gscratch + (size_t)inst * a.scratch_floats : smem;
  double *pv = vs + V.pv, *bv = vs + V.bv, *cb = vs + V.cb;
  double *z = vs + V.z, *lam = vs + V.lam, *y = vs + V.y;
  double *rhat = vs + V.rhat, *om = vs + V.om, *kf = vs + V.kf, *du = vs + V.du;
  double *red = GRID ? smem : vs + V.red;                   // per-CTA scratch
  double *part = GRID ? smem + 64 : vs + V.part;            // per-CTA split-K partials
  double* redall = vs + V.redall;
  __shared__ int s_flag;  // 0 continue, 1 done, 2 rebuild
  __shared__ double s_rho;

  const size_t sN = (size_t)inst * N;
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
  const float* X23 = L.X23 + sN * c * L.ld2n;
  const double* pb0 = L.pb0 + sN * 2 * n;
  const float* XK = L.XK + sN * (n + c) * L.ldm;
  const double* kk0 = L.kk0 + sN * m;
  const float* Bcm = L.Bcm + sN * m * L.ldn;
  const float* ZD = L.ZD + sN * (n + m) * L.ldc;
  const int warp = tid >> 5, lane = tid & 31, nwarp = nthr >> 5;

  double* w = vs + V.w;
  // the scan plans, copied to shared memory (every op / layer lookup is on a phase's critical
  // path); a GRID launch (one large instance) reads them from global memory instead
  const int4* s_cvf_ops = L.cvf_ops;
  const int4* s_cot_ops = L.cot_ops;
  const int* s_cvf_loff = L.cvf_loff;
  const int* s_cot_loff = L.cot_loff;
  const int* s_cvf_out = L.cvf_out;
  const int* s_cot_out = L.cot_out;
  const int* s_cvf_blive = L.cvf_blive;
  if (!GRID) {
    int4* p_cvf_ops = reinterpret_cast<int4*>(vs + V.plan);
    int4* p_cot_ops = p_cvf_ops + L.cvf_nops;
    int* p_cvf_loff = reinterpret_cast<int*>(p_cot_ops + L.cot_nops);
    int* p_cot_loff = p_cvf_loff + L.cvf_layers + 1;
    int* p_cvf_out = p_cot_loff + L.cot_layers + 1;
    int* p_cot_out = p_cvf_out + N + 1;
    int* p_cvf_blive = p_cot_out + N;
    for (int i = tid; i < L.cvf_layers; i += nthr) p_cvf_blive[i] = L.cvf_blive[i];
    for (int i = tid; i < L.cvf_nops; i += nthr) p_cvf_ops[i] = L.cvf_ops[i];
    for (int i = tid; i < L.cot_nops; i += nthr) p_cot_ops[i] = L.cot_ops[i];
    for (int i = tid; i <= L.cvf_layers; i += nthr) p_cvf_loff[i] = L.cvf_loff[i];
    for (int i = tid; i <= L.cot_layers; i += nthr) p_cot_loff[i] = (N > 0) ? L.cot_loff[i] : 0;
    for (int i = tid; i <= N; i += nthr) p_cvf_out[i] = L.cvf_out[i];
    for (int i = tid; i < N; i += nthr) p_cot_out[i] = L.cot_out[i];
    s_cvf_ops = p_cvf_ops; s_cot_ops = p_cot_ops; s_cvf_loff = p_cvf_loff; s_cot_loff = p_cot_loff;
    s_cvf_out = p_cvf_out; s_cot_out = p_cot_out; s_cvf_blive = p_cvf_blive;
  }
  __syncthreads();
  // dx_k lives in the COT outputs (k >= 1) or dx0
  auto dxp = [&](int k) -> const double* { return k == 0 ? dx0 : cb + (size_t)s_cot_out[k - 1] * n; };

  const bool admm = a.mode == MODE_ADMM;
  double rho = 0.0;
  int it = 0;
  if (admm) {
    rho = a.state.rho[inst];
    it = a.stats.iterations[inst];
    const double* zg = a.state.z + (size_t)inst * mtot;
    const double* lg = a.state.lam + (size_t)inst * mtot;
    const double* yg = a.state.y + (size_t)inst * mtot;
    for (int e = GRID ? gt : tid; e < mtot; e += GRID ? gs : nthr) {  // GRID: shared copy, one writer
      z[e] = zg[e]; lam[e] = lg[e]; y[e] = yg[e];
      w[e] = yg[e] - zg[e];
    }
  }
  // Consumer ranks of every scan slot (clusters only).  Stage k's leaf terms,
  // feedforward, constraint rows and state live on rank srank(k) = k % cs; op
  // oi of a layer runs on rank oi / ceil(ops / cs).  A slot goes to the ranks
  // of the ops that read it and of the stage that reads it as p+ / dx.
  unsigned* cvf_mask = reinterpret_cast<unsigned*>(vs + V.masks);
  unsigned* cot_mask = cvf_mask + L.cvf_nslots;
  auto srank = [&](int k) { return k % cs; };
  if (!GRID)
    for (int i = tid; i < L.cvf_nslots + L.cot_nslots; i += nthr) cvf_mask[i] = 0u;
  __syncthreads();
  if (!GRID && cs > 1) {
    for (int lay = 0; lay < L.cvf_layers; ++lay) {  // op oi (both halves) on rank oi / per
      const int o0 = s_cvf_loff[lay], no = s_cvf_loff[lay + 1] - o0, per = (no + cs - 1) / cs;
      for (int oi = tid; oi < no; oi += nthr) {
        const int4 op = s_cvf_ops[o0 + oi];
        atomicOr(cvf_mask + op.y, 1u << (oi / per));
        atomicOr(cvf_mask + op.z, 1u << (oi / per));
      }
    }
    for (int p = tid; p <= N; p += nthr) atomicOr(cvf_mask + s_cvf_out[p], 1u << srank(max(p - 1, 0)));
    for (int lay = 0; lay < L.cot_layers; ++lay) {
      const int o0 = s_cot_loff[lay], no = s_cot_loff[lay + 1] - o0, per = (no + cs - 1) / cs;
      for (int oi = tid; oi < no; oi += nthr) {
        const int4 op = s_cot_ops[o0 + oi];
        atomicOr(cot_mask + op.y, 1u << (oi / per));
        atomicOr(cot_mask + op.z, 1u << (oi / per));
      }
    }
    for (int k = 1 + tid; k <= N; k += nthr) atomicOr(cot_mask + s_cot_out[k - 1], 1u << srank(k));
  }
  // stages owned by this rank: k = rank, rank + cs, ... < N
  const int nls = (rank < N) ? (N - rank + cs - 1) / cs : 0;
  cl.sync();  // replicas of every CTA exist before the first remote store
  bool tr_on = a.trace != nullptr && rank == 0 && tid == 0 && blockIdx.y == 0;
  int tn = 0;
  auto TR = [&]() {
    if (tr_on && tn < 255) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[++tn] = t;
      a.trace[0] = tn;
    }
  };
  TR();

  // one CTA per instance: every stage's operators are contiguous, so whole phases are
  // prefetched into L2 one phase ahead (the next layer's records, the next phase's
  // stage operators)
  const bool pf = a.prefetch == 2 && cs == 1 && admm && tid == 0;  // stage operators too (GSLS_REPLAY_PREFETCH=2)
  if (pf) prefetch_l2_range(X23, (size_t)N * c * L.ld2n * sizeof(float));
  for (;;) {
    if (pf && L.cvf_layers > 0)
      prefetch_l2_range(cvf_rec + (size_t)s_cvf_loff[0] * 4 * MS,
                        (size_t)(s_cvf_loff[1] - s_cvf_loff[0]) * 4 * MS * sizeof(float));
    // ---- CVF leaves: [p; b]_k = pb0_k + X23_k (y - z)_k (fused augment_linear +
    //      _linear_element_terms, admm.py:113-121, lqr.py:338-342) --------------------
    if (admm) {
      const int RB2 = (2 * n + 31) >> 5;
      for (int t = warp; t < nls * RB2; t += nwarp) {
        const int k = rank + (t / RB2) * cs, rb = t % RB2;
        double acc[4];
        warp_stage_mv<8>(X23 + (size_t)k * c * L.ld2n, L.ld2n, rb, w + k * c, c, nullptr, nullptr, 0, acc);
        if (lane < 8) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int row = rb * 32 + 4 * lane + r;
            if (row < 2 * n) {
              const double v = pb0[(size_t)k * 2 * n + row] + acc[r];
              if (row < n) cl.put_mask(pv + k * n + row, v, cvf_mask[k]);
              else cl.put_mask(bv + k * n + row - n, v, cvf_mask[k]);
            }
          }
        }
      }
      if (rank == srank(N))
        for (int i = tid; i < n; i += nthr) {
          double s = 0.0;
          for (int f = 0; f < nf; ++f) s = fma((double)CNq[f * n + i], w[N * c + f], s);
          cl.put_mask(pv + N * n + i, qN_lin[i] + rho * s, cvf_mask[N]);
          cl.put_mask(bv + N * n + i, 0.0, cvf_mask[N]);
        }
      cl.sync();
      TR();
    } else {  // LQR mode: plain linear terms (lqr.py:338-342)
      for (int e = gt; e < N * m; e += gs) cl.put(rhat + e, r_lin[e]);
      for (int e = gt; e < N * n; e += gs) cl.put(pv + e, q_lin[e]);
      for (int i = gt; i < n; i += gs) {
        cl.put(pv + N * n + i, qN_lin[i]);
        cl.put(bv + N * n + i, 0.0);
      }
      cl.sync();
      TR();
      gdotc<4>(cs, N * m, m, gt, gs,
              [&](int e, int t) { const int k = e / m, i = e - k * m;
                                  return (double)Rinv[((size_t)k * m + i) * m + t] * rhat[k * m + t]; },
              [&](int e, double s) { cl.put(om + e, s); });
      cl.sync();
      TR();
      gdotc<4>(cs, N * n, m, gt, gs,
              [&](int e, int l) { const int k = e / n, i = e - k * n;
                                  return (double)Shat[((size_t)k * m + l) * n + i] * om[k * m + l]; },
              [&](int e, double s) { cl.put(pv + e, pv[e] - s); });
      gdotc<4>(cs, N * n, m, gt, gs,
              [&](int e, int l) { const int k = e / n, i = e - k * n;
                                  return (double)Bq[((size_t)k * n + i) * m + l] * om[k * m + l]; },
              [&](int e, double s) { cl.put(bv + e, bq[e] - s); });
      cl.sync();
      TR();
    }

    // ---- CVF replay (reverse tree): ops of a layer spread over the cluster ------
    for (int lay = 0; lay < L.cvf_layers; ++lay) {
      const int o0 = s_cvf_loff[lay], no = s_cvf_loff[lay + 1] - o0;
      if (pf && lay + 1 == L.cvf_layers) {  // the feedforward's stage operators
        prefetch_l2_range(XK, (size_t)N * (n + c) * L.ldm * sizeof(float));
        prefetch_l2_range(Bcm, (size_t)N * m * L.ldn * sizeof(float));
      }
      if (tid == 0 && lay + 1 < L.cvf_layers && a.prefetch) {  // next layer's records -> L2 during this round
        const int p0 = s_cvf_loff[lay + 1], pn = s_cvf_loff[lay + 2] - p0, pp = (pn + cs - 1) / cs;
        const int plo = min(pn, rank * pp), pnl = min(pn, plo + pp) - plo;
        // ops with a live b: all four operators (contiguous); the rest: [Ups X] only
        const int pl = max(0, min(plo + pnl, s_cvf_blive[lay + 1]) - plo);
        if (pl > 0) prefetch_l2_range(cvf_rec + (size_t)(p0 + plo) * 4 * MS, (size_t)pl * 4 * MS * sizeof(float));
        for (int q = plo + pl; q < plo + pnl; ++q)
          prefetch_l2_range(cvf_rec + (size_t)(p0 + q) * 4 * MS, (size_t)2 * MS * sizeof(float));
      }
      if (no == 0) continue;
      const int per = (no + cs - 1) / cs;
      const int lo = min(no, rank * per), nl = min(no, lo + per) - lo;
      if (nl > 0) {
        // p = p_earlier + Ups p_later + X b_earlier, b = b_later + Psi b_earlier - Y p_later
        // (lqr.py:242-246 with the recorded X = Ups Pr, -Y = -Psi Cl): one round per layer.
        // Tasks [0, nl): the p halves; [nl, nl + nb): the b halves of the ops whose result
        // a later op reads (the layer's first s_cvf_blive[lay] ops; the b of the scan's
        // final outputs is never read, plan.h partition_unread_last)
        const int nb = max(0, min(lo + nl, s_cvf_blive[lay]) - lo);
        mv_round(nl + nb, n, ldg, part, cl, [&](int ti) {
          const bool bh = ti >= nl;
          const int oi = lo + (bh ? ti - nl : ti);
          const int4 op = s_cvf_ops[o0 + oi];
          const float* rec = cvf_rec + (size_t)(o0 + oi) * 4 * MS;
          if (!bh)
            return MvTask{rec + 0 * MS, pv + op.z * n, pv + op.y * n, 1.0, pv + op.x * n, cvf_mask[op.x],
                          rec + 1 * MS, bv + op.y * n, 1.0};
          return MvTask{rec + 2 * MS, bv + op.y * n, bv + op.z * n, 1.0, bv + op.x * n, cvf_mask[op.x],
                        rec + 3 * MS, pv + op.z * n, 1.0};  // the record holds -Y
        }, (tr_on && lay == 3) ? a.trace + 200 : nullptr);
      }
      cl.sync();
      TR();
    }

    if (pf && L.cot_layers > 0)
      prefetch_l2_range(cot_rec + (size_t)s_cot_loff[0] * MS, (size_t)(s_cot_loff[1] - s_cot_loff[0]) * MS * sizeof(float));
    // ---- feedforward k = -Gamma (B'(p+ + P+ b) + r) and COT leaves ---------------
    //      (lqr.py:345-356; ADMM: kf = kk0 + X5 p+ + X4 (y - z), cb = B kf + b)
    if (admm) {
      const int RBm = (m + 15) >> 4;
      for (int t = warp; t < nls * RBm; t += nwarp) {
        const int k = rank + (t / RBm) * cs, rb = t % RBm;
        double acc[4];
        const float* xk_ = XK + (size_t)k * (n + c) * L.ldm;
        warp_stage_mv<4>(xk_, L.ldm, rb, pv + (size_t)s_cvf_out[k + 1] * n, n, xk_ + (size_t)n * L.ldm, w + k * c, c,
                         acc);
        if (lane < 4) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int row = rb * 16 + 4 * lane + r;
            if (row < m) kf[k * m + row] = kk0[(size_t)k * m + row] + acc[r];  // read on this rank only
          }
        }
      }
      __syncthreads();
      TR();
      const int RBn = (n + 31) >> 5;
      for (int t = warp; t < nls * RBn; t += nwarp) {
        const int k = rank + (t / RBn) * cs, rb = t % RBn;
        double acc[4];
        warp_stage_mv<8>(Bcm + (size_t)k * m * L.ldn, L.ldn, rb, kf + k * m, m, nullptr, nullptr, 0, acc);
        if (lane < 8) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int row = rb * 32 + 4 * lane + r;
            if (row < n) {
              const double bb = acc[r] + bq[(size_t)k * n + row];
              cl.put_mask(cb + k * n + row, (k == 0) ? v0[row] + bb : bb, cot_mask[k]);
            }
          }
        }
      }
      cl.sync();
      TR();
    } else {
      gdotc<8>(cs, N * m, n, gt, gs,
              [&](int e, int i) { const int k = e / m, l = e - k * m;
                                  return (double)Bq[((size_t)k * n + i) * m + l] *
                                         (pv[(size_t)s_cvf_out[k + 1] * n + i] + cvec[(size_t)k * n + i]); },
              [&](int e, double s) { cl.put(om + e, s + rhat[e]); });
      cl.sync();
      TR();
      gdotc<4>(cs, N * m, m, gt, gs,
              [&](int e, int t) { const int k = e / m, l = e - k * m;
                                  return (double)Gam[((size_t)k * m + l) * m + t] * om[k * m + t]; },
              [&](int e, double s) { cl.put(kf + e, -s); });
      cl.sync();
      TR();
      gdotc<4>(cs, N * n, m, gt, gs,
              [&](int e, int l) { const int k = e / n;
                                  return (double)Bq[(size_t)e * m + l] * kf[k * m + l]; },
              [&](int e, double s) { const int k = e / n, i = e - k * n;
                                     const double bb = s + bq[e];
                                     cl.put(cb + e, (k == 0) ? v0[i] + bb : bb); });
      cl.sync();
      TR();
    }

    // ---- COT replay (forward tree): 1 round per layer -------------------------
    for (int lay = 0; lay < L.cot_layers; ++lay) {
      const int o0 = s_cot_loff[lay], no = s_cot_loff[lay + 1] - o0;
      if (pf && lay + 1 == L.cot_layers) {  // the constraint phase, then the next iteration's leaves
        prefetch_l2_range(ZD, (size_t)N * (n + m) * L.ldc * sizeof(float));
        prefetch_l2_range(X23, (size_t)N * c * L.ld2n * sizeof(float));
      }
      if (tid == 0 && lay + 1 < L.cot_layers && a.prefetch) {
        const int p0 = s_cot_loff[lay + 1], pn = s_cot_loff[lay + 2] - p0, pp = (pn + cs - 1) / cs;
        const int plo = min(pn, rank * pp), pnl = min(pn, plo + pp) - plo;
        if (pnl > 0) prefetch_l2_range(cot_rec + (size_t)(p0 + plo) * MS, (size_t)pnl * MS * sizeof(float));
      }
      if (no == 0) continue;
      const int per = (no + cs - 1) / cs;
      const int lo = min(no, rank * per), nl = min(no, lo + per) - lo;
      if (nl > 0)
        mv_round(nl, n, ldg, part, cl, [&](int ti) {
          const int oi = lo + ti;
          const int4 op = s_cot_ops[o0 + oi];
          return MvTask{cot_rec + (size_t)(o0 + oi) * MS, cb + op.y * n, cb + op.z * n, 1.0, cb + op.x * n,
                        cot_mask[op.x], nullptr, nullptr, 0.0};
        });
      cl.sync();
      TR();
    }

    if (!admm) {
      // ---- du = K dx + k ------------------------------------------------------------
      gdotc<8>(cs, N * m, n, gt, gs,
              [&](int e, int i) { const int k = e / m;
                                  return (double)Kg[(size_t)e * n + i] * dxp(k)[i]; },
              [&](int e, double s) { cl.put(du + e, s + kf[e]); });
      cl.sync();
      TR();
      if (rank == 0) {
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
            a.p_out[(size_t)inst * (N + 1) * n + e] = pv[s_cvf_out[k] * n + i];
          }
      }
      cl.sync();  // no CTA leaves while others may still store into its replica
      return;
    }

    // ---- ADMM: G = Z dx + D kf (= C dx + D du), projection, dual ascent,
    //      residuals (admm.py:91-97, :130-135, :184-189) ----------------------------
    const double* fst = a.qp.f + sN * c;
    const double* fN = a.qp.fN + (size_t)inst * nf;
    double rp = 0.0, rdz = 0.0;
    auto project = [&](int e, double g, double fe) {
      const double zo = z[e];
      const double zn = fmin(g + y[e], fe);
      const double ln = lam[e] + rho * (g - zn);
      const double yn = ln / rho;
      lam[e] = ln;  // stage rows live on their owner rank only
      y[e] = yn;
      z[e] = zn;
      w[e] = yn - zn;
      rp = fmax(rp, fabs(g - zn));
      rdz = fmax(rdz, fabs(zn - zo));
    };
    {
      const int RBc = (c + 31) >> 5;
      for (int t = warp; t < nls * RBc; t += nwarp) {
        const int k = rank + (t / RBc) * cs, rb = t % RBc;
        double acc[4];
        const float* zd_ = ZD + (size_t)k * (n + m) * L.ldc;
        warp_stage_mv<8>(zd_, L.ldc, rb, dxp(k), n, zd_ + (size_t)n * L.ldc, kf + k * m, m, acc);
        if (lane < 8) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int row = rb * 32 + 4 * lane + r;
            if (row < c) project(k * c + row, acc[r], fst[(size_t)k * c + row]);
          }
        }
      }
      for (int f = (rank == srank(N)) ? tid : nf; f < nf; f += nthr) {
        const double* xN = dxp(N);
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = fma((double)CNq[f * n + i], xN[i], s);
        project(N * c + f, s, fN[f]);
      }
    }
    rp = block_max_d(rp, red);
    rdz = block_max_d(rdz, red + 32);
    if (tid == 0) {
      cl.put(redall + 2 * rank, rp);
      cl.put(redall + 2 * rank + 1, rdz);
    }
    cl.sync();
    TR();
    if (tid == 0) {
      double r_p = 0.0, r_dz = 0.0;
      for (int r = 0; r < cs; ++r) {
        r_p = fmax(r_p, redall[2 * r]);
        r_dz = fmax(r_dz, redall[2 * r + 1]);
      }
      ++it;
      const double r_d = rho * r_dz;
      const bool lead = rank == 0;
      if (lead) {
        a.state.iteration[inst] += 1;
        a.state.r_primal[inst] = r_p;
        a.state.r_dual[inst] = r_d;
      }
      int flag = 0;
      double rho_new = rho;
      if (r_p <= a.set.tol_primal && r_d <= a.set.tol_dual) {
        if (lead) a.stats.converged[inst] = 1;
        flag = 1;
      } else {
        bool changed = false;
        if (it % a.set.sigma == 0) {
          const double ratio = sqrt(fmax(r_p, 1e-30) / fmax(r_d, 1e-30));
          const double prop = fmin(fmax(rho * ratio, a.set.rho_min), a.set.rho_max);
          if (prop > 5.0 * rho || prop < rho / 5.0) {
            rho_new = prop;
            if (lead) {
              a.state.rho[inst] = prop;
              a.state.generation[inst] += 1;
              a.stats.rho_changes[inst] += 1;
            }
            changed = true;
          }
        }
        if (it >= a.set.max_iter) flag = 1;
        else if (changed) flag = 2;
        else if (a.cap > 0 && it >= a.cap) flag = 3;  // paused: resumes bitwise-identically in the next launch
      }
      if (lead) a.stats.iterations[inst] = it;
      s_flag = flag;
      s_rho = rho_new;
    }
    __syncthreads();
    const int flag = s_flag;
    tr_on = false;
    if (flag == 0) continue;
    const double rho_new = s_rho;
    // each rank writes back what it owns: stage k's rows on srank(k), terminal rows on srank(N)
    auto owns_row = [&](int e) { return srank(e < N * c ? e / c : N) == rank; };
    if (rho_new != rho)  // committed change rescales y = lam / rho (admm.py:149)
      for (int e = tid; e < mtot; e += nthr)
        if (owns_row(e)) y[e] = lam[e] / rho_new;
    __syncthreads();
    {
      double* zg = a.state.z + (size_t)inst * mtot;
      double* lg = a.state.lam + (size_t)inst * mtot;
      double* yg = a.state.y + (size_t)inst * mtot;
      for (int e = tid; e < mtot; e += nthr)
        if (owns_row(e)) { zg[e] = z[e]; lg[e] = lam[e]; yg[e] = y[e]; }
      if (flag == 1) {
        double* gdx = a.dx + (size_t)inst * (N + 1) * n;
        double* gdu = a.du + (size_t)inst * N * m;
        for (int e = tid; e < (N + 1) * n; e += nthr) {
          const int p = e / n, i = e - p * n;
          if ((p == 0 ? 0 : srank(p)) == rank) gdx[e] = dxp(p)[i];
          if (srank(max(p - 1, 0)) == rank)  // cost-to-go gradient of the last replay
            L.last_p[(size_t)inst * (N + 1) * n + e] = pv[s_cvf_out[p] * n + i];
        }
        for (int e = tid; e < N * m; e += nthr) {  // du = K dx + k (lqr.py:359-363), once at exit
          const int k = e / m;
          if (srank(k) != rank) continue;
          const double* xk = dxp(k);
          double s = 0.0;
          for (int i = 0; i < n; ++i) s = fma((double)Kg[(size_t)e * n + i], xk[i], s);
          gdu[e] = s + kf[e];
          L.last_k[(size_t)inst * N * m + e] = kf[e];
        }
      }
      if (rank == 0 && tid == 0) a.status[inst] = (flag == 2) ? ST_REBUILD : (flag == 3) ? ST_CONTINUE : ST_DONE;
    }
    cl.sync();
    TR();
    return;
  }
}

// ===========================================================================
// Staged ADMM replay (TMA-fed).
//
// The per-iteration matrix stream of an instance is static: the fused stage
// operators and the recorded scan matrices, in phase order.  Each CTA builds
// its own ordered item list once (the items of the stages / ops it owns) and
// streams the items through a ring of R shared-memory slots with 1-D bulk
// copies (cp.async.bulk, mbarrier complete_tx), R items ahead of the
// consumers, across phase and iteration boundaries.  Every matvec then reads
// shared memory only; the loads of the next items overlap the current
// phase's arithmetic, barriers and DSMEM exchanges.  All 16 warps work on one
// item at a time (row blocks x k-slices, partial sums combined in a fixed
// order), so an item costs two CTA barriers.
//
// Vectors are the replay vectors of k_replay with physical slot compression
// (plan.h compress_slots); y is not stored (y = lambda / rho after every
// ascent, admm.py:134).
// ===========================================================================

enum { IT_P1 = 0, IT_CVF1, IT_CVF2, IT_FF1, IT_FF2, IT_COT, IT_G };

constexpr int kTraceIter = 5;  // GSLS_REPLAY_TRACE samples this ADMM iteration (warm caches)

struct StagedLayout {
  // byte offsets into dynamic shared memory
  int ring, pv, bv, cb, t1, t2, w, kf, dx0, part, red, redall, masks, ops, phys, items, gseq, phase, mbar, total;
  int slot;  // bytes per ring slot
  int R;     // ring slots
  int max_items, nphase;
};

// Precomputed item: everything the item loop needs, so the hot path does no
// index arithmetic or integer division.  Vector operands are shared-memory
// byte offsets from the dynamic shared base (-1: none).
struct __align__(16) ItemDesc {
  const float* src;   // bulk-copy source
  const double* pre;  // global addend (leaf constants, kk0, b, f) or null
  unsigned bytes;
  int kind, rows, ld, K1, K2, kslog, kc;
  int x1, x2, add, dst, dst2;
  unsigned mask;
  int e0, pre2;  // E_G first row; 1: add Abar_0 dx0 (FF2, k = 0)
  double sgn;
};

__host__ __device__ inline int stage_slot_bytes(int n, int m, int c, int ld2n, int ldm, int ldn, int ldc, int ldg) {
  int b = 2 * n * ldg;                  // recorded n x 2n replay operator [Ups X] / [Psi -Y]
  b = b > c * ld2n ? b : c * ld2n;      // X23
  b = b > (n + c) * ldm ? b : (n + c) * ldm;
  b = b > m * ldn ? b : m * ldn;
  b = b > (n + m) * ldc ? b : (n + m) * ldc;
  return ((b * 4 + 127) / 128) * 128;
}

__host__ __device__ inline int staged_part_tasks(const DevLqr& L, int G) {  // partial tasks per group half
  const int W = (kReplayThreads / 32) / G;
  int rows = 2 * L.n;
  rows = rows > L.c ? rows : L.c;
  const int rb = (rows + 31) / 32;
  return W > rb ? W : rb;
}

__host__ __device__ inline StagedLayout staged_layout(const DevLqr& L, int max_layer, int R, int max_items, int G) {
  StagedLayout S{};
  const int n = L.n, m = L.m, N = L.N;
  int o = 0;
  auto take = [&](int bytes, int align) { o = (o + align - 1) / align * align; int r = o; o += bytes; return r; };
  S.slot = stage_slot_bytes(n, m, L.c, L.ld2n, L.ldm, L.ldn, L.ldc, L.ldg);
  S.R = R;
  S.ring = take(S.slot * R, 128);
  S.pv = take(L.cvf_nphys * n * 8, 16);
  S.bv = take(L.cvf_nphys * n * 8, 16);
  S.cb = take(L.cot_nphys * n * 8, 16);
  S.t1 = take(0, 16);  // (unused since the one-round CVF replay)
  S.t2 = take(0, 16);
  // z, lam, y stay in global memory (only their owner rows' G epilogue touches them)
  S.w = take(L.mtot * 8, 16);
  S.kf = take(N * m * 8, 16);
  S.dx0 = take(n * 8, 16);
  {  // per item group: two halves x max(W, row blocks) (row block, slice) tasks x 32 rows; also
     // holds the setup's item list (<= kReplayThreads int2)
    const int pb = G * 2 * staged_part_tasks(L, G) * 32 * 8;
    S.part = take(pb > 2 * kReplayThreads * 8 ? pb : 2 * kReplayThreads * 8, 16);
  }
  S.red = take(64 * 8, 16);
  S.redall = take(2 * kMaxCluster * 8, 16);
  S.masks = take((L.cvf_nslots + L.cot_nslots) * 4, 16);
  S.ops = take((L.cvf_nops + L.cot_nops) * 16 + (2 * L.cvf_layers + L.cot_layers + 2 + 2 * N + 2) * 4, 16);
  S.phys = take((L.cvf_nslots + L.cot_nslots) * 4, 16);
  S.max_items = max_items;
  S.items = take(S.max_items * (int)sizeof(ItemDesc), 16);
  S.gseq = take((S.max_items + 2 * 8 + 2) * 4, 16);  // per-group item sequences + offsets (<= 8 groups)
  S.nphase = L.cvf_layers + L.cot_layers + 5;
  S.phase = take((S.nphase + 1) * 4, 16);
  S.mbar = take(R * 8, 8);
  S.total = o;
  return S;
}

__device__ inline void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(count) : "memory");
}
__device__ inline void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ inline void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}

enum { E_SET = 0, E_PUT, E_P1, E_KF, E_CB, E_G };

// Epilogue of one item: what thread i < rows does with its row sum s.
struct ItemEpi {
  int kind;
  double* dst;         // output vector (E_P1: the p leaf)
  double* dst2;        // E_P1: the b leaf
  const double* add;   // shared-memory addend (E_SET, E_PUT)
  const double* pre;   // global addend, loaded before the wait (E_P1, E_KF, E_CB, E_G: f)
  const double* pre2;  // second global addend (E_CB at k = 0: Abar_0 dx0)
  double sgn;
  unsigned mask;       // consumer ranks (E_PUT, E_P1, E_CB)
  int e0;              // E_G: first stacked constraint row of the stage
};

// G item groups (compile-time: the index arithmetic of the hot loop folds for each size)
template <int G>
__global__ void __launch_bounds__(kReplayThreads, 1) k_admm_staged(ReplayArgs a, int R, int max_items) {
  const DevLqr& L = a.L;
  if (a.count && (int)blockIdx.y >= *a.count) return;
  const int inst = a.list ? a.list[blockIdx.y] : (int)blockIdx.y;
  if (L.err[inst].key != 0) {  // its (re)build raised: the host driver decides
    if (cluster_rank() == 0 && threadIdx.x == 0) a.status[inst] = ST_BUILD_ERR;
    return;
  }
  const int n = L.n, m = L.m, c = L.c, nf = L.nf, N = L.N, ldg = L.ldg, mtot = L.mtot;
  const size_t MS = (size_t)n * ldg;
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
  Cl cl;
  cl.rank = cluster_rank();
  cl.cs = cluster_size();
  const int rank = (int)cl.rank, cs = (int)cl.cs;
  const StagedLayout SL = staged_layout(L, a.max_layer, R, max_items, G);
  extern __shared__ __align__(128) unsigned char smb[];
  unsigned char* ring = smb + SL.ring;
  double* pv = reinterpret_cast<double*>(smb + SL.pv);
  double* bv = reinterpret_cast<double*>(smb + SL.bv);
  double* cb = reinterpret_cast<double*>(smb + SL.cb);
  // z, lam, y of the constraint rows live in global memory: a row is read and written only by
  // its owning rank's G epilogue, once per iteration, with the reads issued before the item's
  // wait (shared memory holds w = y - z, the vector the matvecs read)
  double* z = a.state.z + (size_t)inst * L.mtot;
  double* lam = a.state.lam + (size_t)inst * L.mtot;
  double* y = a.state.y + (size_t)inst * L.mtot;
  double* w = reinterpret_cast<double*>(smb + SL.w);
  double* kf = reinterpret_cast<double*>(smb + SL.kf);
  double* dx0s = reinterpret_cast<double*>(smb + SL.dx0);
  double* part = reinterpret_cast<double*>(smb + SL.part);
  double* red = reinterpret_cast<double*>(smb + SL.red);
  double* redall = reinterpret_cast<double*>(smb + SL.redall);
  unsigned* cvf_mask = reinterpret_cast<unsigned*>(smb + SL.masks);
  unsigned* cot_mask = cvf_mask + L.cvf_nslots;
  int4* s_cvf_ops = reinterpret_cast<int4*>(smb + SL.ops);
  int4* s_cot_ops = s_cvf_ops + L.cvf_nops;
  int* s_cvf_loff = reinterpret_cast<int*>(s_cot_ops + L.cot_nops);
  int* s_cot_loff = s_cvf_loff + L.cvf_layers + 1;
  int* s_cvf_out = s_cot_loff + L.cot_layers + 1;
  int* s_cot_out = s_cvf_out + N + 1;
  int* s_cvf_blive = s_cot_out + N;
  int* cvf_phys = reinterpret_cast<int*>(smb + SL.phys);
  int* cot_phys = cvf_phys + L.cvf_nslots;
  ItemDesc* desc = reinterpret_cast<ItemDesc*>(smb + SL.items);
  int2* items = reinterpret_cast<int2*>(smb + SL.part);  // setup only: (kind | which << 8 | loc << 16, index)
  int* phase_off = reinterpret_cast<int*>(smb + SL.phase);
  int* gseq = reinterpret_cast<int*>(smb + SL.gseq);  // [P] items in group consumption order
  int* goff = gseq + max_items;                        // [G + 1] group offsets into gseq
  uint64_t* full = reinterpret_cast<uint64_t*>(smb + SL.mbar);
  __shared__ int s_flag, s_nitems;
  __shared__ double s_rho;

  // ---- one-time setup: plan, physical slots, consumer masks, item list ------------
  for (int i = tid; i < L.cvf_nops; i += nthr) s_cvf_ops[i] = L.cvf_ops[i];
  for (int i = tid; i < L.cot_nops; i += nthr) s_cot_ops[i] = L.cot_ops[i];
  for (int i = tid; i <= L.cvf_layers; i += nthr) s_cvf_loff[i] = L.cvf_loff[i];
  for (int i = tid; i <= L.cot_layers; i += nthr) s_cot_loff[i] = (N > 0) ? L.cot_loff[i] : 0;
  for (int i = tid; i <= N; i += nthr) s_cvf_out[i] = L.cvf_out[i];
  for (int i = tid; i < N; i += nthr) s_cot_out[i] = L.cot_out[i];
  for (int i = tid; i < L.cvf_layers; i += nthr) s_cvf_blive[i] = L.cvf_blive[i];
  for (int i = tid; i < L.cvf_nslots; i += nthr) cvf_phys[i] = L.cvf_phys[i];
  for (int i = tid; i < L.cot_nslots; i += nthr) cot_phys[i] = L.cot_phys[i];
  for (int i = tid; i < L.cvf_nslots + L.cot_nslots; i += nthr) cvf_mask[i] = 0u;
  if (tid < R) mbar_init(full + tid, 1);
  __syncthreads();
  auto srank = [&](int k) { return k % cs; };
  if (cs > 1) {
    for (int lay = 0; lay < L.cvf_layers; ++lay) {  // half-op h on rank h / per (cvf_half)
      const int o0 = s_cvf_loff[lay], no = s_cvf_loff[lay + 1] - o0, nh = no + s_cvf_blive[lay];
      const int per = (nh + cs - 1) / cs;
      for (int h = tid; h < nh; h += nthr) {
        const int4 op = s_cvf_ops[o0 + (h < no ? h : h - no)];
        atomicOr(cvf_mask + op.y, 1u << (h / per));
        atomicOr(cvf_mask + op.z, 1u << (h / per));
      }
    }
    for (int p = tid; p <= N; p += nthr) atomicOr(cvf_mask + s_cvf_out[p], 1u << srank(max(p - 1, 0)));
    for (int lay = 0; lay < L.cot_layers; ++lay) {
      const int o0 = s_cot_loff[lay], no = s_cot_loff[lay + 1] - o0, per = (no + cs - 1) / cs;
      for (int oi = tid; oi < no; oi += nthr) {
        const int4 op = s_cot_ops[o0 + oi];
        atomicOr(cot_mask + op.y, 1u << (oi / per));
        atomicOr(cot_mask + op.z, 1u << (oi / per));
      }
    }
    for (int k = 1 + tid; k <= N; k += nthr) atomicOr(cot_mask + s_cot_out[k - 1], 1u << srank(k));
  }
  if (tid == 0) {  // this rank's items in consumption order, phase by phase
    int ni = 0, ph = 0;
    auto add = [&](int kind, int which, int idx, int loc = 0) {
      items[ni++] = make_int2(kind | (which << 8) | (loc << 16), idx);
    };
    phase_off[ph++] = ni;
    for (int k = rank; k < N; k += cs) add(IT_P1, 0, k);
    for (int lay = 0; lay < L.cvf_layers; ++lay) {
      // half-ops: p = p_e + [Ups X] [p_l; b_e] (which 0) for every op (h < no), then
      // b = b_l + [Psi -Y] [b_e; p_l] (which 1) for the layer's first s_cvf_blive ops (the
      // others' results are read by no later op, so their b is dead)
      const int o0 = s_cvf_loff[lay], no = s_cvf_loff[lay + 1] - o0, nh = no + s_cvf_blive[lay];
      const int per = (nh + cs - 1) / cs;
      const int lo = min(nh, rank * per), hi = min(nh, lo + per);
      phase_off[ph++] = ni;
      for (int h = lo; h < hi; ++h) add(IT_CVF1, h < no ? 0 : 1, o0 + (h < no ? h : h - no));
    }
    phase_off[ph++] = ni;
    for (int k = rank; k < N; k += cs) add(IT_FF1, 0, k);
    phase_off[ph++] = ni;
    for (int k = rank; k < N; k += cs) add(IT_FF2, 0, k);
    for (int lay = 0; lay < L.cot_layers; ++lay) {
      const int o0 = s_cot_loff[lay], no = s_cot_loff[lay + 1] - o0, per = (no + cs - 1) / cs;
      const int lo = min(no, rank * per), hi = min(no, lo + per);
      phase_off[ph++] = ni;
      for (int oi = lo; oi < hi; ++oi) add(IT_COT, 0, o0 + oi);
    }
    phase_off[ph++] = ni;
    for (int k = rank; k < N; k += cs) add(IT_G, 0, k);
    phase_off[ph] = ni;
    s_nitems = ni;
    // group g consumes the items j of every phase with (j - phase start) = g (mod G), in order
    int o = 0;
    for (int g = 0; g < G; ++g) {
      goff[g] = o;
      for (int q = 0; q < ph; ++q)
        for (int jj = phase_off[q] + g; jj < phase_off[q + 1]; jj += G) gseq[o++] = jj;
    }
    goff[G] = o;
  }
  // fence: mbarrier inits visible to the async proxy before the first bulk copy
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int P = s_nitems;

  // ---- instance data --------------------------------------------------------------
  const size_t sN = (size_t)inst * N;
  const double* bq = a.qp.b + sN * n;
  const float* CNq = a.qp.CN + (size_t)inst * nf * n;
  const double* qN_lin = a.qp.qN + (size_t)inst * n;
  const float* Kg = L.K + sN * m * n;
  const double* v0 = L.v0 + (size_t)inst * n;
  const float* cvf_rec = L.cvf_rec + (size_t)inst * L.cvf_nops * 4 * MS;
  const float* cot_rec = L.cot_rec + (size_t)inst * L.cot_nops * MS;
  const float* X23 = L.X23 + sN * c * L.ld2n;
  const double* pb0 = L.pb0 + sN * 2 * n;
  const float* XK = L.XK + sN * (n + c) * L.ldm;
  const double* kk0 = L.kk0 + sN * m;
  const float* Bcm = L.Bcm + sN * m * L.ldn;
  const float* ZD = L.ZD + sN * (n + m) * L.ldc;
  const double* fst = a.qp.f + sN * c;
  const double* fN = a.qp.fN + (size_t)inst * nf;
  auto PV = [&](int s) { return pv + (size_t)cvf_phys[s] * n; };
  auto BV = [&](int s) { return bv + (size_t)cvf_phys[s] * n; };
  auto CB = [&](int s) { return cb + (size_t)cot_phys[s] * n; };
  auto dxp = [&](int k) -> const double* { return k == 0 ? dx0s : CB(s_cot_out[k - 1]); };

  // ---- item descriptors (parallel over items) ------------------------------------------
  {
    auto off = [&](const void* p) { return p ? (int)((const unsigned char*)p - smb) : -1; };
    for (int j = tid; j < P; j += nthr) {
      const int2 itm = items[j];
      const int kind = itm.x & 0xff, which = (itm.x >> 8) & 0xff, idx = itm.y;
      ItemDesc d{};
      d.kind = kind; d.rows = n; d.ld = ldg; d.K1 = n; d.K2 = 0; d.x2 = -1; d.add = -1; d.dst2 = -1;
      d.sgn = 1.0; d.pre = nullptr; d.pre2 = 0; d.mask = 0u; d.e0 = 0;
      d.bytes = (unsigned)MS * 4;
      switch (kind) {
        case IT_P1:  // [p; b]_k = pb0_k + X23_k w_k (fused leaves, admm.py:113-121, lqr.py:338-342)
          d.src = X23 + (size_t)idx * c * L.ld2n; d.bytes = c * L.ld2n * 4;
          d.rows = 2 * n; d.ld = L.ld2n; d.K1 = c; d.x1 = off(w + idx * c);
          d.dst = off(PV(idx)); d.dst2 = off(BV(idx)); d.pre = pb0 + (size_t)idx * 2 * n; d.mask = cvf_mask[idx];
          break;
        case IT_CVF1: {  // p = p_e + [Ups X] [p_l; b_e] | b = b_l + [Psi -Y] [b_e; p_l] (lqr.py:242-246)
          const int4 op = s_cvf_ops[idx];
          d.src = cvf_rec + ((size_t)idx * 4 + 2 * which) * MS;  // n x 2n column-major operator
          d.bytes = (unsigned)MS * 8;
          d.K1 = n; d.K2 = n;
          d.x1 = off(which ? BV(op.y) : PV(op.z));
          d.x2 = off(which ? PV(op.z) : BV(op.y));
          d.add = off(which ? BV(op.z) : PV(op.y));
          d.dst = off(which ? BV(op.x) : PV(op.x));
          d.mask = cvf_mask[op.x];
          break;
        }
        case IT_FF1:  // kf = kk0 + [X5 X4] [p+; w] (lqr.py:345-346)
          d.src = XK + (size_t)idx * (n + c) * L.ldm; d.bytes = (n + c) * L.ldm * 4;
          d.rows = m; d.ld = L.ldm; d.K1 = n; d.x1 = off(PV(s_cvf_out[idx + 1])); d.K2 = c; d.x2 = off(w + idx * c);
          d.dst = off(kf + idx * m); d.pre = kk0 + (size_t)idx * m;
          break;
        case IT_FF2:  // COT leaf b = B kf + b (+ Abar_0 dx0) (lqr.py:349-356)
          d.src = Bcm + (size_t)idx * m * L.ldn; d.bytes = m * L.ldn * 4;
          d.rows = n; d.ld = L.ldn; d.K1 = m; d.x1 = off(kf + idx * m);
          d.dst = off(CB(idx)); d.pre = bq + (size_t)idx * n; d.pre2 = (idx == 0); d.mask = cot_mask[idx];
          break;
        case IT_COT: {  // b = A_later b_earlier + b_later (lqr.py:281-285)
          const int4 op = s_cot_ops[idx];
          d.src = cot_rec + (size_t)idx * MS;
          d.x1 = off(CB(op.y)); d.add = off(CB(op.z)); d.dst = off(CB(op.x)); d.mask = cot_mask[op.x];
          break;
        }
        default:  // G = [Z D] [dx; kf] = C dx + D du, then the projection (admm.py:91-97)
          d.src = ZD + (size_t)idx * (n + m) * L.ldc; d.bytes = (n + m) * L.ldc * 4;
          d.rows = c; d.ld = L.ldc; d.K1 = n; d.x1 = off(dxp(idx)); d.K2 = m; d.x2 = off(kf + idx * m);
          d.pre = fst + (size_t)idx * c; d.e0 = idx * c;
          break;
      }
      const int RB = (d.rows + 31) >> 5;
      const int Wg = (nthr >> 5) / G;  // warps of an item group
      int kslog = 0;  // KS = W / RB (power of two): one group's partial half holds <= max(W, RB) tasks
      while ((1 << (kslog + 1)) <= Wg && (RB << (kslog + 1)) <= Wg) ++kslog;  // (rows = 0: KS = W)
      const int KS = 1 << kslog, K = d.K1 + d.K2;
      d.kslog = kslog;
      d.kc = (((K + KS - 1) / KS) + 3) & ~3;
      desc[j] = d;
    }
  }
  __syncthreads();
  // Ring schedule: group g owns slots g, g + G, ... (Rg = R / G of them) and consumes its
  // item sequence gseq[goff[g] ..] in order, so every slot has one consumer that waits on
  // its phases in order (no mbarrier parity aliasing between groups).  The group's t-th
  // item of this launch sits in slot g + G (t mod Rg); after reading it the group refills
  // the slot with its item t + Rg.
  const int W = (nthr >> 5) / G, grp = warp / W, wg = warp - grp * W, gtid = tid - grp * W * 32, gsz = W * 32;
  const int Rg = R / G, g0 = goff[grp], Pg = goff[grp + 1] - g0;
  const int issuer = gsz - 32;  // the group's last warp: off the epilogue's first rows
  if (gtid == issuer && Pg > 0)
    for (int t = 0; t < Rg; ++t) {
      const int jj = gseq[g0 + t % Pg], sl = grp + G * t;
      bulk_load(ring + (size_t)sl * SL.slot, desc[jj].src, desc[jj].bytes, full + sl);
    }

  double rho = a.state.rho[inst];
  int it = a.stats.iterations[inst];
  {
    for (int e = tid; e < mtot; e += nthr) w[e] = y[e] - z[e];
    for (int i = tid; i < n; i += nthr) dx0s[i] = a.qp.dx0[(size_t)inst * n + i];
  }
  cl.sync();  // every replica exists before the first remote store

  // Item groups: G groups of W warps take the items of a phase round-robin, each group with
  // its own named barrier, ring slots and partial-sum halves, so up to G items are in flight
  // per CTA (small clusters hold many items per rank and phase; G = 1 at 16-CTA clusters).
  const int PT = staged_part_tasks(L, G) * 32;  // doubles per group half
  // partial half; ring position (0 .. Rg-1) and parity; sequence position of the next refill
  int half = 0, gi = 0, gpar = 0, rpos = Pg > 0 ? Rg % Pg : 0;
  const int nph = L.cvf_layers + L.cot_layers + 4;  // P1, CVF layers, FF1, FF2, COT layers, G
  const int ph_ff1 = L.cvf_layers + 1, ph_g = nph - 1;

  int tr_it = 0;
  for (;;) {
    double rp = 0.0, rdz = 0.0;
    if (a.trace && tid == 0 && rank == 0 && blockIdx.y == 0 && tr_it == kTraceIter) a.trace[250] = clock64();
    for (int ph = 0; ph < nph; ++ph) {
      // ---- the phase's items: one matvec each, read from the ring ------------------------
      for (int j = phase_off[ph] + grp; j < phase_off[ph + 1]; j += G) {
        const ItemDesc& d = desc[j];
        const int rows = d.rows, ld = d.ld, K1 = d.K1, kind = d.kind;
        const double* x1 = reinterpret_cast<const double*>(smb + d.x1);
        const double* x2 = reinterpret_cast<const double*>(smb + (d.x2 < 0 ? d.x1 : d.x2));
        double pre_v = 0.0;  // global addend of this thread's first row, loaded before the wait
        if (gtid < rows && d.pre) pre_v = d.pre[gtid] + (d.pre2 ? v0[gtid] : 0.0);
        double zo_v = 0.0, y_v = 0.0, l_v = 0.0;  // G rows: the ADMM state, loaded before the wait
        if (kind == IT_G && gtid < rows) {
          const int e = d.e0 + gtid;
          zo_v = z[e];
          y_v = y[e];
          l_v = lam[e];
        }
        const int slot = grp + G * gi;
        mbar_wait(full + slot, (unsigned)gpar);
        const float* M = reinterpret_cast<const float*>(ring + (size_t)slot * SL.slot);
        double* pt = part + (size_t)(2 * grp + half) * PT;
        const int kslog = d.kslog, KS = 1 << kslog, kc = d.kc, K = K1 + d.K2;
        const int ntask = ((rows + 31) >> 5) << kslog;
        for (int t = wg; t < ntask; t += (G == 1 ? ntask : W)) {  // G = 1: ntask <= 16 warps, one task each
          const int rb = t >> kslog, ks = t & (KS - 1);
          const int rq = lane & 7, gq = lane >> 3;
          const int row0 = rb * 32 + 4 * rq;
          const int k0 = ks * kc, k1 = min(K, k0 + kc);
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          if (row0 < ld) {
#pragma unroll 4
            for (int k = k0 + gq; k < k1; k += 4) {
              const uint4 v = *reinterpret_cast<const uint4*>(M + k * ld + row0);
              const double xk = (k < K1) ? x1[k] : x2[k - K1];
              // rows 0-1 widen on the conversion pipe, rows 2-3 on the integer pipe (scaled)
              a0 = fma((double)__uint_as_float(v.x), xk, a0);
              a1 = fma((double)__uint_as_float(v.y), xk, a1);
              a2 = fma(widen_scaled(v.z), xk, a2);
              a3 = fma(widen_scaled(v.w), xk, a3);
            }
            a2 *= kWidenUnscale;
            a3 *= kWidenUnscale;
          }
#pragma unroll
          for (int o = 8; o <= 16; o <<= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, o);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o);
            a2 += __shfl_xor_sync(0xffffffffu, a2, o);
            a3 += __shfl_xor_sync(0xffffffffu, a3, o);
          }
          if (gq == 0) {
            double* pp = pt + (t << 5) + 4 * rq;  // (rb * KS + ks) * 32
            pp[0] = a0; pp[1] = a1; pp[2] = a2; pp[3] = a3;
          }
        }
        // One (group) barrier per item: the slot is refilled right after it and the partial
        // sums alternate halves, so this epilogue overlaps the group's next item.
        if (G == 1) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(gsz) : "memory");
        if (gtid == issuer) {  // the group's item Rg positions on (its sequence wraps per iteration)
          const int jn = gseq[g0 + rpos];
          bulk_load(ring + (size_t)slot * SL.slot, desc[jn].src, desc[jn].bytes, full + slot);
        }
        if (++rpos == Pg) rpos = 0;
        if (++gi == Rg) { gi = 0; gpar ^= 1; }
        half ^= 1;
        auto epi = [&](int i, double pv_) {
          const double* pr = pt + (((i >> 5) << kslog) << 5) + (i & 31);
          double sum = 0.0;
          for (int ks = 0; ks < KS; ++ks) sum += pr[ks << 5];
          double* dst = reinterpret_cast<double*>(smb + d.dst);
          switch (kind) {
            case IT_CVF1:
            case IT_COT:
              cl.put_mask(dst + i, reinterpret_cast<const double*>(smb + d.add)[i] + d.sgn * sum, d.mask);
              break;
            case IT_P1:
              cl.put_mask(i < n ? dst + i : reinterpret_cast<double*>(smb + d.dst2) + (i - n), pv_ + sum, d.mask);
              break;
            case IT_FF1: dst[i] = pv_ + sum; break;
            case IT_FF2: cl.put_mask(dst + i, pv_ + sum, d.mask); break;
            default: {  // z = min(G + y, f); lam += rho (G - z); y = lam / rho (admm.py:130-135)
              const int e = d.e0 + i;
              const bool own = i == gtid;
              const double zo = own ? zo_v : z[e];
              const double zn = fmin(sum + (own ? y_v : y[e]), pv_);
              const double ln = (own ? l_v : lam[e]) + rho * (sum - zn);
              const double yn = ln / rho;
              lam[e] = ln;
              y[e] = yn;
              z[e] = zn;
              w[e] = yn - zn;
              rp = fmax(rp, fabs(sum - zn));
              rdz = fmax(rdz, fabs(zn - zo));
            }
          }
        };
        if (gtid < rows) epi(gtid, pre_v);
        if (G > 1)
          for (int i = gtid + gsz; i < rows; i += gsz)  // rows beyond the group (P1 items of n > 64 at W = 4)
          epi(i, d.pre ? d.pre[i] + (d.pre2 ? v0[i] : 0.0) : 0.0);
      }
      // ---- phase boundary -----------------------------------------------------------
      if (a.trace && tid == 0 && rank == 0 && blockIdx.y == 0 && tr_it == kTraceIter && 2 * ph + 1 < 250)
        a.trace[2 * ph + 1] = clock64();
      if (ph == 0) {  // terminal leaf (qN + rho CN' w_N, 0) on its owner
        if (rank == srank(N))
          for (int i = tid; i < n; i += nthr) {
            double sum = 0.0;
            for (int f = 0; f < nf; ++f) sum = fma((double)CNq[f * n + i], w[N * c + f], sum);
            cl.put_mask(PV(N) + i, qN_lin[i] + rho * sum, cvf_mask[N]);
            cl.put_mask(BV(N) + i, 0.0, cvf_mask[N]);
          }
        cl.sync();
      } else if (ph == ph_g) {  // terminal constraint rows on their owner
        if (rank == srank(N))
          for (int f = tid; f < nf; f += nthr) {
            const double* xN = dxp(N);
            double sum = 0.0;
            for (int i = 0; i < n; ++i) sum = fma((double)CNq[f * n + i], xN[i], sum);
            const int e = N * c + f;
            const double zo = z[e];
            const double zn = fmin(sum + y[e], fN[f]);
            const double ln = lam[e] + rho * (sum - zn);
            const double yn = ln / rho;
            lam[e] = ln;
            y[e] = yn;
            z[e] = zn;
            w[e] = yn - zn;
            rp = fmax(rp, fabs(sum - zn));
            rdz = fmax(rdz, fabs(zn - zo));
          }
      } else if (ph == ph_ff1) {
        __syncthreads();  // kf complete (CTA-local)
      } else {
        cl.sync();  // CVF layers, FF2, COT layers: remote consumers
      }
      if (a.trace && tid == 0 && rank == 0 && blockIdx.y == 0 && tr_it == kTraceIter && 2 * ph + 2 < 250)
        a.trace[2 * ph + 2] = clock64();
    }
    if (a.trace && tid == 0 && rank == 0 && blockIdx.y == 0 && tr_it == kTraceIter) a.trace[0] = nph;
    ++tr_it;
    const double rpb = block_max_d(rp, red);
    const double rdb = block_max_d(rdz, red + 32);
    if (tid == 0) {
      cl.put(redall + 2 * rank, rpb);
      cl.put(redall + 2 * rank + 1, rdb);
    }
    cl.sync();
    if (tid == 0) {
      double r_p = 0.0, r_dz = 0.0;
      for (int r = 0; r < cs; ++r) {
        r_p = fmax(r_p, redall[2 * r]);
        r_dz = fmax(r_dz, redall[2 * r + 1]);
      }
      ++it;
      const double r_d = rho * r_dz;
      const bool lead = rank == 0;
      if (lead) {
        a.state.iteration[inst] += 1;
        a.state.r_primal[inst] = r_p;
        a.state.r_dual[inst] = r_d;
      }
      int flag = 0;
      double rho_new = rho;
      if (r_p <= a.set.tol_primal && r_d <= a.set.tol_dual) {
        if (lead) a.stats.converged[inst] = 1;
        flag = 1;
      } else {
        bool changed = false;
        if (it % a.set.sigma == 0) {
          const double ratio = sqrt(fmax(r_p, 1e-30) / fmax(r_d, 1e-30));
          const double prop = fmin(fmax(rho * ratio, a.set.rho_min), a.set.rho_max);
          if (prop > 5.0 * rho || prop < rho / 5.0) {
            rho_new = prop;
            if (lead) {
              a.state.rho[inst] = prop;
              a.state.generation[inst] += 1;
              a.stats.rho_changes[inst] += 1;
            }
            changed = true;
          }
        }
        if (it >= a.set.max_iter) flag = 1;
        else if (changed) flag = 2;
        else if (a.cap > 0 && it >= a.cap) flag = 3;  // paused: resumes bitwise-identically in the next launch
      }
      if (lead) a.stats.iterations[inst] = it;
      s_flag = flag;
      s_rho = rho_new;
    }
    __syncthreads();
    const int flag = s_flag;
    if (flag == 0) continue;

    // ---- exit: drain the in-flight bulk copies, write back what this rank owns -------
    if (Pg > 0)  // the group's Rg in-flight copies land in its next ring positions, in order
      for (int q = 0, sl = gi, pa = gpar; q < Rg; ++q) {
        mbar_wait(full + grp + G * sl, (unsigned)pa);
        if (++sl == Rg) { sl = 0; pa ^= 1; }
      }
    __syncthreads();
    const double rho_new = s_rho;
    auto owns_row = [&](int e) { return srank(e < N * c ? e / c : N) == rank; };
    if (rho_new != rho)  // a committed change rescales y (admm.py:149); z, lam are already in place
      for (int e = tid; e < mtot; e += nthr)
        if (owns_row(e)) y[e] = lam[e] / rho_new;
    if (flag == 1) {
      double* gdx = a.dx + (size_t)inst * (N + 1) * n;
      double* gdu = a.du + (size_t)inst * N * m;
      for (int e = tid; e < (N + 1) * n; e += nthr) {
        const int p = e / n, i = e - p * n;
        if ((p == 0 ? 0 : srank(p)) == rank) gdx[e] = dxp(p)[i];
        if (srank(max(p - 1, 0)) == rank) L.last_p[(size_t)inst * (N + 1) * n + e] = PV(s_cvf_out[p])[i];
      }
      for (int e = tid; e < N * m; e += nthr) {  // du = K dx + k (lqr.py:359-363), once at exit
        const int k = e / m;
        if (srank(k) != rank) continue;
        const double* xk = dxp(k);
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = fma((double)Kg[(size_t)e * n + i], xk[i], s);
        gdu[e] = s + kf[e];
        L.last_k[(size_t)inst * N * m + e] = kf[e];
      }
    }
    if (rank == 0 && tid == 0) a.status[inst] = (flag == 2) ? ST_REBUILD : (flag == 3) ? ST_CONTINUE : ST_DONE;
    cl.sync();
    return;
  }
}

// ---------------------------------------------------------------------------
// host side

// Cluster size for a replay launch: spread each instance over up to 16 SMs
// while the whole batch still fits in one wave (small batches are latency-
// bound on one SM's L2 bandwidth); 1 for large batches.  GSLS_REPLAY_CLUSTER
// overrides (power of two <= 16).
static int replay_cluster(Ctx* c, int count, size_t smem_bytes, const void* kern) {
  if (c->d_scratch) return 1;  // vectors in global memory: no DSMEM replicas
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int want = 16;
  if (const char* e = getenv("GSLS_REPLAY_CLUSTER")) want = std::max(1, std::min(16, atoi(e)));
  // any size up to 16 (the staged kernel's ownership is k mod cs / ceil(ops / cs)): the
  // ADMM tail's few remaining instances spread over every SM (e.g. 49 instances x 3)
  const char* p2 = getenv("GSLS_REPLAY_CLUSTER_POW2");
  for (int cs = want; cs >= 2; cs = (p2 && p2[0] == '1') ? cs >> 1 : cs - 1) {
    if ((long long)count * cs > sms) continue;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs, count);
    cfg.blockDim = dim3(kReplayThreads);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (ncl >= count) return cs;
  }
  return 1;
}

static int launch_replay(Ctx* c, ReplayArgs& a, int count, cudaStream_t st) {
  if (count == 0) return GSLS_OK;
  a.L = c->dev;
  {
    const char* pf = getenv("GSLS_REPLAY_PREFETCH");
    a.prefetch = pf ? (pf[0] - '0') : 1;  // 0 off, 1 the next layer's records, 2 also stage operators
  }
  a.max_layer = std::max(1, std::max(c->cvf_max_layer, c->cot_max_layer));
  size_t sb = 0;
  if (c->d_scratch) {
    a.gscratch = c->d_scratch;
    a.scratch_floats = (long long)c->scratch_floats;
  } else {
    a.gscratch = nullptr;
    a.scratch_floats = 0;
    sb = c->scratch_floats * sizeof(double);
  }
  static bool attrs_set = false;
  if (!attrs_set) {
    GSLS_CUDA_CHECK(cudaFuncSetAttribute((const void*)k_replay<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kReplaySmemMax)));
    attrs_set = true;
  }
  // Vectors too large for shared memory (long horizons, e.g. cfg-E at N = 2047): each
  // instance runs over the whole GPU as a cooperative grid (k_replay<true>), instances in
  // turn.  GSLS_REPLAY_GRID=0 keeps one CTA per instance (diagnostics).
  const char* genv = getenv("GSLS_REPLAY_GRID");
  if (c->d_scratch && !(genv && genv[0] == '0')) {
    const size_t gsb = (64 + kReplayThreads) * sizeof(double);
    static int per_sm = 0, sms = 0;
    if (!per_sm) {
      int dev = 0;
      GSLS_CUDA_CHECK(cudaGetDevice(&dev));
      GSLS_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      GSLS_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_replay<true>, kReplayThreads, gsb));
      if (per_sm < 1) per_sm = 1;
    }
    const int grid = per_sm * sms;
    ProfScope ps(P_REPLAY, st, (double)count);
    for (int i = 0; i < count; ++i) {
      ReplayArgs ai = a;
      ai.list = (a.list ? a.list : c->d_inst_all) + i;
      ai.trace = nullptr;
      void* args[] = {&ai};
      GSLS_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_replay<true>, dim3(grid, 1), dim3(kReplayThreads), args,
                                                  gsb, st));
    }
    GSLS_CUDA_CHECK(cudaGetLastError());
    return GSLS_OK;
  }
  // One CTA per instance (cluster launches of the ADMM loop go to k_admm_staged).
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1, count);
  cfg.blockDim = dim3(kReplayThreads);
  cfg.dynamicSmemBytes = sb;
  cfg.stream = st;
  cfg.attrs = nullptr;
  cfg.numAttrs = 0;
  static unsigned long long* trace = nullptr;
  const bool tracing = getenv("GSLS_REPLAY_TRACE") != nullptr;
  if (tracing && !trace) GSLS_CUDA_CHECK(cudaMalloc(&trace, 256 * sizeof(unsigned long long)));
  a.trace = tracing ? trace : nullptr;
  if (tracing) GSLS_CUDA_CHECK(cudaMemsetAsync(trace, 0, 256 * sizeof(unsigned long long), st));
  {
    ProfScope ps(P_REPLAY, st, (double)count);
    GSLS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_replay<false>, a));
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  if (tracing) {
    unsigned long long h[256];
    GSLS_CUDA_CHECK(cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st));
    GSLS_CUDA_CHECK(cudaStreamSynchronize(st));
    fprintf(stderr, "replay trace count=%d:", count);
    for (unsigned long long i = 2; i <= h[0]; ++i) fprintf(stderr, " %.2f", (h[i] - h[i - 1]) * 1e-3);
    fprintf(stderr, " | first iteration %.2f us | mv_round layer 3:", h[0] > 1 ? (h[h[0]] - h[1]) * 1e-3 : 0.0);
    for (int j = 1; j < 5; ++j) fprintf(stderr, " %llu", h[200 + j] - h[200 + j - 1]);
    fprintf(stderr, " cycles");
    fprintf(stderr, "\n");
  }
  return GSLS_OK;
}

// Staged ADMM launch: ring slots R chosen to fill shared memory (2..8); returns
// GSLS_ERR_TOO_LARGE when even R = 2 does not fit (the caller falls back to k_replay).
static int launch_admm_staged(Ctx* c, ReplayArgs& a, int count, cudaStream_t st) {
  if (count == 0) return GSLS_OK;
  a.L = c->dev;
  a.max_layer = std::max(1, std::max(c->cvf_max_layer, c->cot_max_layer));
  a.gscratch = nullptr;
  a.scratch_floats = 0;
  a.trace = nullptr;
  const size_t limit = 227 * 1024 - 1024;
  static bool attrs_set = false;
  if (!attrs_set) {
    for (const void* k : {(const void*)k_admm_staged<1>, (const void*)k_admm_staged<2>, (const void*)k_admm_staged<4>}) {
      GSLS_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit));
      GSLS_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    attrs_set = true;
  }
  // items per rank bound for the largest cluster this batch can use (fewer ranks -> more items)
  const int cs0 = replay_cluster(c, count, limit, (const void*)k_admm_staged<1>);  // occupancy at the largest footprint
  // item groups (k_admm_staged): small clusters hold many items per rank and phase, so up to
  // 4 items run concurrently there; 16-CTA clusters (batch-1 latency) hold 1-2 per phase
  // (measured, q61 / h75: 4 groups of 4 warps on clusters <= 4 cut the B = 1024 ADMM tail
  // waves 1.66 -> 0.94 ms; at 16-CTA clusters 2 groups are fastest for batch-1 latency)
  int G = cs0 <= 4 ? 4 : 2;
  if (const char* ge = getenv("GSLS_STAGED_GROUPS")) G = std::max(1, std::min(8, atoi(ge)));
  G = G >= 4 ? 4 : (G >= 2 ? 2 : 1);  // groups of 4 / 8 / 16 warps (ring slots per group >= 2)
  const int Nn = c->dims.N;
  auto cdiv = [](int x, int y) { return (x + y - 1) / y; };
  int max_items = 4 * cdiv(Nn, cs0) + 8;
  for (int l = 0; l < c->cvf.layers; ++l) max_items += cdiv(2 * (c->cvf_layer_off[l + 1] - c->cvf_layer_off[l]), cs0);
  for (int l = 0; l < c->cot.layers; ++l) max_items += cdiv(c->cot_layer_off[l + 1] - c->cot_layer_off[l], cs0);
  if (max_items > kReplayThreads) return GSLS_ERR_TOO_LARGE;  // setup list lives in the partial buffer
  int R = 0;
  size_t sb = 0;
  int min_rg = 1;
  if (const char* e = getenv("GSLS_STAGED_MIN_RG")) min_rg = std::max(1, atoi(e));
  for (;;) {  // R: the largest multiple of G (ring slots per group) that fits, >= min_rg per group if G > 1
    for (int r = 8; r >= 2; --r) {
      if (r % G || (G > 1 && r / G < min_rg)) continue;
      const StagedLayout SL = staged_layout(c->dev, a.max_layer, r, max_items, G);
      if ((size_t)SL.total <= limit) { R = r; sb = SL.total; break; }
    }
    if (R || G == 1) break;
    G >>= 1;
  }
  if (R == 0) return GSLS_ERR_TOO_LARGE;
  const int cs = cs0;
  if (getenv("GSLS_REPLAY_VERBOSE"))
    fprintf(stderr, "staged replay: count=%d cs=%d R=%d G=%d max_items=%d smem=%zu\n", count, cs, R, G, max_items, sb);
  // One CTA per instance (large batches) too: with 4 item groups the staged stream keeps
  // more operator bytes in flight than k_replay's layer rounds (B = 1024, 10-iteration wave
  // of 1024 instances: 14.1 vs 17.8 ms); GSLS_REPLAY_STAGED=0 selects k_replay (A/B).
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(cs, count);
  cfg.blockDim = dim3(kReplayThreads);
  cfg.dynamicSmemBytes = sb;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static unsigned long long* trace = nullptr;
  const bool tracing = getenv("GSLS_REPLAY_TRACE") != nullptr;
  if (tracing && !trace) GSLS_CUDA_CHECK(cudaMalloc(&trace, 256 * sizeof(unsigned long long)));
  a.trace = tracing ? trace : nullptr;
  if (tracing) GSLS_CUDA_CHECK(cudaMemsetAsync(trace, 0, 256 * sizeof(unsigned long long), st));
  {
    ProfScope ps(P_REPLAY, st, (double)count);
    if (G == 4) GSLS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_admm_staged<4>, a, R, max_items));
    else if (G == 2) GSLS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_admm_staged<2>, a, R, max_items));
    else GSLS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_admm_staged<1>, a, R, max_items));
    GSLS_CUDA_CHECK(cudaGetLastError());
  }
  if (tracing) {
    unsigned long long h[256];
    GSLS_CUDA_CHECK(cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st));
    GSLS_CUDA_CHECK(cudaStreamSynchronize(st));
    fprintf(stderr, "staged R=%d cs=%d phases %llu (items | boundary) cycles:", R, cs, h[0]);
    unsigned long long prev = h[250];
    for (unsigned long long p = 0; p < h[0]; ++p) {
      fprintf(stderr, " %llu|%llu", h[2 * p + 1] - prev, h[2 * p + 2] - h[2 * p + 1]);
      prev = h[2 * p + 2];
    }
    fprintf(stderr, "\n");
  }
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
  if (rc == GSLS_ERR_LOWRANK) {  // indefinite P met by a factored combine: dense re-run
    if ((rc = build_cache(c, qp, nullptr, nullptr, B, st))) return rc;
    rc = check_errors(c, st, "lqr build");
  }
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

// ---- graph-captured ADMM loop ---------------------------------------------------
// Under stream capture (one MPC step recorded as a CUDA graph) the host-driven wave
// loop below cannot run: it reads each wave's exit status back.  The captured form is a
// conditional WHILE node whose body is [count builds | cache build of the build list |
// replay of the live list | decide], all sized for the whole batch and guarded by the
// device-side counts (d_counts[0] live, [1] build); `decide` keeps the instances that
// committed a rho change, in index order, and re-arms the loop while any is left.
__global__ void k_loop_init(int* live, int* build, int* counts, int B, int prebuilt, int32_t* cache_builds) {
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    live[i] = i;
    build[i] = i;
    cache_builds[i] = prebuilt ? 1 : 0;
  }
  if (threadIdx.x == 0) {
    counts[0] = B;
    counts[1] = prebuilt ? 0 : B;
  }
}

__global__ void k_loop_count_builds(const int* build, const int* counts, int32_t* cache_builds) {
  for (int i = threadIdx.x; i < counts[1]; i += blockDim.x) cache_builds[build[i]] += 1;
}

__global__ void k_loop_decide(const int32_t* status, int* live, int* build, int* counts,
                              cudaGraphConditionalHandle h) {
  if (threadIdx.x != 0) return;
  int cnt = 0;
  const int nl = counts[0];
  for (int i = 0; i < nl; ++i) {
    const int inst = live[i];
    if (status[inst] == ST_REBUILD) build[cnt++] = inst;
  }
  for (int i = 0; i < cnt; ++i) live[i] = build[i];
  counts[0] = cnt;
  counts[1] = cnt;
  cudaGraphSetConditional(h, cnt > 0 ? 1u : 0u);
}

static int admm_solve_captured(Ctx* c, const gsls_qp_t* qp, const gsls_admm_settings_t* s, gsls_admm_state_t* state,
                               gsls_admm_stats_t* stats, double* dx, double* du, cudaStream_t st) {
  const int B = c->dims.batch;
  if (c->d_scratch) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "graph capture needs the shared-memory replay (N too large)");
    return GSLS_ERR_ARG;
  }
  GSLS_CUDA_CHECK(cudaMemsetAsync(stats->iterations, 0, sizeof(int32_t) * B, st));
  GSLS_CUDA_CHECK(cudaMemsetAsync(stats->converged, 0, sizeof(int32_t) * B, st));
  GSLS_CUDA_CHECK(cudaMemsetAsync(stats->rho_changes, 0, sizeof(int32_t) * B, st));
  const bool prebuilt = c->admm_prebuilt;
  c->admm_prebuilt = false;
  c->cache_valid = false;
  k_loop_init<<<1, 256, 0, st>>>(c->d_inst_list, c->d_build_list, c->d_counts, B, prebuilt ? 1 : 0,
                                 stats->cache_builds);
  GSLS_CUDA_CHECK(cudaGetLastError());
  cudaStreamCaptureStatus cst;
  cudaGraph_t graph = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  GSLS_CUDA_CHECK(cudaStreamGetCaptureInfo(st, &cst, nullptr, &graph, &deps, &ndeps));
  cudaGraphConditionalHandle h;
  GSLS_CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  GSLS_CUDA_CHECK(cudaGraphAddNode(&node, graph, deps, ndeps, &cp));
  GSLS_CUDA_CHECK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaStream_t bs = c->body_stream;
  GSLS_CUDA_CHECK(cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  int rc = GSLS_OK;
  k_loop_count_builds<<<1, 256, 0, bs>>>(c->d_build_list, c->d_counts, stats->cache_builds);
  GSLS_CUDA_CHECK(cudaGetLastError());
  c->dev.build_count = c->d_counts + 1;
  rc = build_cache(c, qp, state->rho, c->d_build_list, B, bs);
  c->dev.build_count = nullptr;
  if (!rc) {
    ReplayArgs a{};
    a.qp = *qp;
    a.mode = MODE_ADMM;
    a.set = *s;
    a.state = *state;
    a.stats = *stats;
    a.status = c->d_status;
    a.dx = dx; a.du = du;
    a.list = c->d_inst_list;
    a.count = c->d_counts;
    a.cap = 0;
    rc = launch_admm_staged(c, a, B, bs);
    if (rc == GSLS_ERR_TOO_LARGE) rc = launch_replay(c, a, B, bs);
  }
  if (!rc) {
    k_loop_decide<<<1, 32, 0, bs>>>(c->d_status, c->d_inst_list, c->d_build_list, c->d_counts, h);
    if (cudaGetLastError() != cudaSuccess) rc = GSLS_ERR_CUDA;
  }
  cudaGraph_t done = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(bs, &done);
  if (rc) return rc;
  GSLS_CUDA_CHECK(ec);
  return GSLS_OK;
}

int admm_solve(Ctx* c, const gsls_qp_t* qp, const gsls_admm_settings_t* s, gsls_admm_state_t* state,
               gsls_admm_stats_t* stats, double* dx, double* du, cudaStream_t st) {
  const int B = c->dims.batch;
  if (s->sigma < 2 || s->max_iter < 1 || !(s->rho0 > 0) || !(s->tol_primal > 0) || !(s->tol_dual > 0)) {
    set_error(GSLS_ERR_ARG, -1, 0, 0, 0, "invalid ADMM settings");
    return GSLS_ERR_ARG;
  }
  {
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    GSLS_CUDA_CHECK(cudaStreamIsCapturing(st, &cst));
    if (cst == cudaStreamCaptureStatusActive) return admm_solve_captured(c, qp, s, state, stats, dx, du, st);
  }
  GSLS_CUDA_CHECK(cudaMemsetAsync(stats->iterations, 0, sizeof(int32_t) * B, st));
  GSLS_CUDA_CHECK(cudaMemsetAsync(stats->converged, 0, sizeof(int32_t) * B, st));
  GSLS_CUDA_CHECK(cudaMemsetAsync(stats->rho_changes, 0, sizeof(int32_t) * B, st));
  std::vector<int> builds(B, 0), list(B), status(B), rebuild;
  for (int i = 0; i < B; ++i) list[i] = i;
  rebuild = list;
  c->cache_valid = false;  // the ADMM rebuilds the cache at augmented costs
  bool prebuilt = c->admm_prebuilt;  // first build already issued by admm_build (possibly on another stream)
  c->admm_prebuilt = false;
  // Large batches: every launch pauses the undecided instances at the next rho decision
  // point (iteration sigma, 2 sigma, ...), so the instances that commit a rho change there
  // are rebuilt as one batched wave instead of waiting behind instances that iterate on
  // without one (up to max_iter); paused instances resume, bitwise identically, in the next
  // launch together with the rebuilt ones.  Once few instances remain (<= 2 per SM) the
  // last launches run uncapped.
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const char* capenv = getenv("GSLS_ADMM_FIRST_CAP");
  int cap = (B > sms) ? s->sigma : 0;
  if (capenv) cap = atoi(capenv);
  const bool verbose = getenv("GSLS_ADMM_VERBOSE") != nullptr;  // per-wave timing (diagnostics)
  // GSLS_ADMM_SERIAL=1: rebuild waves on the calling stream before the replay of every live
  // instance (no side-stream overlap), so per-family device times add up (bench phases)
  const char* serenv = getenv("GSLS_ADMM_SERIAL");
  const bool serial = serenv && serenv[0] == '1';
  // Lagged rebuilds (large waves only): the instances that committed a rho change are rebuilt
  // on the side stream during the next wave and rejoin one wave later, catching up by running
  // to the following decision point, instead of replaying behind their rebuild in the same
  // wave.  Every instance's iterates are the same either way (pauses resume bitwise).
  // GSLS_ADMM_LAG_MIN: smallest wave (instances) that lags, default 2 per SM (where a
  // wave's replay outlasts a lagged instance's catch-up); 0 disables.  B = 1024: bulk waves
  // 56.8 -> 53.1 ms, step 240.7 -> 237.4 ms, the tail unchanged (50 waves either way).
  const char* lagenv = getenv("GSLS_ADMM_LAG_MIN");
  const int lag_min = lagenv ? atoi(lagenv) : 2 * sms;
  std::vector<char> lagged(B, 0);  // built during the last wave, not yet replayed
  cudaEvent_t ev[3] = {};
  if (verbose) for (auto& e : ev) cudaEventCreate(&e);
  int wave = 0;
  auto replay_wave = [&](const std::vector<int>& ids, int* dlist, cudaStream_t sx) -> int {
    if (ids.empty()) return GSLS_OK;
    GSLS_CUDA_CHECK(cudaMemcpyAsync(dlist, ids.data(), sizeof(int) * ids.size(), cudaMemcpyHostToDevice, sx));
    ReplayArgs a{};
    a.qp = *qp;
    a.mode = MODE_ADMM;
    a.set = *s;
    a.state = *state;
    a.stats = *stats;
    a.status = c->d_status;
    a.dx = dx; a.du = du;
    a.list = dlist;
    a.cap = cap;
    const char* sg = getenv("GSLS_REPLAY_STAGED");
    int rc = (sg && sg[0] == '0') ? GSLS_ERR_TOO_LARGE : launch_admm_staged(c, a, (int)ids.size(), sx);
    if (rc == GSLS_ERR_TOO_LARGE) rc = launch_replay(c, a, (int)ids.size(), sx);
    return rc;
  };
  while (!list.empty()) {
    const int cnt = (int)list.size(), nreb = (int)rebuild.size();
    if (verbose) cudaEventRecord(ev[0], st);
    int rc = GSLS_OK;
    if (prebuilt) {  // the first build already ran (admm_build): one launch over every instance
      for (int i : rebuild) builds[i]++;
      prebuilt = false;
      rc = replay_wave(list, c->d_inst_list, st);
    } else if (nreb == cnt || serial) {  // every live instance needs its (first or re-) build
      GSLS_CUDA_CHECK(cudaMemcpyAsync(c->d_build_list, rebuild.data(), sizeof(int) * nreb, cudaMemcpyHostToDevice, st));
      if ((rc = build_cache(c, qp, state->rho, c->d_build_list, nreb, st))) return rc;
      for (int i : rebuild) builds[i]++;
      rc = replay_wave(list, c->d_inst_list, st);
    } else {
      // instances that committed a rho change are rebuilt and replayed on the side stream
      // while the others continue on the main stream (disjoint instances and cache slices)
      std::vector<int> cont;
      const bool lag = lag_min > 0 && cnt >= lag_min;
      if (lag)  // last wave's lagged instances first: their CTAs start first and have the longest run
        for (int i : list)
          if (lagged[i]) cont.push_back(i);
      for (int i : list)
        if (!(lag && lagged[i]) && std::find(rebuild.begin(), rebuild.end(), i) == rebuild.end()) cont.push_back(i);
      std::fill(lagged.begin(), lagged.end(), 0);
      if (nreb > 0) {
        if (!c->side) {
          // highest priority: the rebuild chain's CTAs (and the rebuilt instances' replay)
          // take SM slots as the main stream's replay CTAs retire, instead of queueing
          // behind the whole wave (GSLS_SIDE_PRIORITY=0: default priority)
          int lo = 0, hi = 0;
          GSLS_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
          const char* pe = getenv("GSLS_SIDE_PRIORITY");
          GSLS_CUDA_CHECK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, (pe && pe[0] == '0') ? lo : hi));
          GSLS_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
          GSLS_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        }
        GSLS_CUDA_CHECK(cudaEventRecord(c->ev_fork, st));
        GSLS_CUDA_CHECK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
        GSLS_CUDA_CHECK(cudaMemcpyAsync(c->d_build_list, rebuild.data(), sizeof(int) * nreb, cudaMemcpyHostToDevice,
                                        c->side));
        if ((rc = build_cache(c, qp, state->rho, c->d_build_list, nreb, c->side))) return rc;
        for (int i : rebuild) builds[i]++;
        if (lag)
          for (int i : rebuild) lagged[i] = 1;
        else if ((rc = replay_wave(rebuild, c->d_build_list, c->side)))
          return rc;
        GSLS_CUDA_CHECK(cudaEventRecord(c->ev_join, c->side));
      }
      rc = replay_wave(cont, c->d_inst_list, st);
      if (nreb > 0) GSLS_CUDA_CHECK(cudaStreamWaitEvent(st, c->ev_join, 0));
    }
    if (rc) return rc;
    if (verbose) cudaEventRecord(ev[1], st);
    rc = check_errors(c, st, "admm");  // synchronizes
    // GSLS_ERR_LOWRANK: a factored combine met an indefinite P; the tree is now dense and
    // the instances whose build failed (ST_BUILD_ERR, state untouched) are rebuilt
    if (rc && rc != GSLS_ERR_LOWRANK) return rc;
    GSLS_CUDA_CHECK(cudaMemcpyAsync(status.data(), c->d_status, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
    GSLS_CUDA_CHECK(cudaStreamSynchronize(st));
    if (verbose) {
      float tw = 0.f;
      cudaEventElapsedTime(&tw, ev[0], ev[1]);
      fprintf(stderr, "admm wave %d: %d instances (%d rebuilt, cap %d): %.3f ms\n", wave, cnt, nreb, cap, tw);
    }
    ++wave;
    std::vector<int> next, nrb;
    for (int i : list) {
      if (lagged[i]) next.push_back(i);  // rebuilt this wave, replays in the next
      else if (status[i] == ST_REBUILD) { next.push_back(i); nrb.push_back(i); }
      else if (status[i] == ST_CONTINUE) next.push_back(i);
      else if (status[i] == ST_BUILD_ERR) { next.push_back(i); nrb.push_back(i); builds[i]--; }
    }
    list.swap(next);
    rebuild.swap(nrb);
    cap = (cap > 0 && !capenv) ? cap + s->sigma : 0;
  }
  GSLS_CUDA_CHECK(cudaMemcpyAsync(stats->cache_builds, builds.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice, st));
  GSLS_CUDA_CHECK(cudaStreamSynchronize(st));
  if (verbose) for (auto& e : ev) cudaEventDestroy(e);
  return GSLS_OK;
}

// The ADMM's first cache build (all instances, at state rho) ahead of the solve, so a
// caller can overlap it with independent work on another stream (the robust RTI step
// builds it while the SLS synthesis runs: the factorization does not depend on the
// tightened offsets f).  The next admm_solve on this context skips that build; the
// caller orders the two streams.
int admm_build(Ctx* c, const gsls_qp_t* qp, const double* rho, cudaStream_t st) {
  int rc = build_cache(c, qp, rho, nullptr, c->dims.batch, st);
  if (rc) return rc;
  c->admm_prebuilt = true;
  return GSLS_OK;
}

}  // namespace gsls
