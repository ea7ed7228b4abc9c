// Shared types and helpers for the GPU-SLS kernels (sm_100a).
//
// Internal storage convention: every n x n matrix kept on the device by the
// solver (scan slot values, recorded aux, SLS grids) is row-major with a
// padded leading dimension LDG = round_up(n, 4) and zero padding columns, so
// rows can be moved with 16-byte vector accesses.  User-facing QP buffers are
// dense row-major without padding (the reference layouts, lqr.py:53-68).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/gsls.h"

namespace gsls {

constexpr int kMaxN = 80;        // largest state dimension supported (75D humanoid + slack)
constexpr int kMaxM = 24;        // largest input dimension (north star: n_u <= 23)

__host__ __device__ inline int round_up(int a, int b) { return (a + b - 1) / b * b; }
__host__ __device__ inline int ldg_of(int n) { return round_up(n, 4); }
// smem leading dimension: multiple of 4 (float4 rows) and == 4 mod 8 so rows
// i and i+4 of a column fall in different banks.
__host__ __device__ inline int lds_of(int n) {
  int l = round_up(n, 4);
  return (l % 8 == 4) ? l : l + 4;
}
__host__ __device__ inline size_t mat_elems(int n) { return (size_t)n * ldg_of(n); }

// Division by a runtime constant d >= 1 for 0 <= x < 2^31: q = umulhi(x, mul) >> sh with the
// round-up multiplier mul = ceil(2^(31 + ceil(log2 d)) / d) (Granlund-Montgomery).  The small
// per-cell kernels index their (row, column) loops with it instead of a ~20-instruction
// integer division per iteration.
struct FastDiv {
  int d;
  unsigned mul, sh;
  __host__ __device__ void init(int dv) {
    d = dv;
    if (dv <= 1) { mul = 0; sh = 0; return; }
    unsigned l = 0;
    while ((1u << l) < (unsigned)dv) ++l;
    const unsigned p = 31 + l;
    mul = (unsigned)(((1ull << p) + (unsigned)dv - 1) / (unsigned)dv);
    sh = p - 32;
  }
#ifdef __CUDACC__
  __device__ __forceinline__ int div(int x) const { return d <= 1 ? x : (int)(__umulhi((unsigned)x, mul) >> sh); }
#endif
};

// Per-instance error record.  Kernels run stages / cells / ops in parallel, but
// the reference raises the FIRST failure of its sequential loops: spd_inverse
// names the lowest stage (lqr.py:204-215), _locate_singular the first valid
// (k, j) in row-major order (sls.py:321-326), linearize the first stage, its
// dynamics before its constraints (sqp.py:122-131), and the phases run in
// order (leaves, then the scan, then the gains; lqr.py:379-402).  So every
// raise is packed into one 64-bit key ordered as (phase, where, aux, label),
// and the record keeps the minimum (atomicMax on the complement; 0 = none).
struct ErrSlot {
  unsigned long long key;
};

struct ErrInfo {
  int code, where, aux, label;
};

__host__ __device__ inline int err_phase(int code, int label) {
  if (code == GSLS_ERR_ILL_CONDITIONED || code == GSLS_ERR_LOWRANK) return 2;  // the combine tree
  if (label == GSLS_LABEL_R_BPB || label == GSLS_LABEL_QU_BPB) return 3;      // gains after the scan
  return 1;                                                                    // leaves / linearize
}

__host__ __device__ inline unsigned long long err_pack(int code, int where, int aux, int label) {
  const unsigned long long p = (unsigned long long)(err_phase(code, label) & 0xF) << 60 |
                               (unsigned long long)((unsigned)where & 0xFFFFFFu) << 36 |
                               (unsigned long long)((unsigned)(aux + 1) & 0xFFFFFu) << 16 |
                               (unsigned long long)(code & 0xFF) << 8 | (unsigned long long)(label & 0xFF);
  return ~p;
}

__host__ __device__ inline ErrInfo err_unpack(unsigned long long key) {
  const unsigned long long p = ~key;
  ErrInfo e;
  e.code = (int)((p >> 8) & 0xFF);
  e.label = (int)(p & 0xFF);
  e.where = (int)((p >> 36) & 0xFFFFFFu);
  e.aux = (int)((p >> 16) & 0xFFFFFu) - 1;
  return e;
}

__device__ inline void raise_err(ErrSlot* e, int code, int where, int aux = -1, int label = 0) {
  if (e == nullptr) return;
  atomicMax(&e->key, err_pack(code, where, aux, label));
}

__device__ inline float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ inline float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide max of non-negative values; `red` needs blockDim/32 floats.
__device__ inline float block_max(float v, float* red) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = 0.f;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) r = fmaxf(r, red[i]);
  __syncthreads();
  return r;
}

}  // namespace gsls

#define GSLS_CUDA_CHECK(expr)                                   \
  do {                                                          \
    cudaError_t _e = (expr);                                    \
    if (_e != cudaSuccess) {                                    \
      gsls::set_last_error(cudaGetErrorString(_e), __FILE__, __LINE__); \
      return GSLS_ERR_CUDA;                                     \
    }                                                           \
  } while (0)

namespace gsls {
void set_last_error(const char* msg, const char* file, int line);
}
