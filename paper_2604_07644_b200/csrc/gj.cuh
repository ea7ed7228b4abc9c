// Gauss-Jordan inverse with register-resident row segments (the CVF combine's
// (I + Pr Cl)^-1, replacing the reference's solve(M1^T, .) / solve(M2^T, .)
// pair, lqr.py:233-235).
#pragma once

#include "common.cuh"

namespace gsls {

__device__ inline void bar_named(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

constexpr int gj_scratch_words(int NP) { return 4 * NP + 48; }

// In-place Gauss-Jordan with partial pivoting.  4 threads per row, each holding
// NP/4 consecutive columns of its row in registers; threads [0, 4*NP) take part
// and synchronize with named barrier 1.  Per pivot step: warp argmax of |a_ik|
// over the column-k owners (first index on ties, as LAPACK i*amax), one smem
// exchange of the pivot row and the displaced row, 2 barriers, NP/4 FMAs per
// thread.  Reads a (smem, row-major, lds); writes the inverse row-major to inv
// and transposed to invT (either may be null or alias a: a is only read before
// the first barrier).
// Returns (block-uniform) false when a pivot is zero / non-finite / below
// rel_tol * max|a| (the ill-conditioned-combine rule, lqr.py:229-232).
// Must be called by the whole CTA (blockDim.x >= 4*NP).
template <int NP>
__device__ bool gj_inverse_rows(const float* a, float* inv, float* invT, int lds, int n, float* scratch,
                                float rel_tol) {
  constexpr int SEG = NP / 4;
  constexpr int NT = NP * 4;
  constexpr int NW = NT / 32;
  static_assert(SEG % 4 == 0, "segments are moved as float4");
  float* prow = scratch;                           // NP
  float* krow = prow + NP;                         // NP
  int* perm = reinterpret_cast<int*>(krow + NP);   // NP
  int* pos = perm + NP;                            // NP
  float* wv = reinterpret_cast<float*>(pos + NP);  // 16
  int* wi = reinterpret_cast<int*>(wv + 16);       // 16
  float* misc = reinterpret_cast<float*>(wi + 16);  // [0] max|a|, [1] fail flag
  const int tid = threadIdx.x;
  const bool part = tid < NT;
  const int row = tid >> 2, q = tid & 3, lane = tid & 31, warp = tid >> 5;
  float r[SEG];
  float mx = 0.f;
#pragma unroll
  for (int c = 0; c < SEG; ++c) {
    const int col = q * SEG + c;
    r[c] = (part && row < n && col < n) ? a[row * lds + col] : 0.f;
    mx = fmaxf(mx, fabsf(r[c]));
  }
  mx = warp_max(mx);
  if (part && lane == 0) wv[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    float m2 = 0.f;
    for (int w = 0; w < NW; ++w) m2 = fmaxf(m2, wv[w]);
    misc[0] = m2;
    misc[1] = 0.f;
  }
  __syncthreads();
  if (part) {
    const float thresh = rel_tol * misc[0];
    for (int k = 0; k < n; ++k) {
      const int qk = k / SEG, ck = k - qk * SEG;
      float mine = 0.f;  // my row's element in column k (valid in the owner lane)
#pragma unroll
      for (int c = 0; c < SEG; ++c)
        if (c == ck) mine = r[c];
      float v = (q == qk && row >= k && row < n) ? fabsf(mine) : -1.f;
      int vi = row;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, vi, o);
        if (ov > v || (ov == v && oi < vi)) { v = ov; vi = oi; }
      }
      if (lane == 0) { wv[warp] = v; wi[warp] = vi; }
      // f = a[row][k] before this step, broadcast from the column-k owner of my row
      const float fk = __shfl_sync(0xffffffffu, mine, (lane & ~3) | qk);
      bar_named(1, NT);
      float bv = -1.f;
      int p = n;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const float ov = wv[w];
        const int oi = wi[w];
        if (ov > bv || (ov == bv && oi < p)) { bv = ov; p = oi; }
      }
      if (row == p) {
#pragma unroll
        for (int c = 0; c < SEG; c += 4)
          *reinterpret_cast<float4*>(prow + q * SEG + c) = make_float4(r[c], r[c + 1], r[c + 2], r[c + 3]);
      }
      if (row == k) {
#pragma unroll
        for (int c = 0; c < SEG; c += 4)
          *reinterpret_cast<float4*>(krow + q * SEG + c) = make_float4(r[c], r[c + 1], r[c + 2], r[c + 3]);
      }
      if (tid == 0) perm[k] = p;
      bar_named(1, NT);
      const float piv = prow[k];
      if (tid == 0 && (!(fabsf(piv) > thresh) || !isfinite(piv))) misc[1] = 1.f;
      const float ip = 1.f / piv;
      float pr[SEG];
#pragma unroll
      for (int c = 0; c < SEG; c += 4) {
        const float4 t = *reinterpret_cast<const float4*>(prow + q * SEG + c);
        pr[c] = t.x; pr[c + 1] = t.y; pr[c + 2] = t.z; pr[c + 3] = t.w;
      }
      if (row == k) {
#pragma unroll
        for (int c = 0; c < SEG; ++c) r[c] = (q * SEG + c == k) ? ip : pr[c] * ip;
      } else {
        float f = fk;
        if (row == p) {  // the displaced row k lands here
#pragma unroll
          for (int c = 0; c < SEG; c += 4) {
            const float4 t = *reinterpret_cast<const float4*>(krow + q * SEG + c);
            r[c] = t.x; r[c + 1] = t.y; r[c + 2] = t.z; r[c + 3] = t.w;
          }
          f = krow[k];
        }
        const float fi = f * ip;
#pragma unroll
        for (int c = 0; c < SEG; ++c) r[c] = (q * SEG + c == k) ? -fi : fmaf(-fi, pr[c], r[c]);
      }
    }
  }
  __syncthreads();
  if (tid == 0) {  // undo the row interchanges as a column permutation, last to first
    for (int j = 0; j < n; ++j) pos[j] = j;  // pos = src map
    for (int k = n - 1; k >= 0; --k) {
      const int pk = perm[k], t = pos[k];
      pos[k] = pos[pk];
      pos[pk] = t;
    }
    for (int j = 0; j < n; ++j) perm[pos[j]] = j;  // perm = destination column of source column
  }
  __syncthreads();
  const bool ok = misc[1] == 0.f;
  if (part && row < n) {
#pragma unroll
    for (int c = 0; c < SEG; ++c) {
      const int col = q * SEG + c;
      if (col < n) {
        const int d = perm[col];
        if (inv) inv[row * lds + d] = r[c];
        if (invT) invT[d * lds + row] = r[c];
      }
    }
  }
  __syncthreads();
  return ok;
}

}  // namespace gsls
