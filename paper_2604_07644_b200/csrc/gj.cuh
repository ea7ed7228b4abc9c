// Gauss-Jordan inverse with register-resident row segments (the CVF combine's
// (I + Pr Cl)^-1, replacing the reference's solve(M1^T, .) / solve(M2^T, .)
// pair, lqr.py:233-235).
#pragma once

#include "common.cuh"

namespace gsls {

__device__ inline void bar_named(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Scratch words: double-buffered per-warp candidate rows + keys, the displaced
// row, the permutation and flags.
constexpr int gj_scratch_words(int NP) { return 2 * (NP / 8) * NP + 2 * NP + 4 * (NP / 8) + 2 * NP + 8; }

// In-place Gauss-Jordan with partial pivoting, one CTA barrier per pivot step.
// 4 threads per row, each holding NP/4 consecutive columns of its row in
// registers; threads [0, 4*NP) take part and synchronize with named barrier 1.
//
// Step k: the column-k owners of rows >= k form keys (bits(|a_ik|) + 1, which
// order like |a_ik|); each warp finds its max with one redux.sync and the
// first lane holding it with a ballot (first index on ties, as LAPACK
// i*amax).  The warp's candidate row is published in a per-warp slot together
// with its key, and row k publishes itself (the row the pivot displaces).
// After the single barrier every thread picks the winning warp (largest key,
// lowest warp on ties = lowest row) and reads the pivot row from that slot.
// Slots are double-buffered by step parity, so the next step's writes never
// race the previous step's reads.
//
// Reads a (smem, row-major, lds); writes the inverse row-major to inv and
// transposed to invT (either may be null or alias a: a is only read before
// the first barrier).  Returns (block-uniform) false when a pivot is zero /
// non-finite / below rel_tol * max|a| (the ill-conditioned-combine rule,
// lqr.py:229-232).  Must be called by the whole CTA (blockDim.x >= 4*NP).
template <int NP>
__device__ bool gj_inverse_rows(const float* a, float* inv, float* invT, int lds, int n, float* scratch,
                                float rel_tol) {
  constexpr int SEG = NP / 4;
  constexpr int NT = NP * 4;
  constexpr int NW = NT / 32;
  static_assert(SEG % 4 == 0, "segments are moved as float4");
  float* cand = scratch;                                        // [2][NW][NP]
  float* krow = cand + 2 * NW * NP;                             // [2][NP]
  unsigned* wkey = reinterpret_cast<unsigned*>(krow + 2 * NP);  // [2][NW]
  int* wrow = reinterpret_cast<int*>(wkey + 2 * NW);            // [2][NW]
  int* perm = wrow + 2 * NW;                                    // NP
  int* pos = perm + NP;                                         // NP
  float* misc = reinterpret_cast<float*>(pos + NP);             // [0] max|a|, [1] fail flag
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
  if (part && lane == 0) cand[warp] = mx;  // partial maxima (cand is free until the loop)
  __syncthreads();
  if (tid == 0) {
    float m2 = 0.f;
    for (int w = 0; w < NW; ++w) m2 = fmaxf(m2, cand[w]);
    misc[0] = m2;
    misc[1] = 0.f;
  }
  __syncthreads();
  if (part) {
    const float thresh = rel_tol * misc[0];
    bool fail = false;
    // k = qk*SEG + ck with ck unrolled, so r[ck] is a static register and the
    // buffer parity (k & 1 == ck & 1) is static too.
    for (int qk = 0; qk < 4; ++qk) {
#pragma unroll
      for (int ck = 0; ck < SEG; ++ck) {
        const int k = qk * SEG + ck;
        if (k < n) {
          const int b = ck & 1;
          const bool own = (q == qk);
          const float mine = r[ck];  // my row's element in column k when own
          const unsigned key = (own && row >= k && row < n) ? __float_as_uint(fabsf(mine)) + 1u : 0u;
          const unsigned wmax = __reduce_max_sync(0xffffffffu, key);
          const unsigned hits = __ballot_sync(0xffffffffu, key == wmax);
          const int wl = __ffs(hits) - 1;  // owner lane of the warp's candidate row
          // f = a[row][k] before this step, from the column-k owner of my row
          const float fk = __shfl_sync(0xffffffffu, mine, (lane & ~3) | qk);
          float* cb = cand + (b * NW + warp) * NP;
          if ((lane >> 2) == (wl >> 2)) {
#pragma unroll
            for (int c = 0; c < SEG; c += 4)
              *reinterpret_cast<float4*>(cb + q * SEG + c) = make_float4(r[c], r[c + 1], r[c + 2], r[c + 3]);
            if (q == 0) {
              wkey[b * NW + warp] = wmax;
              wrow[b * NW + warp] = row;
            }
          }
          if (row == k) {
#pragma unroll
            for (int c = 0; c < SEG; c += 4)
              *reinterpret_cast<float4*>(krow + b * NP + q * SEG + c) =
                  make_float4(r[c], r[c + 1], r[c + 2], r[c + 3]);
          }
          bar_named(1, NT);
          unsigned bk = 0;
          int bw = 0;
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const unsigned kw = wkey[b * NW + w];
            if (kw > bk) { bk = kw; bw = w; }
          }
          const int p = wrow[b * NW + bw];
          const float* prow = cand + (b * NW + bw) * NP;
          const float piv = prow[k];
          const float ip = __frcp_rn(piv);
          if (tid == 0) {
            perm[k] = p;
            if (!(fabsf(piv) > thresh) || !isfinite(piv)) fail = true;
          }
          float pr[SEG];
#pragma unroll
          for (int c = 0; c < SEG; c += 4) {
            const float4 t = *reinterpret_cast<const float4*>(prow + q * SEG + c);
            pr[c] = t.x; pr[c + 1] = t.y; pr[c + 2] = t.z; pr[c + 3] = t.w;
          }
          if (row == k) {
#pragma unroll
            for (int c = 0; c < SEG; ++c) r[c] = pr[c] * ip;
            if (own) r[ck] = ip;
          } else {
            float f = fk;
            if (row == p) {  // the displaced row k lands here
#pragma unroll
              for (int c = 0; c < SEG; c += 4) {
                const float4 t = *reinterpret_cast<const float4*>(krow + b * NP + q * SEG + c);
                r[c] = t.x; r[c + 1] = t.y; r[c + 2] = t.z; r[c + 3] = t.w;
              }
              f = krow[b * NP + k];
            }
            const float fi = f * ip;
#pragma unroll
            for (int c = 0; c < SEG; ++c) r[c] = fmaf(-fi, pr[c], r[c]);
            if (own) r[ck] = -fi;
          }
        }
      }
    }
    if (fail && tid == 0) misc[1] = 1.f;
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
