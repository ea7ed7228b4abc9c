// CTA-level dense kernels for n <= 80 matrices held in shared memory.
//
// * gemm_tn      C = At^T * B with At stored k-major (At[k][i]) and B row-major,
//                4x4 register tiles, both operands read as float4 (the left
//                operand is broadcast across a warp, the right one contiguous).
// * gj_inverse   in-place Gauss-Jordan inverse with partial pivoting (argmax
//                |a_ik|, first index on ties, as LAPACK i*amax) — replaces the
//                reference's solve(M1^T, .) / solve(M2^T, .) pair, lqr.py:233-235.
// * warp_spd_inverse  Cholesky + explicit inverse with the reference pivot /
//                ridge rule (lqr.py:185-220) for m <= 24 blocks, one warp.
#pragma once

#include "common.cuh"

namespace gsls {

// ---- loads / stores between global (ld = ldg) and shared (ld = lds) ----------

// dst[i][j] = src[i][j] for i < rows, j < cols; zero for cols <= j < ldg(cols)
__device__ inline void cta_load(float* dst, int lds, const float* __restrict__ src, int lsrc, int rows,
                                int cols) {
  const int cp = ldg_of(cols);
  for (int e = threadIdx.x; e < rows * cp; e += blockDim.x) {
    const int i = e / cp, j = e - i * cp;
    dst[i * lds + j] = (j < cols) ? src[(size_t)i * lsrc + j] : 0.f;
  }
}

// dst[j][i] = src[i][j] (square n x n); padding columns of dst zeroed.
__device__ inline void cta_load_t(float* dst, int lds, const float* __restrict__ src, int lsrc, int n) {
  const int np = ldg_of(n);
  for (int e = threadIdx.x; e < n * np; e += blockDim.x) {
    const int i = e / np, j = e - i * np;  // i: src row, j: src col (coalesced read)
    if (j < n) dst[j * lds + i] = src[(size_t)i * lsrc + j];
    else dst[i * lds + j] = 0.f;  // row i, padding column j of dst
  }
}

// smem -> smem transpose of the n x n block; padding columns of dst zeroed.
__device__ inline void cta_transpose(float* dst, const float* src, int lds, int n) {
  const int np = ldg_of(n);
  for (int e = threadIdx.x; e < n * np; e += blockDim.x) {
    const int i = e / np, j = e - i * np;
    dst[i * lds + j] = (j < n) ? src[j * lds + i] : 0.f;
  }
}

// smem (lds) -> global (ldg) copy of an n x ldg(n) block, float4 rows.
// Walks the (row, float4 column) chunks e = threadIdx.x, + blockDim.x, ... of an n x 4q
// block with two integer divisions in total (the combine kernels' index math was a
// visible share of their issue slots): f(i, j) with j the first float of the chunk.
template <class F>
__device__ __forceinline__ void cta_chunks(int n, int q, F f) {
  const int nt = blockDim.x;
  int i = threadIdx.x / q, j4 = threadIdx.x - i * q;
  const int di = nt / q, dj = nt - di * q;
  while (i < n) {
    f(i, j4 << 2);
    i += di;
    j4 += dj;
    if (j4 >= q) { j4 -= q; ++i; }
  }
}

__device__ inline void cta_store(float* __restrict__ dst, const float* src, int lds, int n) {
  const int q = ldg_of(n) / 4;
  const int ld = q << 2;
  cta_chunks(n, q, [&](int i, int j) {
    *reinterpret_cast<float4*>(dst + (size_t)i * ld + j) = *reinterpret_cast<const float4*>(src + i * lds + j);
  });
}

// ---- async copies -------------------------------------------------------------

__device__ inline void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ inline void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ inline void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
template <int N>
__device__ inline void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Issues 16-byte cp.async copies of an n x ldg(n) padded global matrix into smem
// (ld = lds); the caller commits / waits.  Padding columns arrive as stored (zero).
__device__ inline void cta_load_async(float* dst, int lds, const float* __restrict__ src, int n) {
  const int q = ldg_of(n) >> 2;
  cta_chunks(n, q, [&](int i, int j) { cp_async16(dst + i * lds + j, src + (size_t)i * (q << 2) + j); });
}

// ---- GEMM ---------------------------------------------------------------------

// C[i][j] = sum_{k<n} At[k][i] * B[k][j] over the padded np x np output, 4x4
// register tile per thread; the epilogue receives whole tiles: epi(i0, j0, acc)
// and must ignore rows i >= n.
template <class Epi>
__device__ inline void gemm_tn(int n, const float* At, const float* B, int lds, Epi epi) {
  const int T = ldg_of(n) >> 2;
  const int tiles = T * T;
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
    const int ti = t / T, tj = t - ti * T;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    const float* pa = At + 4 * ti;
    const float* pb = B + 4 * tj;
#pragma unroll 4
    for (int k = 0; k < n; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(pa + k * lds);
      const float4 b = *reinterpret_cast<const float4*>(pb + k * lds);
      const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        acc[r][0] = fmaf(av[r], b.x, acc[r][0]);
        acc[r][1] = fmaf(av[r], b.y, acc[r][1]);
        acc[r][2] = fmaf(av[r], b.z, acc[r][2]);
        acc[r][3] = fmaf(av[r], b.w, acc[r][3]);
      }
    }
    epi(4 * ti, 4 * tj, acc);
  }
}

// The same product on 8 x 4 register tiles (two 4 x 4 epilogue calls, the lower one only
// inside the padded np rows): one B row load feeds eight rows, halving gemm_tn's shared
// wavefronts per FMA (k_matprod is bound by them).  Every element keeps its fma chain.
template <class Epi>
__device__ inline void gemm_tn84(int n, const float* At, const float* B, int lds, Epi epi) {
  const int np = ldg_of(n), T = np >> 2, TR = (np + 7) >> 3;
  const int tiles = TR * T;
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
    const int ti = t / T, tj = t - ti * T;
    float acc[8][4];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    const float* pa = At + 8 * ti;
    const float* pb = B + 4 * tj;
#pragma unroll 2
    for (int k = 0; k < n; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(pa + k * lds);
      const float4 a1 = *reinterpret_cast<const float4*>(pa + k * lds + 4);
      const float4 b = *reinterpret_cast<const float4*>(pb + k * lds);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        acc[r][0] = fmaf(av[r], b.x, acc[r][0]);
        acc[r][1] = fmaf(av[r], b.y, acc[r][1]);
        acc[r][2] = fmaf(av[r], b.z, acc[r][2]);
        acc[r][3] = fmaf(av[r], b.w, acc[r][3]);
      }
    }
    epi(8 * ti, 4 * tj, *reinterpret_cast<float(*)[4][4]>(&acc[0][0]));
    if (8 * ti + 4 < np) epi(8 * ti + 4, 4 * tj, *reinterpret_cast<float(*)[4][4]>(&acc[4][0]));
  }
}

// epilogues
struct EpiSmem {  // C (smem) = acc (+ I)
  float* C;
  int lds, n;
  bool add_identity;
  __device__ void operator()(int i0, int j0, float (&acc)[4][4]) const {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + r;
      if (i >= n) break;
      float4 v = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
      if (add_identity && i >= j0 && i < j0 + 4) (&v.x)[i - j0] += 1.f;
      *reinterpret_cast<float4*>(C + i * lds + j0) = v;
    }
  }
};

struct EpiGlobalNeg {  // G (global, ld) = -acc
  float* G;
  int ld, n;
  __device__ void operator()(int i0, int j0, float (&acc)[4][4]) const {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + r;
      if (i >= n) break;
      *reinterpret_cast<float4*>(G + (size_t)i * ld + j0) = make_float4(-acc[r][0], -acc[r][1], -acc[r][2], -acc[r][3]);
    }
  }
};

struct EpiGlobal {  // G (global, ld) = acc + add (global, may be null); optional transposed copy Gt
  float* G;
  const float* add;
  int ld, n;
  float* Gt;
  __device__ void operator()(int i0, int j0, float (&acc)[4][4]) const {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + r;
      if (i >= n) break;
      float4 v = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
      if (add) {
        const float4 a = *reinterpret_cast<const float4*>(add + (size_t)i * ld + j0);
        v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
      }
      *reinterpret_cast<float4*>(G + (size_t)i * ld + j0) = v;
    }
    if (Gt) {  // rows i >= n of the tile are zero (zero padding of the operands)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = j0 + c;
        if (j >= n) break;
        *reinterpret_cast<float4*>(Gt + (size_t)j * ld + i0) = make_float4(acc[0][c], acc[1][c], acc[2][c], acc[3][c]);
      }
    }
  }
};

// ---- Gauss-Jordan inverse -------------------------------------------------------

// Scratch: buf needs 3*ldg(n) floats + 2*n ints (after the floats).
// Returns (block-uniform) false when a pivot is zero / non-finite / below
// rel_tol * max|a| (the ill-conditioned-combine rule, lqr.py:229-232).
__device__ inline bool gj_inverse(float* a, float* out, int lds, int n, float* buf, float rel_tol) {
  const int np = ldg_of(n);
  float* rbuf = buf;
  float* fbuf = buf + np;
  float* misc = buf + 2 * np;           // misc[0]: max|a|, misc[1]: fail flag
  int* perm = reinterpret_cast<int*>(buf + 3 * np);
  int* src = perm + n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;

  // max |a| for the relative pivot threshold
  if (warp == 0) {
    float mx = 0.f;
    for (int e = lane; e < n * n; e += 32) mx = fmaxf(mx, fabsf(a[(e / n) * lds + e % n]));
    mx = warp_max(mx);
    if (lane == 0) { misc[0] = mx; misc[1] = 0.f; }
  }
  __syncthreads();
  const float thresh = rel_tol * misc[0];

  for (int k = 0; k < n; ++k) {
    if (warp == 0) {
      float best = -1.f;
      int bi = n;
      for (int i = k + lane; i < n; i += 32) {
        const float v = fabsf(a[i * lds + k]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      const int p = bi;
      if (p != k) {
        for (int j = lane; j < n; j += 32) {
          const float t = a[k * lds + j];
          a[k * lds + j] = a[p * lds + j];
          a[p * lds + j] = t;
        }
      }
      __syncwarp();
      const float piv = a[k * lds + k];
      if (lane == 0) {
        perm[k] = p;
        if (!(fabsf(piv) > thresh) || !isfinite(piv)) misc[1] = 1.f;
      }
      const float inv = 1.f / piv;
      for (int j = lane; j < n; j += 32) rbuf[j] = (j == k) ? inv : a[k * lds + j] * inv;
      for (int i = lane; i < n; i += 32) fbuf[i] = (i == k) ? 0.f : a[i * lds + k];
    }
    __syncthreads();
    for (int i = warp; i < n; i += nw) {
      const float f = fbuf[i];
      for (int j = lane; j < n; j += 32) {
        if (i == k) a[i * lds + j] = rbuf[j];
        else if (j == k) a[i * lds + j] = -f * rbuf[k];
        else a[i * lds + j] = fmaf(-f, rbuf[j], a[i * lds + j]);
      }
    }
    __syncthreads();
  }
  // undo the row interchanges as a column permutation (applied last-to-first)
  if (threadIdx.x == 0) {
    for (int j = 0; j < n; ++j) src[j] = j;
    for (int k = n - 1; k >= 0; --k) {
      const int p = perm[k];
      const int t = src[k];
      src[k] = src[p];
      src[p] = t;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * np; e += blockDim.x) {
    const int i = e / np, j = e - i * np;
    out[i * lds + j] = (j < n) ? a[i * lds + src[j]] : 0.f;
  }
  __syncthreads();
  return misc[1] == 0.f;
}

// ---- SPD inverse (one warp, m <= 24) ---------------------------------------------

// M (ld = ldm) is read; inv (ld = ldm) is written.  work: 2 * 24 * 25 elements.
// Returns 0 ok, 1 singular (after the ridge retry).  Pivot rule of lqr.py:185-220:
// Cholesky; min pivot^2 < 1e-10 or failure -> retry with ridge 1e-9 (no pivot
// test) -> failure is SingularStageError.
template <class T>
__device__ inline int warp_spd_inverse(const T* M, int ldm, T* inv, int m, T* work, int ld = kMaxM + 1,
                                       int xoff = kMaxM * (kMaxM + 1)) {
  // work: L (m x ld) at 0 and X = L^-1 (m x ld) at xoff; the defaults fit any m <= kMaxM
  // (callers that read L^-1 afterwards index it with them)
  const int lane = threadIdx.x & 31;
  T* L = work;
  T* X = work + xoff;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const T ridge = attempt ? T(1e-9) : T(0);
    for (int e = lane; e < m * m; e += 32) {
      const int i = e / m, j = e % m;
      L[i * ld + j] = M[i * ldm + j] + ((i == j) ? ridge : T(0));
    }
    __syncwarp();
    bool ok = true, small = false;
    T rd = T(0);  // lane j keeps 1 / L[j][j]: multiplies instead of divisions on the chain
    for (int j = 0; j < m; ++j) {
      const T d = L[j * ld + j];
      if (!(d > T(0)) || !isfinite((double)d)) { ok = false; break; }
      const T r = rsqrt(d);
      const T piv = d * r;
      if ((double)piv * (double)piv < 1e-10) small = true;
      __syncwarp();
      if (lane == j) {
        L[j * ld + j] = piv;
        rd = r;
      }
      if (lane > j && lane < m) L[lane * ld + j] *= r;
      __syncwarp();
      if (lane > j && lane < m) {  // row lane: independent updates, loads batched 4 deep
        const T lij = L[lane * ld + j];
        T* row = L + lane * ld;
        int l = j + 1;
        for (; l + 3 <= lane; l += 4) {
          const T c0 = L[l * ld + j], c1 = L[(l + 1) * ld + j], c2 = L[(l + 2) * ld + j], c3 = L[(l + 3) * ld + j];
          const T v0 = row[l], v1 = row[l + 1], v2 = row[l + 2], v3 = row[l + 3];
          row[l] = fma(-lij, c0, v0);
          row[l + 1] = fma(-lij, c1, v1);
          row[l + 2] = fma(-lij, c2, v2);
          row[l + 3] = fma(-lij, c3, v3);
        }
        for (; l <= lane; ++l) row[l] = fma(-lij, L[l * ld + j], row[l]);
      }
      __syncwarp();
    }
    if (!ok || (attempt == 0 && small)) {
      if (attempt == 1) return 1;
      continue;
    }
    {  // X = L^{-1}: lane j solves L x = e_j, right-looking with X's column j as the
       // accumulators (row i still receives -L[i][k] x_k for k = j .. i-1 in ascending order,
       // the same fma chain as the row-by-row solve, but the rows below k update in parallel)
      const int j = lane;
      if (j < m)
        for (int i = 0; i < m; ++i) X[i * ld + j] = (i == j) ? T(1) : T(0);
      for (int k = 0; k < m; ++k) {
        const T rk = __shfl_sync(0xffffffffu, rd, k);
        if (j < m && k >= j) {
          const T xk = X[k * ld + j] * rk;
          X[k * ld + j] = xk;
          int i = k + 1;
          for (; i + 3 < m; i += 4) {
            const T l0 = L[i * ld + k], l1 = L[(i + 1) * ld + k], l2 = L[(i + 2) * ld + k], l3 = L[(i + 3) * ld + k];
            const T a0 = X[i * ld + j], a1 = X[(i + 1) * ld + j], a2 = X[(i + 2) * ld + j], a3 = X[(i + 3) * ld + j];
            X[i * ld + j] = fma(-l0, xk, a0);
            X[(i + 1) * ld + j] = fma(-l1, xk, a1);
            X[(i + 2) * ld + j] = fma(-l2, xk, a2);
            X[(i + 3) * ld + j] = fma(-l3, xk, a3);
          }
          for (; i < m; ++i) X[i * ld + j] = fma(-L[i * ld + k], xk, X[i * ld + j]);
        }
      }
    }
    __syncwarp();
    for (int e = lane; e < m * m; e += 32) {  // inv = X^T X
      const int i = e / m, j = e % m;
      T s = T(0);
      for (int k = max(i, j); k < m; ++k) s = fma(X[k * ld + i], X[k * ld + j], s);
      inv[i * ldm + j] = s;
    }
    __syncwarp();
    return 0;
  }
  return 1;
}

}  // namespace gsls
