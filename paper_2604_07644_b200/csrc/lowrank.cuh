// Factored CVF combine: the matrix half of the CVF combine (Eq. 28,
// lqr.py:226-239) when the earlier operand's C is carried as a factor.
//
// Every CVF leaf has C = B R^-1 B' (rank m; lqr.py:318-320, sls.py:262-264) and
// a combine's C = Psi C_l A_r' + C_r has rank <= rank C_l + rank C_r, so for the
// first tree levels C_l = F F' with F only n x r (r = m, 2m, 4m, ...).  The
// scan plan (lqr.cu upload_plan) tracks each slot's representation; with
// S = I_r + F' P_r F = L L' (Sylvester: det M1 = det S), Fh = F L^-T and
// V = P_r Fh the combine needs no n x n inverse:
//
//     M1^-1 = I - V Fh'        M2^-1 = I - Fh V'       M1^-1 P_r = P_r - V V'
//     Ups' = A_l - Fh (V' A_l)     X' = (P_r - V V') A_l     P = A_l' X' + P_l
//     U' = Fh' A_r'     Psi' = A_r' - V U'     A = Psi A_l
//     -Y' = -Fh U'      C = U U' + C_r   (or the factor [U, F_r])
//
// exactly the dense kernel's outputs (same record layout: Ups', X', Psi', -Y'
// row-major) in exact arithmetic.  The n x n Gauss-Jordan pivot chain becomes
// an r x r Cholesky; r <= 48 at the benched shapes.
//
// The Cholesky runs as a blocked right-looking elimination over the stacked
// rows [S; F; W] (W = P_r F): eliminating S's columns turns the F rows into
// F L^-T and the W rows into W L^-T = V in place (panels of 4 columns, two
// barriers per panel).  Every pivot of S is >= 1 when P_r is positive
// semidefinite (S >= I); a pivot below 0.5 means P_r is indefinite and the
// CTA reports failure, so the caller re-runs the scan with dense combines
// (which also owns the ill-conditioned-combine rule, lqr.py:229-232).
#pragma once

#include "smallmat.cuh"

namespace gsls {

// ---- generalized GEMMs (4x4 register tiles, float4 smem operands) ----------------
//
// Small outputs (an n x r or r x r product has only a few dozen 4x4 tiles) split K
// over KS adjacent lanes so the whole CTA works; the KS partial tiles are summed
// with a fixed butterfly of warp shuffles (deterministic), and the part-0 lane
// runs the epilogue.

__device__ inline int gemm_ks(int tiles, int K) {
  int ks = 1;
  while (ks < 8 && tiles * ks * 2 <= (int)blockDim.x && K >= 8 * ks) ks <<= 1;
  return ks;
}

__device__ inline void ks_reduce(float (&acc)[4][4], int ks) {
  for (int o = 1; o < ks; o <<= 1) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] += __shfl_xor_sync(0xffffffffu, acc[a][b], o);
  }
}

// C[i][j] = sum_{k<K} At[k][i] B[k][j] for i < round_up(M,4), j < round_up(Nc,4).
template <class Epi>
__device__ inline void gemm_tn_mn(int M, int Nc, int K, const float* At, int lda, const float* B, int ldb,
                                  Epi epi) {
  const int TM = (M + 3) >> 2, TN = (Nc + 3) >> 2, tiles = TM * TN;
  const int ks = gemm_ks(tiles, K), kslog = __ffs(ks) - 1;  // ks: a power of two
  const int work = tiles * ks;
  for (int base = 0; base < work; base += blockDim.x) {
    const int t = base + threadIdx.x;
    const int tile = t >> kslog, part = t & (ks - 1);
    const bool valid = t < work;
    const int ti = valid ? tile / TN : 0, tj = valid ? tile - ti * TN : 0;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    const float* pa = At + 4 * ti;
    const float* pb = B + 4 * tj;
    const int kend = valid ? K : 0;
#pragma unroll 4
    for (int k = part; k < kend; k += ks) {
      const float4 a = *reinterpret_cast<const float4*>(pa + k * lda);
      const float4 b = *reinterpret_cast<const float4*>(pb + k * ldb);
      const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        acc[r][0] = fmaf(av[r], b.x, acc[r][0]);
        acc[r][1] = fmaf(av[r], b.y, acc[r][1]);
        acc[r][2] = fmaf(av[r], b.z, acc[r][2]);
        acc[r][3] = fmaf(av[r], b.w, acc[r][3]);
      }
    }
    if (ks > 1) ks_reduce(acc, ks);
    if (valid && part == 0) epi(4 * ti, 4 * tj, acc);
  }
}

// C[i][j] = sum_{k<K} A[i][k] B[k][j], A row-major; K a multiple of 4 (the
// operands' padding columns / rows in [K, round_up) are zero).
template <class Epi>
__device__ inline void gemm_nn_mn(int M, int Nc, int K, const float* A, int lda, const float* B, int ldb,
                                  Epi epi) {
  const int TM = (M + 3) >> 2, TN = (Nc + 3) >> 2, tiles = TM * TN;
  const int ks = gemm_ks(tiles, K), kslog = __ffs(ks) - 1;  // ks: a power of two
  const int work = tiles * ks;
  for (int base = 0; base < work; base += blockDim.x) {
    const int t = base + threadIdx.x;
    const int tile = t >> kslog, part = t & (ks - 1);
    const bool valid = t < work;
    const int ti = valid ? tile / TN : 0, tj = valid ? tile - ti * TN : 0;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    const float* pa = A + 4 * ti * lda;
    const float* pb = B + 4 * tj;
    const int kend = valid ? K : 0;
#pragma unroll 2
    for (int k = 4 * part; k < kend; k += 4 * ks) {
      float4 ar[4], bk[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) ar[r] = *reinterpret_cast<const float4*>(pa + r * lda + k);
#pragma unroll
      for (int q = 0; q < 4; ++q) bk[q] = *reinterpret_cast<const float4*>(pb + (k + q) * ldb);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float av[4] = {ar[r].x, ar[r].y, ar[r].z, ar[r].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[r][0] = fmaf(av[q], bk[q].x, acc[r][0]);
          acc[r][1] = fmaf(av[q], bk[q].y, acc[r][1]);
          acc[r][2] = fmaf(av[q], bk[q].z, acc[r][2]);
          acc[r][3] = fmaf(av[q], bk[q].w, acc[r][3]);
        }
      }
    }
    if (ks > 1) ks_reduce(acc, ks);
    if (valid && part == 0) epi(4 * ti, 4 * tj, acc);
  }
}

// ---- epilogues (rows >= rows are dropped) -------------------------------------

struct EpiS {  // D (smem) = acc
  float* D;
  int ld, rows;
  __device__ void operator()(int i0, int j0, float (&acc)[4][4]) const {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (i0 + r >= rows) break;
      *reinterpret_cast<float4*>(D + (i0 + r) * ld + j0) = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
    }
  }
};

struct EpiSId {  // D (smem) = acc + I
  float* D;
  int ld, rows;
  __device__ void operator()(int i0, int j0, float (&acc)[4][4]) const {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + r;
      if (i >= rows) break;
      float4 v = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
      if (i >= j0 && i < j0 + 4) (&v.x)[i - j0] += 1.f;
      *reinterpret_cast<float4*>(D + i * ld + j0) = v;
    }
  }
};

// D (smem) = Base (smem, may alias D) - acc; optional global copy G (ld gld), optional
// transposed global copy Gt.
struct EpiSub {
  float* D;
  const float* Base;
  int ld, rows;
  float* G;
  int gld;
  __device__ void operator()(int i0, int j0, float (&acc)[4][4]) const {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + r;
      if (i >= rows) break;
      const float4 b = *reinterpret_cast<const float4*>(Base + i * ld + j0);
      const float4 v = make_float4(b.x - acc[r][0], b.y - acc[r][1], b.z - acc[r][2], b.w - acc[r][3]);
      if (D) *reinterpret_cast<float4*>(D + i * ld + j0) = v;
      if (G) *reinterpret_cast<float4*>(G + (size_t)i * gld + j0) = v;
    }
  }
};

// G (global) = acc (+ add: global, may be null / may alias G); optional transposed copy Gt;
// optional smem copy D (ld dld).
struct EpiG {
  float* G;
  const float* add;
  int ld, rows;
  float* Gt;
  float* D;
  int dld;
  float scale;  // 1 or -1
  const float* sadd = nullptr;  // smem addend (ld dld), used instead of add when set
  __device__ void operator()(int i0, int j0, float (&acc)[4][4]) const {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + r;
      if (i >= rows) break;
      float4 v = make_float4(scale * acc[r][0], scale * acc[r][1], scale * acc[r][2], scale * acc[r][3]);
      if (sadd) {
        const float4 a = *reinterpret_cast<const float4*>(sadd + i * dld + j0);
        v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
      } else if (add) {
        const float4 a = *reinterpret_cast<const float4*>(add + (size_t)i * ld + j0);
        v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
      }
      if (G) *reinterpret_cast<float4*>(G + (size_t)i * ld + j0) = v;
      if (D) *reinterpret_cast<float4*>(D + i * dld + j0) = v;
    }
    if (Gt) {  // rows i >= rows of the tile are zero (zero padding of the operands)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = j0 + c;
        if (j >= rows) break;
        *reinterpret_cast<float4*>(Gt + (size_t)j * ld + i0) =
            make_float4(scale * acc[0][c], scale * acc[1][c], scale * acc[2][c], scale * acc[3][c]);
      }
    }
  }
};

// ---- blocked Cholesky of S with the F / W rows carried along ---------------------

// Rows: S rows [0, R) at Sb, F rows [0, n) at Fb, W rows [0, n) at Wb (ld lds each);
// R a multiple of 4 with S = I on the padding rows/columns.  On return the F rows
// hold F L^-T and the W rows W L^-T (S's lower part is overwritten with L).
// Returns false (block-uniform) if a pivot falls below 0.5 or is not finite.
__device__ inline bool chol_stack(float* Sb, float* Fb, float* Wb, int lds, int R, int n) {
  const int nrow = R + 2 * n;
  auto row = [&](int i) -> float* {
    return i < R ? Sb + i * lds : (i < R + n ? Fb + (i - R) * lds : Wb + (i - R - n) * lds);
  };
  for (int jb = 0; jb < R; jb += 4) {
    // panel diagonal block D = Lp Lp' (every thread, redundantly; block-uniform result)
    float d[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(Sb + (jb + r) * lds + jb);
      d[r][0] = v.x; d[r][1] = v.y; d[r][2] = v.z; d[r][3] = v.w;
    }
    float li[4][4];  // Lp^-1 (lower)
    bool ok = true;
    {
      float l[4][4] = {}, rd[4];  // rd[c] = 1 / l[c][c]
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float s = d[c][c];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < c) s = fmaf(-l[c][q], l[c][q], s);
        ok = ok && (s >= 0.5f) && isfinite(s);
        const float rs = rsqrtf(fmaxf(s, 1e-30f));
        l[c][c] = s * rs;
        rd[c] = rs;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r > c) {
            float t = d[r][c];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q < c) t = fmaf(-l[r][q], l[c][q], t);
            l[r][c] = t * rs;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r < c) { li[r][c] = 0.f; continue; }
          float t = (r == c) ? 1.f : 0.f;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q >= c && q < r) t = fmaf(-l[r][q], li[q][c], t);
          li[r][c] = t * rd[r];
        }
      }
    }
    if (!ok) return false;
    // phase A: rows below the panel get their panel entries z -> z Lp^-T
    for (int i = jb + 4 + threadIdx.x; i < nrow; i += blockDim.x) {
      float* p = row(i) + jb;
      const float4 z = *reinterpret_cast<const float4*>(p);
      const float zv[4] = {z.x, z.y, z.z, z.w};
      float o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q <= c) s = fmaf(zv[q], li[c][q], s);
        o[c] = s;
      }
      *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();
    // phase B: trailing update Z[i][t] -= sum_c z~[i][c] L[t][c] for t >= jb + 4
    // consecutive threads take consecutive rows of one column group: the row loads are
    // conflict-free (ld = 4 mod 8 words) and the group's L rows are broadcasts
    const int g0 = (jb >> 2) + 1, ng = (R >> 2) - g0;
    if (ng > 0) {
      // thread -> (row, pass): the row's panel entries z are loaded once and the column
      // groups g0 + pass, g0 + pass + npass, ... updated in turn (one division per panel)
      const int rows_below = nrow - (jb + 4), nt = blockDim.x;
      const int npass = max(1, nt / rows_below);           // threads per row
      const int pass = threadIdx.x / rows_below, ii0 = threadIdx.x - pass * rows_below;
      const int stride = rows_below > nt ? nt : rows_below;  // more rows than threads: loop
      for (int ii = (pass < npass ? ii0 : rows_below); ii < rows_below; ii += stride) {
        const int i = jb + 4 + ii;
        float* p = row(i);
        const float4 z = *reinterpret_cast<const float4*>(p + jb);
        for (int gg = pass; gg < ng; gg += npass) {
        const int g = g0 + gg;
        if (i < R && 4 * g > i) break;  // S: lower triangle (and diagonal blocks) only
        float4 acc = *reinterpret_cast<const float4*>(p + 4 * g);
        float* accv = &acc.x;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float4 lt = *reinterpret_cast<const float4*>(Sb + (4 * g + t) * lds + jb);
          float s = accv[t];
          s = fmaf(-z.x, lt.x, s);
          s = fmaf(-z.y, lt.y, s);
          s = fmaf(-z.z, lt.z, s);
          s = fmaf(-z.w, lt.w, s);
          accv[t] = s;
        }
        *reinterpret_cast<float4*>(p + 4 * g) = acc;
        }
      }
    }
    __syncthreads();
  }
  return true;
}

}  // namespace gsls
