// Gauss-Jordan inverse with register-resident row segments (the CVF combine's
// (I + Pr Cl)^-1, replacing the reference's solve(M1^T, .) / solve(M2^T, .)
// pair, lqr.py:233-235).
#pragma once

#include "common.cuh"

namespace gsls {

// Blocked Gauss-Jordan inverse with partial pivoting and no row interchanges,
// panels of 8 pivot columns, with look-ahead.  A dedicated panel warp (warp
// NT/32, so blockDim >= 4*NP + 32) eliminates the n x 8 panel t+1 in its
// registers (warp redux argmax over the rows not yet pivoted, first index on
// ties as LAPACK i*amax; the in-place rule turns the panel into [D; -A_op D]
// with D the inverse of the pivot block) while the row threads apply panel
// t's rank-8 update to their register tiles:
//     new[i][c] = (i pivot ? 0 : old[i][c]) + sum_s panel[i][s] old[p_s][c].
// The panel warp first brings panel t+1's columns up to date itself (from the
// published rows and panel t), so the two overlap completely; two barriers
// per panel.  Without interchanges the result is the inverse with rows and
// columns permuted by the pivot order: inv[q(i)][p(c)] = W[i][c] (p(k) = pivot
// row of step k, q = p^-1).
//
// Row threads [0, 4*NP) each own a 4 x TC (row, column) tile, TC = NP / 16,
// i.e. columns TC*cg .. TC*cg + TC - 1 of rows 4*rg .. 4*rg + 3.  The tiles of
// the last column group may reach past n: the shared-memory row stride must
// cover them, lds >= round_up(n, TC) (gj_lds(NP, n)), and those padding
// columns stay zero (they start at zero and every pivot row's padding is zero).
//
// a: input (smem, row-major, lds), read into registers first; work: an NP x lds
// smem buffer (may alias a); inv / invT outputs (may alias a / work: written
// after the last read).  Returns (block-uniform) false when a pivot is zero /
// non-finite / below rel_tol * max|a| (the ill-conditioned-combine rule,
// lqr.py:229-232).  Scratch: gjl_scratch_words(NP).
constexpr int gjl_scratch_words(int NP) { return 2 * NP * 8 + 2 * NP + 16; }

// Row stride for gj_inverse_lookahead44<NP> on n x n: lds_of(n) widened so the
// register tiles of the last column group (TC = NP / 16 columns) stay inside a row.
__host__ __device__ inline int gj_lds(int NP, int n) { return lds_of(round_up(n, NP / 16)); }

#ifdef GJ_TRACE  // tools/micro/gj_test.cu: clock64 probes of thread 0 and the panel warp
__device__ long long g_gj_trace[256];
#define GJT(i) do { if (threadIdx.x == 0 || threadIdx.x == NT) g_gj_trace[(threadIdx.x == NT ? 128 : 0) + (i)] = clock64(); } while (0)
#define GJS(i) do { if (threadIdx.x == NT) g_gj_trace[200 + (i)] = clock64(); } while (0)
#else
#define GJT(i) do { } while (0)
#define GJS(i) do { } while (0)
#endif


template <int NP>
__device__ bool gj_inverse_lookahead44(const float* a, float* work, float* inv, float* invT, int lds, int n,
                                     float* scratch, float rel_tol) {
  constexpr int NT = NP * 4;  // row threads
  constexpr int NW = NT / 32;
  constexpr int PW = 8;
  constexpr int PROWS = (NP + 31) / 32;
  static_assert(NP <= 128, "row index packed in 7 key bits");
  float* pan0 = scratch;                                   // [2][NP][PW] eliminated panels (double buffer)
  int* prow = reinterpret_cast<int*>(pan0 + 2 * NP * PW);  // [NP] pivot row of step k
  int* pstep = prow + NP;                                  // [NP] step at which row i pivoted (-1)
  float* misc = reinterpret_cast<float*>(pstep + NP);      // [0] max|a|, [1] fail
  const int tid = threadIdx.x;
  const bool part = tid < NT;
  const bool pwarp = (tid >> 5) == NW;  // the panel warp
  constexpr int TC = NP / 16;  // columns per row thread: 4 (NP = 64) or 5 (NP = 80)
  static_assert(NP == 64 || NP == 80, "4 x TC row tiles: (NP / 4) x 16 == NP * 4 row threads");
  const int lane = tid & 31, warp = tid >> 5;
  const int rg = tid >> 4, cg = tid & 15;  // rows 4rg..4rg+3, columns TC cg..TC cg+TC-1
  float r[4][TC];
  float mx = 0.f;
  GJT(0);
#pragma unroll
  for (int rr = 0; rr < 4; ++rr)
#pragma unroll
    for (int cc = 0; cc < TC; ++cc) {
      const int row = 4 * rg + rr, col = TC * cg + cc;
      r[rr][cc] = (part && row < n && col < n) ? a[row * lds + col] : 0.f;
      mx = fmaxf(mx, fabsf(r[rr][cc]));
    }
  auto publish_rows = [&]() {  // this thread's TC-column segment of its 4 rows
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      if (4 * rg + rr >= n) break;
      float* dst = work + (4 * rg + rr) * lds + TC * cg;
      if constexpr (TC == 4) {
        *reinterpret_cast<float4*>(dst) = make_float4(r[rr][0], r[rr][1], r[rr][2], r[rr][3]);
      } else {
#pragma unroll
        for (int cc = 0; cc < TC; ++cc) dst[cc] = r[rr][cc];
      }
    }
  };
  mx = warp_max(mx);
  if (part && lane == 0) pan0[warp] = mx;
  for (int i = tid; i < NP; i += blockDim.x) pstep[i] = -1;
  __syncthreads();  // a fully read (work / inv may alias it from here on)
  GJT(1);
  if (tid == 0) {
    float m2 = 0.f;
    for (int w = 0; w < NW; ++w) m2 = fmaxf(m2, pan0[w]);
    misc[0] = m2;
    misc[1] = 0.f;
  }
  // zero the columns past round_up(n, 4) the 8-wide panel loads may touch (never published)
  for (int e = tid; e < n * 8; e += blockDim.x) {
    const int i = e >> 3, cc = ((n + 3) & ~3) + (e & 7);
    if (cc < lds) work[i * lds + cc] = 0.f;
  }
  // publish the rows (pre-panel-0 state)
  if (part && TC * cg < n) publish_rows();
  __syncthreads();
  const float thresh = rel_tol * misc[0];
  GJT(2);
  const int npan = (n + PW - 1) / PW;
  // Panel warp: eliminate panel t (columns k0..k0+pw) from its values pv (post panels < t).
  auto factor = [&](float (&pv)[PROWS][PW], int k0, float* pan) {
    const int pw = min(PW, n - k0);
    bool used[PROWS];
#pragma unroll
    for (int h = 0; h < PROWS; ++h) {
      const int i = lane + 32 * h;
      used[h] = !(i < n) || pstep[i] >= 0;
    }
    if (k0 == 0) GJS(0);
    bool fail = false;
    // pivot-search key of row i for the current step: |value| bits, row index in the low 7
    unsigned best = 0u;
#pragma unroll
    for (int h = 0; h < PROWS; ++h) {
      const unsigned key = used[h] ? 0u : ((__float_as_uint(fabsf(pv[h][0])) & ~127u) | (unsigned)(127 - (lane + 32 * h)));
      best = max(best, key);
    }
#pragma unroll
    for (int s = 0; s < PW; ++s) {
      if (s < pw) {
        const unsigned wbest = __reduce_max_sync(0xffffffffu, best);
        const int pr = 127 - (int)(wbest & 127u);
        const int ph = pr >> 5, pl = pr & 31;
        float prv[PW];
#pragma unroll
        for (int t = 0; t < PW; ++t) {
          float v = 0.f;
#pragma unroll
          for (int h = 0; h < PROWS; ++h) if (h == ph) v = pv[h][t];
          prv[t] = __shfl_sync(0xffffffffu, v, pl);
        }
        const float piv = prv[s];
        if (!(fabsf(piv) > thresh) || !isfinite(piv)) fail = true;
        // next step's key without the reciprocal: |piv a_{i,s+1} - a_{i,s} prv_{s+1}| =
        // |piv| |a'_{i,s+1}|, and |piv| is common to every row, so the argmax is that of the
        // updated column; the pivot search of step s+1 then overlaps this step's update
        if (s + 1 < PW) {
          best = 0u;
#pragma unroll
          for (int h = 0; h < PROWS; ++h) {
            const bool live = !(used[h] || (lane + 32 * h) == pr);
            const float sc = fmaf(piv, pv[h][s + 1], -(pv[h][s] * prv[s + 1]));
            const unsigned key = live ? ((__float_as_uint(fabsf(sc)) & ~127u) | (unsigned)(127 - (lane + 32 * h))) : 0u;
            best = max(best, key);
          }
        }
        // MUFU reciprocal + one Newton step (~28 cycles on the pivot chain vs ~78 for
        // __frcp_rn's range-checked path; tools/micro/redux.cu).  |piv| > thresh > 0 here.
        float ip;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ip) : "f"(piv));
        ip = fmaf(ip, fmaf(-piv, ip, 1.f), ip);
        // branch-free: every row takes the elimination update, the pivot row (lane-uniform
        // values prv * ip) is selected in afterwards
        float pip[PW];
#pragma unroll
        for (int t = 0; t < PW; ++t) pip[t] = (t == s) ? ip : prv[t] * ip;
#pragma unroll
        for (int h = 0; h < PROWS; ++h) {
          const bool isp = (lane + 32 * h) == pr;
          const float fi = pv[h][s] * ip;
#pragma unroll
          for (int t = 0; t < PW; ++t) {
            const float e = (t == s) ? -fi : fmaf(-fi, prv[t], pv[h][t]);
            pv[h][t] = isp ? pip[t] : e;
          }
          used[h] = used[h] || isp;
        }
        if (lane == 0) {
          prow[k0 + s] = pr;
          pstep[pr] = k0 + s;
        }
        if (k0 == 0) GJS(1 + s);
      }
    }
#pragma unroll
    for (int h = 0; h < PROWS; ++h) {
      const int i = lane + 32 * h;
      if (i < NP) {
        *reinterpret_cast<float4*>(pan + i * PW) = make_float4(pv[h][0], pv[h][1], pv[h][2], pv[h][3]);
        *reinterpret_cast<float4*>(pan + i * PW + 4) = make_float4(pv[h][4], pv[h][5], pv[h][6], pv[h][7]);
      }
    }
    if (lane == 0 && fail) misc[1] = 1.f;
  };
  if (pwarp) {  // panel 0 from the published rows
    float pv[PROWS][PW];
#pragma unroll
    for (int h = 0; h < PROWS; ++h) {
      const int i = lane + 32 * h;
#pragma unroll
      for (int t = 0; t < PW; ++t) pv[h][t] = (i < n && t < min(PW, n)) ? work[i * lds + t] : 0.f;
    }
    factor(pv, 0, pan0);
  }
  __syncthreads();
  GJT(3);
  for (int t = 0; t < npan; ++t) {
    const int k0 = t * PW, pw = min(PW, n - k0);
    if (t < 8) GJT(8 + 4 * t);
    const float* pan = pan0 + (t & 1) * NP * PW;
    if (pwarp) {
      if (t + 1 < npan) {  // panel t+1's columns after panel t, for every row, then eliminate them
        const int k1 = k0 + PW, pw1 = min(PW, n - k1);
        // pivot rows' panel-(t+1) segments: lane-uniform, loaded once as float4 pairs
        float prs[PW][PW];
#pragma unroll
        for (int s = 0; s < PW; ++s) {
          const float* pr = work + prow[k0 + min(s, pw - 1)] * lds + k1;
          const float4 u = *reinterpret_cast<const float4*>(pr);
          const float4 w = *reinterpret_cast<const float4*>(pr + 4);
          const bool live = s < pw;
          prs[s][0] = live ? u.x : 0.f; prs[s][1] = live ? u.y : 0.f; prs[s][2] = live ? u.z : 0.f;
          prs[s][3] = live ? u.w : 0.f; prs[s][4] = live ? w.x : 0.f; prs[s][5] = live ? w.y : 0.f;
          prs[s][6] = live ? w.z : 0.f; prs[s][7] = live ? w.w : 0.f;
        }
        float pv[PROWS][PW];
#pragma unroll
        for (int h = 0; h < PROWS; ++h) {
          const int i = lane + 32 * h;
          const bool valid = i < n;
          const int st = valid ? pstep[i] : -1;
          const bool mine = st >= k0 && st < k0 + pw;
          float cf[PW], v[PW];
          if (valid) {
            const float4 c0 = *reinterpret_cast<const float4*>(pan + i * PW);
            const float4 c1 = *reinterpret_cast<const float4*>(pan + i * PW + 4);
            cf[0] = c0.x; cf[1] = c0.y; cf[2] = c0.z; cf[3] = c0.w; cf[4] = c1.x; cf[5] = c1.y; cf[6] = c1.z; cf[7] = c1.w;
            const float4 o0 = *reinterpret_cast<const float4*>(work + i * lds + k1);
            const float4 o1 = *reinterpret_cast<const float4*>(work + i * lds + k1 + 4);
            v[0] = o0.x; v[1] = o0.y; v[2] = o0.z; v[3] = o0.w; v[4] = o1.x; v[5] = o1.y; v[6] = o1.z; v[7] = o1.w;
          } else {
#pragma unroll
            for (int c = 0; c < PW; ++c) { cf[c] = 0.f; v[c] = 0.f; }
          }
#pragma unroll
          for (int c = 0; c < PW; ++c) v[c] = mine ? 0.f : v[c];
#pragma unroll
          for (int s = 0; s < PW; ++s)
#pragma unroll
            for (int c = 0; c < PW; ++c) v[c] = fmaf(cf[s], prs[s][c], v[c]);
#pragma unroll
          for (int c = 0; c < PW; ++c) pv[h][c] = (valid && c < pw1) ? v[c] : 0.f;
        }
        factor(pv, k1, pan0 + ((t + 1) & 1) * NP * PW);
        if (t < 8) GJT(9 + 4 * t);
      }
    } else if (part) {  // rank-pw update of this thread's 4x4 tile, panel columns replaced
      float cf[4][PW];
      bool mine[4];
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const int i = 4 * rg + rr;
        const float4 u = *reinterpret_cast<const float4*>(pan + i * PW);
        const float4 w = *reinterpret_cast<const float4*>(pan + i * PW + 4);
        cf[rr][0] = u.x; cf[rr][1] = u.y; cf[rr][2] = u.z; cf[rr][3] = u.w;
        cf[rr][4] = w.x; cf[rr][5] = w.y; cf[rr][6] = w.z; cf[rr][7] = w.w;
        const int st = pstep[i];  // entries of panel t+1 may land concurrently: never in [k0, k0 + pw)
        mine[rr] = (st >= k0 && st < k0 + pw);
      }
      float v[4][TC];
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
#pragma unroll
        for (int cc = 0; cc < TC; ++cc) v[rr][cc] = mine[rr] ? 0.f : r[rr][cc];
      if (TC * cg < n) {
#pragma unroll
        for (int s = 0; s < PW; ++s) {
          if (s < pw) {
            const float* pr = work + prow[k0 + s] * lds + TC * cg;
            float tt[TC];
            if constexpr (TC == 4) {
              const float4 q4 = *reinterpret_cast<const float4*>(pr);
              tt[0] = q4.x; tt[1] = q4.y; tt[2] = q4.z; tt[3] = q4.w;
            } else {
#pragma unroll
              for (int cc = 0; cc < TC; ++cc) tt[cc] = pr[cc];
            }
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
              const float f = cf[rr][s];
#pragma unroll
              for (int cc = 0; cc < TC; ++cc) v[rr][cc] = fmaf(f, tt[cc], v[rr][cc]);
            }
          }
        }
      }
#pragma unroll
      for (int cc = 0; cc < TC; ++cc) {  // panel columns take their eliminated entries
        const int rel = TC * cg + cc - k0;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          float x = v[rr][cc];
#pragma unroll
          for (int s = 0; s < PW; ++s) x = (rel == s && s < pw) ? cf[rr][s] : x;
          r[rr][cc] = x;
        }
      }
      if (t < 8) GJT(9 + 4 * t);
    }
    __syncthreads();  // panel t consumed, panel t+1 factored
    if (t < 8) GJT(10 + 4 * t);
    if (t + 1 < npan) {  // publish the rows after panel t
      if (part && TC * cg < n) publish_rows();
      __syncthreads();
    }
    if (t < 8) GJT(11 + 4 * t);
  }
  GJT(4);
  const bool ok = misc[1] == 0.f;
  if (part) {
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int row = 4 * rg + rr;
      if (row >= n) break;
      const int qi = pstep[row];
#pragma unroll
      for (int cc = 0; cc < TC; ++cc) {
        const int col = TC * cg + cc;
        if (col < n) {
          const int d = prow[col];
          if (inv) inv[qi * lds + d] = r[rr][cc];
          if (invT) invT[d * lds + qi] = r[rr][cc];
        }
      }
    }
  }
  __syncthreads();
  return ok;
}

}  // namespace gsls
