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


// Scratch words of gj_inverse_panel: panel values (NP x 8), pivot rows / steps.
constexpr int gjp_scratch_words(int NP) { return NP * 8 + 2 * NP + 16; }

// Blocked in-place Gauss-Jordan inverse with partial pivoting and no row
// interchanges: panels of 8 pivot columns.  Per panel, one warp eliminates the
// n x 8 panel in its registers (warp-shuffle argmax over the rows not yet
// pivoted, first index on ties as LAPACK i*amax; the in-place rule turns the
// panel into [D; -A_op D] with D the inverse of the pivot block), then every
// thread applies the panel to its columns as one rank-8 update
//     new[i][c] = (i pivot ? 0 : old[i][c]) + sum_s panel[i][s] old[p_s][c],
// so a panel costs two CTA barriers instead of sixteen.  Without interchanges
// the result is the inverse with rows and columns permuted by the pivot order:
// inv[q(i)][p(c)] = W[i][c] (p(k) = pivot row of step k, q = p^-1).
//
// a: input (smem, row-major, lds), read into registers first; work: an NP x lds
// smem buffer (may alias a); inv / invT outputs (may alias a / work: written
// after the last read).  4 threads per row, threads [0, 4*NP) take part;
// named barrier 1.  Returns false when a pivot is zero / non-finite / below
// rel_tol * max|a| (the ill-conditioned-combine rule, lqr.py:229-232).
template <int NP>
__device__ bool gj_inverse_panel(const float* a, float* work, float* inv, float* invT, int lds, int n,
                                 float* scratch, float rel_tol) {
  constexpr int SEG = NP / 4;
  constexpr int NT = NP * 4;
  constexpr int NW = NT / 32;
  constexpr int PW = 8;                                   // panel width
  constexpr int RPL = NP / 32;                            // rows per lane in the panel warp (2 for 64)
  static_assert(NP % 32 == 0 || NP == 80, "panel warp covers NP rows");
  static_assert(NP <= 128, "row index packed in 7 key bits");
  float* pan = scratch;                                   // [NP][PW] eliminated panel
  int* prow = reinterpret_cast<int*>(pan + NP * PW);      // [NP] pivot row of step k
  int* pstep = prow + NP;                                 // [NP] step at which row i pivoted (-1)
  float* misc = reinterpret_cast<float*>(pstep + NP);     // [0] max|a|, [1] fail
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
  if (part && lane == 0) pan[warp] = mx;
  for (int i = tid; i < NP; i += blockDim.x) pstep[i] = -1;
  __syncthreads();  // a fully read (work / inv may alias it from here on)
  if (tid == 0) {
    float m2 = 0.f;
    for (int w = 0; w < NW; ++w) m2 = fmaxf(m2, pan[w]);
    misc[0] = m2;
    misc[1] = 0.f;
  }
  __syncthreads();
  const float thresh = rel_tol * misc[0];
  constexpr int PROWS = (NP + 31) / 32;  // panel rows per lane
  // threads >= NT (CTAs wider than 4*NP) sit out: the named barriers count NT threads
  for (int k0 = 0; part && k0 < n; k0 += PW) {
    const int pw = min(PW, n - k0);
    // ---- publish the rows ----------------------------------------------------------
    if (part && row < n) {
#pragma unroll
      for (int c = 0; c < SEG; c += 4)
        if (q * SEG + c < n)  // 4-column chunks inside the padded row (ld >= round_up(n, 4))
          *reinterpret_cast<float4*>(work + row * lds + q * SEG + c) = make_float4(r[c], r[c + 1], r[c + 2], r[c + 3]);
    }
    bar_named(1, NT);
    // ---- panel elimination by warp 0 (registers + shuffles) --------------------------
    if (warp == 0) {
      float pv[PROWS][PW];
      bool used[PROWS];
#pragma unroll
      for (int h = 0; h < PROWS; ++h) {
        const int i = lane + 32 * h;
        used[h] = !(i < n) || pstep[i] >= 0;
#pragma unroll
        for (int s = 0; s < PW; ++s) pv[h][s] = (i < n && s < pw) ? work[i * lds + k0 + s] : 0.f;
      }
      bool fail = false;
#pragma unroll
      for (int s = 0; s < PW; ++s) {
        if (s < pw) {
          // argmax |pv[i][s]| over unused rows with one redux: key = the bits of |x| with
          // the low 7 mantissa bits replaced by (127 - row), so the lowest row wins ties
          // (as LAPACK i*amax) and near-ties closer than 2^-16 relative
          unsigned best = 0u;
#pragma unroll
          for (int h = 0; h < PROWS; ++h) {
            const int i = lane + 32 * h;
            const unsigned key =
                used[h] ? 0u : ((__float_as_uint(fabsf(pv[h][s])) & ~127u) | (unsigned)(127 - i));
            best = max(best, key);
          }
          const unsigned wbest = __reduce_max_sync(0xffffffffu, best);
          const int pr = 127 - (int)(wbest & 127u);
          const int ph = pr >> 5, pl = pr & 31;
          // pivot row values of the panel, broadcast from its lane
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
          const float ip = __frcp_rn(piv);
#pragma unroll
          for (int h = 0; h < PROWS; ++h) {
            const int i = lane + 32 * h;
            if (i == pr) {  // pivot row: scaled, inverse entry in column s
#pragma unroll
              for (int t = 0; t < PW; ++t) pv[h][t] = (t == s) ? ip : pv[h][t] * ip;
              used[h] = true;
            } else {
              const float fi = pv[h][s] * ip;
#pragma unroll
              for (int t = 0; t < PW; ++t) pv[h][t] = (t == s) ? -fi : fmaf(-fi, prv[t], pv[h][t]);
            }
          }
          if (lane == 0) {
            prow[k0 + s] = pr;
            pstep[pr] = k0 + s;
          }
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
    }
    bar_named(1, NT);
    // ---- rank-pw update of every row, panel columns replaced -------------------------
    if (part) {
      float cf[PW];
      {
        const float4 u = *reinterpret_cast<const float4*>(pan + row * PW);
        const float4 v = *reinterpret_cast<const float4*>(pan + row * PW + 4);
        cf[0] = u.x; cf[1] = u.y; cf[2] = u.z; cf[3] = u.w; cf[4] = v.x; cf[5] = v.y; cf[6] = v.z; cf[7] = v.w;
      }
      const int st = pstep[row];
      const bool mine = (st >= k0 && st < k0 + pw);  // this row pivoted in this panel
      float v[SEG];
#pragma unroll
      for (int c = 0; c < SEG; ++c) v[c] = mine ? 0.f : r[c];
#pragma unroll
      for (int s = 0; s < PW; ++s) {
        if (s < pw) {
          const float* pr = work + prow[k0 + s] * lds + q * SEG;
          const float f = cf[s];
#pragma unroll
          for (int c = 0; c < SEG; c += 4) {
            if (q * SEG + c >= n) break;
            const float4 t = *reinterpret_cast<const float4*>(pr + c);
            v[c] = fmaf(f, t.x, v[c]);
            v[c + 1] = fmaf(f, t.y, v[c + 1]);
            v[c + 2] = fmaf(f, t.z, v[c + 2]);
            v[c + 3] = fmaf(f, t.w, v[c + 3]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < SEG; ++c) {
        const int col = q * SEG + c;
        r[c] = (col >= k0 && col < k0 + pw) ? cf[col - k0] : v[c];
      }
    }
    bar_named(1, NT);  // work is rewritten by the next panel
  }
  __syncthreads();
  const bool ok = misc[1] == 0.f;
  if (part && row < n) {
    const int qi = pstep[row];
#pragma unroll
    for (int c = 0; c < SEG; ++c) {
      const int col = q * SEG + c;
      if (col < n) {
        const int d = prow[col];
        if (inv) inv[qi * lds + d] = r[c];
        if (invT) invT[d * lds + qi] = r[c];
      }
    }
  }
  __syncthreads();
  return ok;
}


// Look-ahead variant of gj_inverse_panel: a dedicated panel warp (warp NT/32,
// so blockDim >= 4*NP + 32) factors panel t+1 while the row threads apply panel
// t's rank-8 update to their registers.  The panel warp first brings panel
// t+1's columns up to date itself (from the published rows and panel t), so
// the two overlap completely; two barriers per panel.  Same arithmetic and
// pivot choices as gj_inverse_panel.  Scratch: gjl_scratch_words(NP).
constexpr int gjl_scratch_words(int NP) { return 2 * NP * 8 + 2 * NP + 16; }

#ifdef GJ_TRACE  // tools/micro/gj_test.cu: clock64 probes of thread 0 and the panel warp
__device__ long long g_gj_trace[256];
#define GJT(i) do { if (threadIdx.x == 0 || threadIdx.x == NT) g_gj_trace[(threadIdx.x == NT ? 128 : 0) + (i)] = clock64(); } while (0)
#define GJS(i) do { if (threadIdx.x == NT) g_gj_trace[200 + (i)] = clock64(); } while (0)
#else
#define GJT(i) do { } while (0)
#define GJS(i) do { } while (0)
#endif

template <int NP>
__device__ bool gj_inverse_lookahead(const float* a, float* work, float* inv, float* invT, int lds, int n,
                                     float* scratch, float rel_tol) {
  constexpr int SEG = NP / 4;
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
  const int row = tid >> 2, q = tid & 3, lane = tid & 31, warp = tid >> 5;
  float r[SEG];
  float mx = 0.f;
  GJT(0);
#pragma unroll
  for (int c = 0; c < SEG; ++c) {
    const int col = q * SEG + c;
    r[c] = (part && row < n && col < n) ? a[row * lds + col] : 0.f;
    mx = fmaxf(mx, fabsf(r[c]));
  }
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
  if (part && row < n) {
#pragma unroll
    for (int c = 0; c < SEG; c += 4)
      if (q * SEG + c < n)
        *reinterpret_cast<float4*>(work + row * lds + q * SEG + c) = make_float4(r[c], r[c + 1], r[c + 2], r[c + 3]);
  }
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
    } else if (part) {  // rank-pw update of this thread's columns, panel columns replaced
      float cf[PW];
      {
        const float4 u = *reinterpret_cast<const float4*>(pan + row * PW);
        const float4 v = *reinterpret_cast<const float4*>(pan + row * PW + 4);
        cf[0] = u.x; cf[1] = u.y; cf[2] = u.z; cf[3] = u.w; cf[4] = v.x; cf[5] = v.y; cf[6] = v.z; cf[7] = v.w;
      }
      const int st = pstep[row];  // entries of panel t+1 may land concurrently: never in [k0, k0 + pw)
      const bool mine = (st >= k0 && st < k0 + pw);
      float v[SEG];
#pragma unroll
      for (int c = 0; c < SEG; ++c) v[c] = mine ? 0.f : r[c];
#pragma unroll
      for (int s = 0; s < PW; ++s) {
        if (s < pw) {
          const float* pr = work + prow[k0 + s] * lds + q * SEG;
          const float f = cf[s];
#pragma unroll
          for (int c = 0; c < SEG; c += 4) {
            if (q * SEG + c >= n) break;
            const float4 tt = *reinterpret_cast<const float4*>(pr + c);
            v[c] = fmaf(f, tt.x, v[c]);
            v[c + 1] = fmaf(f, tt.y, v[c + 1]);
            v[c + 2] = fmaf(f, tt.z, v[c + 2]);
            v[c + 3] = fmaf(f, tt.w, v[c + 3]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < SEG; ++c) {  // panel columns take their eliminated entries (static selects:
        const int rel = q * SEG + c - k0;  // a runtime cf index would put cf in local memory)
        float x = v[c];
#pragma unroll
        for (int s = 0; s < PW; ++s) x = (rel == s && s < pw) ? cf[s] : x;
        r[c] = x;
      }
      if (t < 8) GJT(9 + 4 * t);
    }
    __syncthreads();  // panel t consumed, panel t+1 factored
    if (t < 8) GJT(10 + 4 * t);
    if (t + 1 < npan) {  // publish the rows after panel t
      if (part && row < n) {
#pragma unroll
        for (int c = 0; c < SEG; c += 4)
          if (q * SEG + c < n)
            *reinterpret_cast<float4*>(work + row * lds + q * SEG + c) = make_float4(r[c], r[c + 1], r[c + 2], r[c + 3]);
      }
      __syncthreads();
    }
    if (t < 8) GJT(11 + 4 * t);
  }
  GJT(4);
  const bool ok = misc[1] == 0.f;
  if (part && row < n) {
    const int qi = pstep[row];
#pragma unroll
    for (int c = 0; c < SEG; ++c) {
      const int col = q * SEG + c;
      if (col < n) {
        const int d = prow[col];
        if (inv) inv[qi * lds + d] = r[c];
        if (invT) invT[d * lds + qi] = r[c];
      }
    }
  }
  __syncthreads();
  return ok;
}

template <int NP>
__device__ bool gj_inverse_lookahead44(const float* a, float* work, float* inv, float* invT, int lds, int n,
                                     float* scratch, float rel_tol) {
  constexpr int SEG = NP / 4;
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
