// 3xTF32 tensor-core products of the scan's n x n blocks (n <= 64) on tcgen05 -- the
// tensor-core side of the measured TF32 / 3xTF32 vs FP32-FMA decision.
// Used by tools/micro/tc_test.cu; it was wired into the product's two pure-product
// kernels (k_matprod, k_cot_combine) for the in-product A/B of profiles/r02/tc_ab.txt
// and taken out again: slower there (staging-bound, half the occupancy) and less
// accurate through the SLS product chains.
//
// C = At^T B (the SIMT gemm_tn contract: At[k][i] and B[k][j] row-major in shared
// memory, row stride lds) as one CTA-wide tcgen05.mma chain with the fp32 accumulator
// in TMEM.  fp32 accuracy from TF32 inputs by the split x = hi + lo (hi, lo both
// TF32-rounded): C = At_lo^T B_hi + At_hi^T B_lo + At_hi^T B_hi, 24 MMAs of
// M = N = 64, K = 8 (the lo x lo term is below fp32 rounding).  Measured on B200
// (tools/micro/tc_gemm.cu, profiles/r02/tc_gemm.jsonl): 84 TFLOP/s vs 39 for the
// FP32-SIMT 4x4-tile product at the same error (2.6e-7 of max|C| against float64);
// one TF32 pass (133 TFLOP/s) misses the 1e-4 parity bar (3.7e-4).
//
// Operand staging: both operands are transposed into the canonical K-major
// no-swizzle UMMA layout (core matrix = 8 rows x 4 k, 128 B; see canon_k) with their
// hi / lo split; four 16 KB canonical buffers.  (The MN-major descriptor form on the
// untransposed rows -- idesc bits 15/16 with an 8 k-row x 16 B core matrix -- produced
// an all-zero D on B200, tools/micro/tc_test.cu; the transposing stage costs four
// scalar loads per 16-byte chunk and stays bank-conflict free.)
//
// D layout in TMEM for M = 64 (cta_group::1): row i at lane 32 (i / 16) + i % 16,
// column j at column j (checked by the micro's TMEM dump): warp w reads rows
// 16 (w % 4) .. +15 (lanes 0-15 of its sub-partition), columns 32 (w / 4) .. +31.
#pragma once

#include <cstdint>

namespace gsls {
namespace tc {

constexpr int kCanonFloats = 64 * 64;  // one 64 x 64 canonical operand (16 KB)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // sm_100 descriptor version; base offset 0, SWIZZLE_NONE
  return d;
}

// kind::tf32: D f32 (bits 4-5 = 1), A/B TF32 (7-9, 10-12 = 2), both K-major (bits
// 15, 16 clear), N >> 3 (17-22), M >> 4 (24-28)
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

struct Bufs {
  float* a_hi;  // 4 canonical operands, 16 KB each, 128-byte aligned
  float* a_lo;
  float* b_hi;
  float* b_lo;
  uint64_t* bar;   // MMA-completion mbarrier (shared)
  uint32_t* tmem;  // TMEM base address slot (shared)
};

// Warp 0 allocates 64 TMEM columns and thread 0 initializes the mbarrier; every
// thread must call it, followed by a __syncthreads() (done here).
__device__ inline void setup(const Bufs& b) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(b.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b.bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
}

__device__ inline void teardown(const Bufs& b) {
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(*b.tmem));
  }
}

// K-major canonical (the operand transposed while staging): element (i, k) at
// (i >> 3) * 512 + (k >> 2) * 32 + (i & 7) * 4 + (k & 3); LBO (next 4 k) = 128 B,
// SBO (next 8 rows) = 2048 B.  Four scalar loads (k .. k+3 of column i) per chunk;
// threads in chunk order (i & 7 fastest): conflict-free loads and stores.
__device__ __forceinline__ int canon_k(int i, int k) { return (i >> 3) * 512 + (k >> 2) * 32 + (i & 7) * 4 + (k & 3); }

__device__ inline void stage_k(const float* src, int lds, int n, float* hi, float* lo) {
  const int kr = (n + 7) & ~7;
  for (int c = threadIdx.x; c < kr * 16; c += blockDim.x) {
    const int i = ((c / (8 * (kr >> 2))) << 3) + (c & 7), k4 = ((c >> 3) % (kr >> 2)) << 2;
    float x[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) x[t] = (i < n && k4 + t < n) ? src[(k4 + t) * lds + i] : 0.f;
    float h[4], l[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      h[t] = tf32_rna(x[t]);
      l[t] = tf32_rna(x[t] - h[t]);
    }
    const int o = canon_k(i, k4);
    *reinterpret_cast<float4*>(hi + o) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(lo + o) = make_float4(l[0], l[1], l[2], l[3]);
  }
}

// D (TMEM) = At^T B for an n x n product (n <= 64, padded to 64 x 64); on return the
// product is complete in TMEM (all threads waited on the MMA barrier) and the
// operand buffers At / B may be overwritten.  phase: the caller's mbarrier parity,
// flipped here.  Padding: rows / columns >= n of D are zero when the operands'
// padding is (stage() zero-fills beyond n).
__device__ inline void gemm_tn_3x(int n, const float* At, const float* B, int lds, const Bufs& b, uint32_t& phase) {
  stage_k(At, lds, n, b.a_hi, b.a_lo);
  stage_k(B, lds, n, b.b_hi, b.b_lo);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> MMA reads
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
      constexpr uint32_t idesc = idesc_tf32(64, 64);
      const uint32_t d = *b.tmem;
      const uint32_t ah = smem_u32(b.a_hi), al = smem_u32(b.a_lo), bh = smem_u32(b.b_hi), bl = smem_u32(b.b_lo);
      const int kk_end = (n + 7) >> 3;
      uint32_t acc = 0;
      auto chain = [&](uint32_t ab, uint32_t bb) {
        for (int kk = 0; kk < kk_end; ++kk) {
          const uint64_t da = sdesc(ab + kk * 256, 128, 2048), db = sdesc(bb + kk * 256, 128, 2048);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
          acc = 1;
        }
      };
      chain(al, bh);  // small terms first
      chain(ah, bl);
      chain(ah, bh);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(b.bar)));
    }
    __syncwarp();
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(b.bar)),
      "r"(phase));
  phase ^= 1;
  asm volatile("tcgen05.fence::after_thread_sync;");
}

// 32 consecutive TMEM columns of this warp's sub-partition lanes -> registers
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// TMEM product -> shared memory: C[i][j] (row-major, stride ldc) for i < n, j < ldg (the
// zero padding columns included) and, when Ct is not null, Ct[j][i] for j < n, i < ldg
// (C and Ct hold n rows).  Warps 0-7 of the CTA do the reads (the TMEM lane
// restriction: warp w sees sub-partition w % 4); other warps only join the barriers.
// Ends with a barrier.
__device__ inline void store_smem(const Bufs& b, int n, int ldg, float* C, int ldc, float* Ct, int ldct) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 8) {
    const int sub = warp & 3, c0 = (warp >> 2) * 32;
    float v[32];
    ld32(*b.tmem + ((uint32_t)(32 * sub) << 16) + c0, v);
    const int i = 16 * sub + lane;
    if (lane < 16 && i < ldg) {
      if (i < n) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          if (c0 + j < ldg)
            *reinterpret_cast<float4*>(C + i * ldc + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
      if (Ct) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c0 + j < n) Ct[(c0 + j) * ldct + i] = v[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
}

}  // namespace tc
}  // namespace gsls
