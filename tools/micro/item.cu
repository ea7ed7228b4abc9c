// Isolates the staged-replay item loop: 16 warps, one n x 2n f32 matvec with f64 x per item,
// partial sums + one __syncthreads, then the row epilogue.  Flags add the bulk-copy refill
// (1), DSMEM puts to `fan` other ranks (2), a cluster barrier every item pair (4).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ inline void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count) : "memory");
}
__device__ inline void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(b), "r"(parity) : "memory");
}
__device__ inline void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst), b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ inline void st_remote(const double* local, unsigned rank, double v) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(local);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
constexpr int NT = 512, R = 4;
__device__ __forceinline__ double widen(uint32_t u) {
  const uint32_t hi = ((u >> 3) & 0x0FFFFFFFu) | (u & 0x80000000u);
  return __hiloint2double((int)hi, (int)(u << 29));
}
template <int MODE>
__global__ void __launch_bounds__(NT, 1) k_item(const float* gsrc, int n, int ld, int items, int flags, int fan, int kslog,
                                               long long* out) {
  extern __shared__ __align__(128) unsigned char smb[];
  const int slot = ((2 * n * ld * 4) + 127) / 128 * 128;
  float* ring = (float*)smb;
  double* x = (double*)(smb + R * slot);
  double* y = x + 2 * ld;
  double* part = y + 2 * ld;
  uint64_t* full = (uint64_t*)(part + 2 * NT);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned rank, cs;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  for (int i = tid; i < 2 * ld; i += NT) { x[i] = 1.0 + i * 1e-3; y[i] = 0; }
  if (tid == 0) for (int i = 0; i < R; ++i) mbar_init(full + i, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const unsigned bytes = 2 * n * ld * 4;
  if (tid == 0) for (int i = 0; i < R; ++i) bulk_load(ring + i * slot / 4, gsrc, bytes, full + i);
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const int rows = n, K = 2 * n, KS = 1 << kslog, kc = (((K + KS - 1) / KS) + 3) & ~3;
  int cs_ = 0, cp = 0, h = 0;
  long long t0 = 0, tw = 0, tm = 0, tb = 0, te = 0, ta;
  for (int j = 0; j < items; ++j) {
    if (j == 8) t0 = clock64();
    ta = clock64();
    mbar_wait(full + cs_, cp);
    if (j >= 8) tw += clock64() - ta;
    ta = clock64();
    const float* M = ring + cs_ * slot / 4;
    double* pt = part + h * NT;
    if (warp < (((rows + 31) >> 5) << kslog)) {
      const int rb = warp >> kslog, ks = warp & (KS - 1);
      const int rq = lane & 7, gq = lane >> 3, row0 = rb * 32 + 4 * rq;
      const int k0 = ks * kc, k1 = min(K, k0 + kc);
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      if (row0 < ld) {
#pragma unroll 4
        for (int k = k0 + gq; k < k1; k += 4) {
          const float4 v = *reinterpret_cast<const float4*>(M + k * ld + row0);
          const double xk = x[k];
          if (MODE == 0) {
            a0 = fma((double)v.x, xk, a0); a1 = fma((double)v.y, xk, a1);
            a2 = fma((double)v.z, xk, a2); a3 = fma((double)v.w, xk, a3);
          } else if (MODE == 1) {
            a0 = fma(widen(__float_as_uint(v.x)), xk, a0); a1 = fma(widen(__float_as_uint(v.y)), xk, a1);
            a2 = fma(widen(__float_as_uint(v.z)), xk, a2); a3 = fma(widen(__float_as_uint(v.w)), xk, a3);
          } else if (MODE == 2) {
            a0 = fma((double)v.x, xk, a0); a1 = fma((double)v.y, xk, a1);
            a2 = fma(widen(__float_as_uint(v.z)), xk, a2); a3 = fma(widen(__float_as_uint(v.w)), xk, a3);
          } else {
            const float xf = (float)xk;
            a0 += v.x * xf; a1 += v.y * xf; a2 += v.z * xf; a3 += v.w * xf;
          }
        }
      }
#pragma unroll
      for (int o = 8; o <= 16; o <<= 1) {
        a0 += __shfl_xor_sync(~0u, a0, o); a1 += __shfl_xor_sync(~0u, a1, o);
        a2 += __shfl_xor_sync(~0u, a2, o); a3 += __shfl_xor_sync(~0u, a3, o);
      }
      if (gq == 0) { double* pp = pt + (warp << 5) + 4 * rq; pp[0] = a0; pp[1] = a1; pp[2] = a2; pp[3] = a3; }
    }
    if (j >= 8) tm += clock64() - ta;
    ta = clock64();
    __syncthreads();
    if (j >= 8) tb += clock64() - ta;
    ta = clock64();
    if ((flags & 1) && tid == NT - 32) bulk_load(ring + cs_ * slot / 4, gsrc + (j & 7) * 1024, bytes, full + cs_);
    else if (!(flags & 1) && tid == NT - 32) {  // re-arm without traffic: 16-byte copy
      bulk_load(ring + cs_ * slot / 4, gsrc, 16, full + cs_);
    }
    if (++cs_ == R) { cs_ = 0; cp ^= 1; }
    h ^= 1;
    if (tid < rows) {
      const double* pr = pt + (((tid >> 5) << kslog) << 5) + (tid & 31);
      double s = 0;
      for (int q = 0; q < KS; ++q) s += pr[q << 5];
      y[tid] = s;
      if (flags & 2)
        for (int f = 1; f <= fan; ++f) st_remote(y + tid, (rank + f) % cs, s);
    }
    if (j >= 8) te += clock64() - ta;
    if ((flags & 4) && (j & 1))
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  // drain
  for (int q = 0; q < R; ++q) { mbar_wait(full + cs_, cp); if (++cs_ == R) { cs_ = 0; cp ^= 1; } }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (tid == 0 && rank == 0) out[0] = (t1 - t0) / (items - 8);
  if (tid == 0 && rank == 0) { out[1] = tw / (items - 8); out[2] = tm / (items - 8); out[3] = tb / (items - 8); out[4] = te / (items - 8); }
}
int main() {
  float* g; long long* out;
  cudaMalloc(&g, 64 << 20); cudaMemset(g, 0, 64 << 20);
  cudaMallocManaged(&out, 64);
  const int n = 61, ld = 64;
  const int smem = R * (((2 * n * ld * 4) + 127) / 128 * 128) + 4 * ld * 8 + 2 * NT * 8 + 64;
  void* ks[4] = {(void*)k_item<0>, (void*)k_item<1>, (void*)k_item<2>, (void*)k_item<3>};
  for (auto kk : ks) {
    cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  struct C { int cs, flags, fan, kslog, mode; } cfgs[] = {
      {1, 0, 0, 3, 1}, {1, 0, 0, 3, 2}, {1, 0, 0, 3, 3}, {1, 0, 0, 2, 2},
      {1, 0, 0, 3, 0}, {1, 0, 0, 2, 0}, {1, 1, 0, 3, 0}, {16, 0, 0, 3, 0}, {16, 1, 0, 3, 0}, {16, 2, 1, 3, 0}, {16, 2, 4, 3, 0},
      {16, 2, 15, 3, 0}, {16, 3, 2, 3, 0}, {16, 4, 0, 3, 0}, {16, 7, 2, 3, 0}};
  for (auto& c : cfgs) if (c.mode < 0 || c.mode > 3) c.mode = 0;
  for (auto c : cfgs) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(c.cs); cfg.blockDim = dim3(NT); cfg.dynamicSmemBytes = smem; cfg.attrs = at; cfg.numAttrs = 1;
    void* args[] = {0}; (void)args;
    auto kf = c.mode == 0 ? k_item<0> : c.mode == 1 ? k_item<1> : c.mode == 2 ? k_item<2> : k_item<3>;
    cudaLaunchKernelEx(&cfg, kf, (const float*)g, n, ld, 200, c.flags, c.fan, c.kslog, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode=%d cs=%2d flags=%d fan=%2d KS=%2d: %lld cycles/item (wait %lld matvec %lld bar %lld epi %lld) %s\n", c.mode, c.cs, c.flags, c.fan, 1 << c.kslog, out[0], out[1], out[2], out[3], out[4],
           e ? cudaGetErrorString(e) : "");
  }
}
