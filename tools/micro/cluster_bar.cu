// Microbenchmark: cost of barrier.cluster (release/acquire vs relaxed) and of
// DSMEM broadcast stores, for cluster sizes 1..16 (one CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>

__device__ inline unsigned crank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ inline unsigned csize() { unsigned r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r; }

template <int MODE>
__global__ void k(int iters, int nput, long long* out) {
  extern __shared__ double sm[];
  const unsigned rank = crank(), cs = csize();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE >= 1) {  // each thread < nput broadcasts one double to every rank
      if ((int)threadIdx.x < nput) {
        const unsigned a = (unsigned)__cvta_generic_to_shared(sm + threadIdx.x);
        for (unsigned r = 0; r < cs; ++r) {
          unsigned ra;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
          asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"((double)i) : "memory");
        }
      }
    }
    if (MODE == 2)
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    else
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[blockIdx.y] = t1 - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  const int iters = 2000;
  auto run = [&](auto kern, int cs, int nput, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs, 1); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 150 * 1024;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, kern, iters, nput, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-28s cs=%2d nput=%3d: %7.1f cycles per iteration (%s)\n", name, cs, nput, (double)h / iters,
           cudaGetErrorString(e));
  };
  for (int cs : {1, 2, 4, 8, 16}) {
    run(k<0>, cs, 0, "barrier rel/acq");
    run(k<2>, cs, 0, "barrier relaxed");
    run(k<1>, cs, 64, "put64 + barrier rel/acq");
    run(k<1>, cs, 512, "put512 + barrier rel/acq");
  }
  return 0;
}
