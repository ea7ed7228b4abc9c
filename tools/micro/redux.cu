// Dependent-chain latency of __reduce_max_sync (CREDUX), __shfl_sync and a 5-round shuffle max.
#include <cstdio>
__global__ void k(unsigned* o, long long* c, int iters) {
  unsigned v = threadIdx.x * 7 + o[0];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __reduce_max_sync(0xffffffffu, v) + (threadIdx.x & 3);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (v + i) & 31) + 1;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, s));
    v += threadIdx.x & 1;
  }
  long long t3 = clock64();
  float f = __uint_as_float(v & 0x3fffffff) + 1.0f;
  for (int i = 0; i < iters; ++i) f = __frcp_rn(f) + 1.0f;
  long long t4 = clock64();
  o[threadIdx.x + 32] = v + (unsigned)f;
  if (threadIdx.x == 0) { c[0] = t1 - t0; c[1] = t2 - t1; c[2] = t3 - t2; c[3] = t4 - t3; }
}
int main() {
  unsigned* o; long long* c;
  cudaMallocManaged(&o, 1024); cudaMallocManaged(&c, 64); o[0] = 1;
  const int it = 1000;
  k<<<1, 32>>>(o, c, it); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, it); cudaDeviceSynchronize();
  printf("CREDUX.MAX %.1f  SHFL.IDX %.1f  5-round shfl max %.1f  frcp_rn+FADD %.1f cycles\n", (double)c[0] / it,
         (double)c[1] / it, (double)c[2] / it, (double)c[3] / it);
}
