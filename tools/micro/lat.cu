// Dependent-chain latency (cycles) of fp64 / conversion / shuffle / shared-memory ops.
#include <cstdio>
__global__ void k(double* o, float* fo, long long* c, int iters) {
  double a = o[0], b = o[1];
  float f = fo[0];
  __shared__ double s[64];
  s[threadIdx.x] = a;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, b);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) a = a + b;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) { a = a + (double)f; f = (float)a; }
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) a = __shfl_xor_sync(~0u, a, 1);
  long long t4 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) { idx = (int)s[idx & 63] & 63; }
  long long t5 = clock64();
  float g = f;
  for (int i = 0; i < iters; ++i) g = fmaf(g, 1.0001f, 0.5f);
  long long t6 = clock64();
  o[threadIdx.x] = a + idx + g;
  if (threadIdx.x == 0) { c[0] = t1 - t0; c[1] = t2 - t1; c[2] = t3 - t2; c[3] = t4 - t3; c[4] = t5 - t4; c[5] = t6 - t5; }
}
int main() {
  double* o; float* fo; long long* c;
  cudaMallocManaged(&o, 64 * 8); cudaMallocManaged(&fo, 64 * 4); cudaMallocManaged(&c, 64);
  for (int i = 0; i < 64; ++i) { o[i] = 0.5; fo[i] = 0.25f; }
  const int it = 1024;
  k<<<1, 32>>>(o, fo, c, it); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, fo, c, it); cudaDeviceSynchronize();
  printf("DFMA %.1f  DADD %.1f  F2F.F64+F2F.F32+DADD %.1f  SHFL(f64) %.1f  LDS.64->idx %.1f  FFMA %.1f cycles\n",
         (double)c[0] / it, (double)c[1] / it, (double)c[2] / it, (double)c[3] / it, (double)c[4] / it, (double)c[5] / it);
}
