// Shared-memory read bandwidth (bytes/clk/SM) for LDS.128 patterns.
#include <cstdio>
template <int PAT>
__global__ void __launch_bounds__(512, 1) k(int reps, int ld, long long* out, float* sink) {
  extern __shared__ __align__(16) float sm[];
  for (int i = threadIdx.x; i < 48 * 1024 / 4 * 4; i += 512) sm[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 8
    for (int it = 0; it < 16; ++it) {
      int off;
      if (PAT == 0) off = (it * 16 + warp) * 128 + lane * 4;                       // contiguous 512 B / warp
      else off = (it * 4 + (lane >> 3)) * ld + (warp & 1) * 32 + 4 * (lane & 7);   // replay pattern
      off = (off + (r & 7) * 2048) & (48 * 1024 - 1);
      const float4 v = *reinterpret_cast<const float4*>(sm + off);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  long long t1 = clock64();
  sink[threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
  long long* out; float* sink;
  cudaMallocManaged(&out, 8); cudaMalloc(&sink, 4096);
  const int smem = 48 * 1024 * 4;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 1000;
  for (int ld : {64, 68, 72}) {
    k<0><<<1, 512, smem>>>(reps, ld, out, sink); cudaDeviceSynchronize();
    const double b0 = 512.0 * 16 * 16 * reps / out[0];
    k<1><<<1, 512, smem>>>(reps, ld, out, sink); cudaDeviceSynchronize();
    printf("ld=%d  contiguous: %.1f B/clk   replay pattern: %.1f B/clk\n", ld, b0, 512.0 * 16 * 16 * reps / out[0]);
  }
}
