// Measured FP32 FFMA throughput of the whole GPU (the combine's roofline denominator):
// every SM runs independent FFMA chains; reports TFLOP/s (FMA = 2 flop) from CUDA events.
#include <cstdio>
__global__ void __launch_bounds__(512) k(float* out, int iters, float s) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f);
  }
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += a[i];
  if (t == 1.2345f) out[threadIdx.x] = t;
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 4096);
  const int iters = 1 << 16, blocks = sms * 4, threads = 512;
  k<<<blocks, threads>>>(out, 256, 0.999f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(out, iters, 0.999f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * 16 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  printf("{\"fp32_ffma_tflops\": %.2f, \"sms\": %d, \"method\": \"16 independent FFMA chains x 512 threads x 4 CTAs/SM, best of 5, CUDA events\"}\n", best, sms);
}
