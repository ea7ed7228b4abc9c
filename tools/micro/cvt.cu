// Per-SM throughput of f32->f64 conversion, fp64 FMA and an integer widening trick.
#include <cstdio>
#include <cstdint>
__global__ void k_cvt(const float* in, double* out, int iters, long long* cyc) {
  float f0 = in[threadIdx.x], f1 = f0 + 1.f, f2 = f0 + 2.f, f3 = f0 + 3.f;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 += (double)f0; a1 += (double)f1; a2 += (double)f2; a3 += (double)f3;
    f0 += 1e-7f; f1 += 1e-7f; f2 += 1e-7f; f3 += 1e-7f;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dfma(const float* in, double* out, int iters, long long* cyc) {
  double x = in[threadIdx.x], a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 1, b1 = 2, b2 = 3, b3 = 4;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = fma(b0, x, a0); a1 = fma(b1, x, a1); a2 = fma(b2, x, a2); a3 = fma(b3, x, a3);
    b0 = fma(b0, x, a3); b1 = fma(b1, x, a2); b2 = fma(b2, x, a1); b3 = fma(b3, x, a0);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + b0 + b1 + b2 + b3;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
__device__ __forceinline__ double widen(uint32_t u) {  // f * 2^-896, exact for finite f
  const uint32_t hi = ((u >> 3) & 0x0FFFFFFFu) | (u & 0x80000000u);
  return __hiloint2double((int)hi, (int)(u << 29));
}
__global__ void k_trick(const float* in, double* out, int iters, long long* cyc) {
  uint32_t u0 = __float_as_uint(in[threadIdx.x]), u1 = u0 + 1, u2 = u0 + 2, u3 = u0 + 3;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 += widen(u0); a1 += widen(u1); a2 += widen(u2); a3 += widen(u3);
    u0 += 5; u1 += 5; u2 += 5; u3 += 5;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  float* in; double* out; long long* cyc;
  cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 4096);
  cudaMalloc(&out, 148 * 1024 * 8); cudaMallocManaged(&cyc, 8);
  const int iters = 4096;
  for (int t = 128; t <= 1024; t *= 2) {
    k_cvt<<<1, t>>>(in, out, iters, cyc); cudaDeviceSynchronize();
    printf("threads %4d  cvt.f64.f32: %.1f /clk/SM", t, 4.0 * iters * t / cyc[0]);
    k_dfma<<<1, t>>>(in, out, iters, cyc); cudaDeviceSynchronize();
    printf("  dfma: %.1f /clk/SM", 8.0 * iters * t / cyc[0]);
    k_trick<<<1, t>>>(in, out, iters, cyc); cudaDeviceSynchronize();
    printf("  trick(+dadd): %.1f /clk/SM\n", 4.0 * iters * t / cyc[0]);
  }
  return 0;
}
