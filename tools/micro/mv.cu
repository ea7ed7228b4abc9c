// Throughput of the replay item matvec (n x 2n f32, f64 x) with 16 warps, no epilogue.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double widen(uint32_t u) {
  const uint32_t hi = ((u >> 3) & 0x0FFFFFFFu) | (u & 0x80000000u);
  return __hiloint2double((int)hi, (int)(u << 29));
}
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int n, int ld, int reps, int kslog, long long* out, double* sink) {
  extern __shared__ __align__(16) unsigned char smb[];
  float* M = (float*)smb;
  double* x = (double*)(smb + 2 * n * ld * 4);
  for (int i = threadIdx.x; i < 2 * n * ld; i += 512) M[i] = 1.0f + (i & 7);
  for (int i = threadIdx.x; i < 2 * n; i += 512) x[i] = 0.5 + i;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, rows = n, K = 2 * n;
  const int KS = 1 << kslog, kc = (((K + KS - 1) / KS) + 3) & ~3;
  double tot = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (warp < (((rows + 31) >> 5) << kslog)) {
      const int rb = warp >> kslog, ks = warp & (KS - 1);
      const int rq = lane & 7, gq = lane >> 3, row0 = rb * 32 + 4 * rq;
      const int k0 = ks * kc, k1 = min(K, k0 + kc);
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      float f0 = 0, f1 = 0, f2 = 0, f3 = 0;
#pragma unroll 4
      for (int k = k0 + gq; k < k1; k += 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(M + k * ld + row0);
        const double xk = x[k];
        if (MODE == 0) {
          a0 = fma((double)__uint_as_float(v.x), xk, a0); a1 = fma((double)__uint_as_float(v.y), xk, a1);
          a2 = fma((double)__uint_as_float(v.z), xk, a2); a3 = fma((double)__uint_as_float(v.w), xk, a3);
        } else if (MODE == 1) {
          a0 = fma(widen(v.x), xk, a0); a1 = fma(widen(v.y), xk, a1); a2 = fma(widen(v.z), xk, a2); a3 = fma(widen(v.w), xk, a3);
        } else if (MODE == 2) {
          a0 = fma((double)__uint_as_float(v.x), xk, a0); a1 = fma((double)__uint_as_float(v.y), xk, a1);
          a2 = fma(widen(v.z), xk, a2); a3 = fma(widen(v.w), xk, a3);
        } else {  // smem only
          const float xf = __int_as_float(__double2loint(xk));
          f0 += __uint_as_float(v.x) * xf; f1 += __uint_as_float(v.y) * xf; f2 += __uint_as_float(v.z) * xf; f3 += __uint_as_float(v.w) * xf;
        }
      }
      tot += a0 + a1 + a2 + a3 + f0 + f1 + f2 + f3;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  sink[threadIdx.x] = tot;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / reps;
}
int main() {
  long long* out; double* sink;
  cudaMallocManaged(&out, 8); cudaMalloc(&sink, 4096);
  const int n = 61, ld = 64, smem = 2 * n * ld * 4 + 2 * n * 8;
  void* ks[4] = {(void*)k<0>, (void*)k<1>, (void*)k<2>, (void*)k<3>};
  for (auto f : ks) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[4] = {"f2f", "int-trick", "half/half", "smem-only(f32)"};
  for (int kslog = 1; kslog <= 3; ++kslog)
    for (int m = 0; m < 4; ++m) {
      void* args[] = {(void*)&n, (void*)&ld, nullptr, (void*)&kslog, (void*)&out, (void*)&sink};
      int reps = 200; args[2] = &reps;
      cudaLaunchKernel(ks[m], dim3(1), dim3(512), args, smem, 0);
      cudaDeviceSynchronize();
      printf("KS=%d %-15s %lld cycles / matvec (%d x %d)\n", 1 << kslog, names[m], out[0], n, 2 * n);
    }
}
