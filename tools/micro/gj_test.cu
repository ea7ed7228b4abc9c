// Unit test of the production shared-memory Gauss-Jordan inverse (gj.cuh) on random matrices,
// including every n in (64, 80] whose last column tile reaches past round_up(n, 4).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/micro/gj_test.cu -o tools/micro/gj_test
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#define GJ_LA(NP_) gj_inverse_lookahead44<NP_>
#ifndef GJ_REPS
#define GJ_REPS 9
#endif

#include "../../paper_2604_07644_b200/csrc/gj.cuh"
using namespace gsls;
namespace gsls { void set_last_error(const char*, const char*, int) {} }

template <int NP>
__global__ void __launch_bounds__(NP == 64 ? 288 : 416) k(const float* A, float* out, int n, int* ok) {
  extern __shared__ float sm[];
  const int lds = gj_lds(NP, n);
  float* a = sm;
  float* work = a + NP * lds;
  float* invT = work + NP * lds;
  float* scr = invT + NP * lds;
  for (int e = threadIdx.x; e < n * lds; e += blockDim.x) a[e] = (e % lds < n) ? A[(e / lds) * n + e % lds] : 0.f;
  __syncthreads();
  bool r;
  long long t0 = clock64();
  for (int rep = 0; rep < GJ_REPS; ++rep) {  // timing repetitions (a is re-read each time)
    GJ_LA(NP)(a, work, nullptr, invT, lds, n, scr, 1e-10f);
    for (int e = threadIdx.x; e < n * lds; e += blockDim.x) a[e] = (e % lds < n) ? A[(e / lds) * n + e % lds] : 0.f;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    printf("  n=%d lookahead: %lld cycles per inverse (incl. reload)\n", n, (t1 - t0) / GJ_REPS);
#ifdef GJ_TRACE
    const long long* g = g_gj_trace;
    printf("   t0: setup %lld publish %lld panel0 %lld | panels (upd | sync | publish):", g[1] - g[0], g[2] - g[1], g[3] - g[2]);
    for (int t = 0; t < 8 && g[8 + 4 * t]; ++t) printf(" %lld|%lld|%lld", g[9 + 4 * t] - g[8 + 4 * t], g[10 + 4 * t] - g[9 + 4 * t], g[11 + 4 * t] - g[10 + 4 * t]);
    printf("\n   panel warp factor(t+1):");
    for (int t = 0; t < 8 && g[128 + 8 + 4 * t]; ++t) printf(" %lld", g[128 + 9 + 4 * t] - g[128 + 8 + 4 * t]);
    printf("  total %lld\n   factor(panel 0) steps:", g[4] - g[0]);
    for (int q = 1; q <= 8; ++q) printf(" %lld", g[200 + q] - g[200 + q - 1]);
#endif
    printf("\n");
  }
  // canary: a row of the buffer past the matrix must come back untouched
  const bool canary = n < NP;  // row n of work exists and nothing may write it
  for (int e = threadIdx.x; canary && e < lds; e += blockDim.x) work[n * lds + e] = 7.f;
  __syncthreads();
  r = GJ_LA(NP)(a, work, work, invT, lds, n, scr, 1e-10f);
  for (int e = threadIdx.x; canary && e < lds; e += blockDim.x)
    if (work[n * lds + e] != 7.f) r = false;
  __syncthreads();
  if (threadIdx.x == 0) *ok = r;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    out[e] = work[(e / n) * lds + e % n];
    out[n * n + e] = invT[(e % n) * lds + e / n];
  }
}

int main() {
  int bad = 0;
  for (int n : {6, 8, 13, 57, 61, 64, 65, 66, 67, 68, 70, 75, 76, 77, 79, 80}) {
    std::vector<float> h(n * n);
    srand(n);
    for (int i = 0; i < n * n; ++i) h[i] = (rand() / (float)RAND_MAX - 0.5f) + ((i / n == i % n) ? 2.f : 0.f);
    float *dA, *dO; int* dok;
    cudaMalloc(&dA, n * n * 4); cudaMalloc(&dO, 2 * n * n * 4); cudaMalloc(&dok, 4);
    cudaMemcpy(dA, h.data(), n * n * 4, cudaMemcpyHostToDevice);
    const int sb = (3 * 80 * gj_lds(80, n) + 4096) * 4;
    cudaFuncSetAttribute(k<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb); cudaFuncSetAttribute(k<80>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
    {
      if (n <= 64) k<64><<<1, 288, sb>>>(dA, dO, n, dok); else k<80><<<1, 416, sb>>>(dA, dO, n, dok);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      std::vector<float> o(2 * n * n); int ok;
      cudaMemcpy(o.data(), dO, 2 * n * n * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(&ok, dok, 4, cudaMemcpyDeviceToHost);
      double err = 0, errT = 0;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          double s = 0, sT = 0;
          for (int t = 0; t < n; ++t) { s += (double)o[i * n + t] * h[t * n + j]; sT += (double)o[n * n + i * n + t] * h[t * n + j]; }
          err = fmax(err, fabs(s - (i == j)));
          errT = fmax(errT, fabs(sT - (i == j)));
        }
      const bool pass = ok && e == cudaSuccess && err < 1e-3 && errT < 1e-3;
      bad += !pass;
      printf("n=%d ok=%d |inv*A-I|=%.3g |invT'*A-I|=%.3g (%s) %s\n", n, ok, err, errT, cudaGetErrorString(e),
             pass ? "PASS" : "FAIL");
    }
  }
  return bad != 0;
}
