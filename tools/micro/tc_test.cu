// Unit test of csrc/tc.cuh (the product path's 3xTF32 tcgen05 GEMM): C = At^T B for
// n = 4 .. 64 from row-major smem operands (stride lds_of(n), zero padding to ldg),
// read back in both orientations, against a float64 host product; prints one line per
// n and "tc_test ok" when every error is below 1e-6 of max|C| and the padding is zero.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2604_07644_b200/csrc -I. -o tc_test tc_test.cu
#include <cmath>
#include <cstdio>
#include <random>
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "smallmat.cuh"
#include "tc.cuh"

namespace gsls {
void set_last_error(const char*, const char*, int) {}
}
using namespace gsls;

__global__ void __launch_bounds__(256) k_test(const float* At, const float* B, float* C, float* Ct, int n) {
  const int ldg = ldg_of(n), lds = lds_of(n);
  C += (size_t)blockIdx.x * n * ldg;  // many CTAs per SM (TMEM allocation shared): one output each
  Ct += (size_t)blockIdx.x * n * ldg;
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem;
  tc::Bufs tb{sm, sm + tc::kCanonFloats, sm + 2 * tc::kCanonFloats, sm + 3 * tc::kCanonFloats, &bar, &tmem};
  float* a = sm + 4 * tc::kCanonFloats;
  float* b = a + (size_t)n * lds;
  cta_load_async(a, lds, At, n);
  cta_load_async(b, lds, B, n);
  cp_async_commit();
  tc::setup(tb);
  cp_async_wait<0>();
  __syncthreads();
  uint32_t phase = 0;
  for (int rep = 0; rep < 2; ++rep) {  // twice: the mbarrier phase flips
    tc::gemm_tn_3x(n, a, b, lds, tb, phase);
    if (rep == 0) {
      tc::store_smem(tb, n, ldg, a + 0, lds, nullptr, lds);  // overwrite At with C, recompute from the original
      cta_load_async(a, lds, At, n);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
    }
  }
  tc::store_smem(tb, n, ldg, a, lds, b, lds);
  cta_store(C, a, lds, n);
  cta_store(Ct, b, lds, n);
  tc::teardown(tb);
}

int main() {
  std::mt19937 rng(3);
  std::normal_distribution<double> nd;
  bool ok = true;
  for (int n : {4, 6, 8, 12, 13, 25, 29, 32, 57, 61, 62, 63, 64}) {
    const int ldg = ldg_of(n), lds = lds_of(n);
    std::vector<float> At((size_t)n * ldg, 0.f), B((size_t)n * ldg, 0.f), C((size_t)n * ldg), Ct((size_t)n * ldg);
    for (int k = 0; k < n; ++k)
      for (int i = 0; i < n; ++i) {
        At[k * ldg + i] = (float)nd(rng);
        B[k * ldg + i] = (float)nd(rng);
      }
    float *dA, *dB, *dC, *dCt;
    cudaMalloc(&dA, sizeof(float) * At.size());
    cudaMalloc(&dB, sizeof(float) * B.size());
    const int grid = 2000;
    cudaMalloc(&dC, sizeof(float) * C.size() * grid);
    cudaMalloc(&dCt, sizeof(float) * Ct.size() * grid);
    cudaMemcpy(dA, At.data(), sizeof(float) * At.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), sizeof(float) * B.size(), cudaMemcpyHostToDevice);
    const size_t sb = (4 * tc::kCanonFloats + 2 * (size_t)n * lds) * sizeof(float);
    cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    k_test<<<grid, 256, sb>>>(dA, dB, dC, dCt, n);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("n=%d: %s\n", n, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> Call(C.size() * grid), Ctall(C.size() * grid);
    cudaMemcpy(Call.data(), dC, sizeof(float) * Call.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(Ctall.data(), dCt, sizeof(float) * Ctall.size(), cudaMemcpyDeviceToHost);
    int differ = 0;  // every CTA's product must equal CTA 0's bitwise
    for (int g = 1; g < grid; ++g)
      for (size_t e = 0; e < C.size(); ++e)
        differ += Call[g * C.size() + e] != Call[e] || Ctall[g * C.size() + e] != Ctall[e];
    if (differ) printf("n=%d: %d elements differ between CTAs\n", n, differ);
    ok &= differ == 0;
    std::copy(Call.begin(), Call.begin() + C.size(), C.begin());
    std::copy(Ctall.begin(), Ctall.begin() + C.size(), Ct.begin());
    double emax = 0, cmax = 0, pad = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < ldg; ++j) {
        double s = 0;
        if (j < n)
          for (int k = 0; k < n; ++k) s += (double)At[k * ldg + i] * (double)B[k * ldg + j];
        if (j >= n) {
          pad = fmax(pad, fabs(C[i * ldg + j]));
          continue;
        }
        emax = fmax(emax, fabs(s - C[i * ldg + j]));
        emax = fmax(emax, fabs(s - Ct[j * ldg + i]));
        cmax = fmax(cmax, fabs(s));
      }
    for (int j = 0; j < n; ++j)
      for (int i = n; i < ldg; ++i) pad = fmax(pad, fabs(Ct[j * ldg + i]));
    const bool good = emax / cmax < 1e-6 && pad == 0.0;
    ok &= good;
    double s00 = 0, s01 = 0, s10 = 0;
    for (int k = 0; k < n; ++k) {
      s00 += (double)At[k * ldg] * B[k * ldg];
      s01 += (double)At[k * ldg] * B[k * ldg + 1];
      s10 += (double)At[k * ldg + 1] * B[k * ldg];
    }
    printf("n=%2d rel err %.3g pad %.3g %s  C00 %.4f (%.4f) C01 %.4f (%.4f) C10 %.4f (%.4f)\n", n, emax / cmax, pad,
           good ? "ok" : "FAIL", C[0], s00, C[1], s01, C[ldg], s10);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
    cudaFree(dCt);
  }
  printf(ok ? "tc_test ok\n" : "tc_test FAILED\n");
  return ok ? 0 : 1;
}
