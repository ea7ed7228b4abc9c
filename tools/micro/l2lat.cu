// Pointer-chase latency of global loads from an L2-resident buffer (single thread).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__global__ void chase(const unsigned* p, int iters, unsigned* out, long long* cyc) {
  unsigned i = 0;
  long long t0 = clock64();
  for (int k = 0; k < iters; ++k) i = p[i];
  long long t1 = clock64();
  out[0] = i;
  cyc[0] = t1 - t0;
}
int main() {
  for (size_t mb : {1, 4, 16, 64}) {
    size_t n = mb * 1024 * 1024 / 4;
    std::vector<unsigned> h(n);
    // random cycle over cache lines (stride 32 words = 128 B)
    size_t lines = n / 32;
    std::vector<unsigned> perm(lines);
    for (size_t i = 0; i < lines; ++i) perm[i] = i;
    unsigned long long x = 88172645463325252ull;
    for (size_t i = lines - 1; i > 0; --i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; size_t j = x % (i + 1); std::swap(perm[i], perm[j]); }
    for (size_t i = 0; i < lines; ++i) h[perm[i] * 32] = perm[(i + 1) % lines] * 32;
    unsigned *d, *o; long long* c;
    cudaMalloc(&d, n * 4); cudaMalloc(&o, 4); cudaMalloc(&c, 8);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    int iters = 20000;
    chase<<<1, 1>>>(d, iters, o, c);  // warm
    chase<<<1, 1>>>(d, iters, o, c);
    long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("buffer %3zu MB: %.0f cycles per dependent load\n", mb, (double)hc / iters);
    cudaFree(d); cudaFree(o); cudaFree(c);
  }
}
