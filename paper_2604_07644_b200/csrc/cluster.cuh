// Thread-block-cluster plumbing shared by the replay kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>

namespace gsls {

// ---- thread-block-cluster plumbing ---------------------------------------------
// A replay instance runs on a cluster of CS CTAs (CS = 1 for large batches).
// Every CTA holds a full replica of the replay vectors in its shared memory;
// each phase's outputs are written to all replicas (DSMEM stores) and phases
// are separated by cluster barriers, so every read is CTA-local.

__device__ inline unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ inline unsigned cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ inline void st_remote(const double* local, unsigned rank, double v) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(local);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

struct Cl {
  unsigned rank, cs;
  __device__ void put(double* p, double v) const {  // write v to p in every replica
    *p = v;
    for (unsigned r = 0; r < cs; ++r)
      if (r != rank) st_remote(p, r, v);
  }
  __device__ void put_mask(double* p, double v, unsigned mask) const {  // local + consumer replicas
    *p = v;
    mask &= ~(1u << rank);
    while (mask) {
      const unsigned r = __ffs(mask) - 1;
      mask &= mask - 1;
      st_remote(p, r, v);
    }
  }
  __device__ void sync() const {
    if (cs == 1) {
      __syncthreads();
    } else {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
  }
};

}  // namespace gsls
