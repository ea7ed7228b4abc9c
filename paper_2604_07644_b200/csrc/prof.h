// Per-kernel-family CUDA-event timing (bench.py roofline evidence).
// When enabled, every launch site records an event pair on its own stream;
// gsls_prof_read() synchronizes, accumulates durations per family and resets.
#pragma once
#include <cuda_runtime.h>

namespace gsls {

enum ProfId {
  P_LEAF = 0, P_CVF_LQR, P_GAINS, P_COT, P_REPLAY, P_SLS_ASSEMBLE, P_SLS_LEAF, P_SLS_CVF, P_SLS_GAINS,
  P_SLS_MATPROD, P_SLS_PHIU, P_SLS_ROWNORM, P_SLS_SMALL, P_LINEARIZE, P_RTI_MISC, P_ROLLOUT, P_COUNT
};

void prof_begin(int id, cudaStream_t st);
void prof_end(int id, cudaStream_t st, double units);

struct ProfScope {
  int id;
  cudaStream_t st;
  double units;
  ProfScope(int i, cudaStream_t s, double u) : id(i), st(s), units(u) { prof_begin(i, s); }
  ~ProfScope() { prof_end(id, st, units); }
};

}  // namespace gsls
