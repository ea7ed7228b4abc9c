// Host-side solver context: scan plans, device workspace and the LQR
// factorization cache for one set of dimensions (gsls_ctx in include/gsls.h).
#pragma once

#include <string>
#include <vector>

#include "common.cuh"
#include "plan.h"

namespace gsls {

constexpr size_t kReplaySmemMax = 220 * 1024;  // replay vectors live in smem up to this size

// Device view of the cache, passed by value to kernels.
struct DevLqr {
  int n, m, c, nf, N, ldg, mtot;
  // CVF plan (reverse scan over N+1 elements)
  const int4* cvf_ops;
  const int* cvf_out;
  const int* cvf_loff;   // layer offsets (cvf_layers + 1)
  const int* cvf_leaf;   // per leaf: bit 3 = C stored as a factor (upload_plan)
  const int* cvf_blive;  // per layer: ops whose result a later op reads (first in the layer;
                         // the rest have a dead b: no [Psi -Y] record, no b replay)
  int cvf_nslots, cvf_nops, cvf_layers;
  // COT plan (forward scan over N elements)
  const int4* cot_ops;
  const int* cot_out;
  const int* cot_loff;
  int cot_nslots, cot_nops, cot_layers;
  // scan values (matrices) per instance: [batch][slots][n*ldg]
  float *Ps, *As, *Cs;   // CVF P, A, C
  float* ATs;            // CVF A transposed (both orientations kept; see k_cvf_combine)
  float* cvf_rec;        // [batch][cvf_nops][4][n*ldg]: Ups, X = Ups Pr, Psi, -Y (Y = Psi Cl), column-major
  float* cotA;           // [batch][cot_nslots][n*ldg]
  float* cotAT;          // transposed
  float* cot_rec;        // [batch][cot_nops][n*ldg]: A_later (column-major)
  // per-stage cache, unpadded row-major: [batch][N][...]
  double* Rhat;          // [batch][N][m*m] augmented R (float64)
  double* Shat64;        // [batch][N][m*n] augmented S (float64, for the gains)
  float *Shat, *Rinv, *Gamma, *K;  // m*n, m*m, m*m, m*n (float32, replay operands)
  double* cvec;          // [batch][N][n]  P_{k+1} b_k
  double* v0;            // [batch][n]     Abar_0 dx0
  double* last_k;        // [batch][N][m]   feedforward of the last replay
  double* last_p;        // [batch][N+1][n] cost-to-go gradients of the last replay
  // Fused per-stage operators of the ADMM iteration (rho-dependent, rebuilt with
  // the cache), float32 column-major with padded leading dimensions so every
  // per-iteration product is a coalesced 16-byte-load matvec (admm.cu):
  //   [pv; bv]_k = pb0_k + X23_k (y - z)_k          X23: rows 2n, cols c, ld ld2n
  //   kf_k       = kk0_k + [X5 X4]_k [p+; w]_k      XK: m x (n + c), ld ldm
  //   cb_k       = B_k kf_k + b_k                   Bcm: n x m, ld ldn
  //   G_k        = [Z D]_k [dx; kf]_k               ZD: c x (n + m), ld ldc  (Z = C + D K)
  int ldm, ldn, ldc, ld2n;
  FastDiv fd_ldg, fd_m, fd_n, fd_c, fd_ldm, fd_ldn, fd_ldc, fd_ld2n;  // the per-stage kernels' loop indices
  float *X23, *XK, *Bcm, *ZD;
  // physical storage of the replay vectors per scan slot (plan.h compress_slots)
  const int* cvf_phys;
  const int* cot_phys;
  int cvf_nphys, cot_nphys;
  double *pb0, *kk0;
  ErrSlot* err;          // [batch]
  // device-side instance count of a build launched over the whole batch (graph-captured
  // ADMM loop): CTAs with blockIdx.y >= *build_count exit at once; nullptr: host-sized grid
  const int* build_count;
};

struct Ctx {
  gsls_dims_t dims{};
  int ldg = 0, mtot = 0;
  ScanPlan cvf, cot;
  std::vector<int> cvf_layer_off, cot_layer_off;  // host copies
  int cvf_max_layer = 0, cot_max_layer = 0;
  std::vector<int> cvf_phys, cot_phys;
  // device allocations
  std::vector<void*> allocs;
  int64_t bytes = 0;
  DevLqr dev{};
  int* d_inst_all = nullptr;   // 0..batch-1
  int* d_inst_list = nullptr;  // scratch list (batch): instances of a replay launch
  int* d_build_list = nullptr; // scratch list (batch): instances of a cache rebuild
  cudaStream_t side = nullptr;  // ADMM driver: rebuild + replay of the rebuilt instances, beside the others
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t step_side = nullptr;  // gsls_rti_step: the ADMM's first build beside the SLS chain
  cudaEvent_t step_fork = nullptr, step_join = nullptr;
  int32_t* d_status = nullptr; // [batch] per-instance ADMM exit status
  int* d_counts = nullptr;     // [2] graph-captured ADMM loop: replay / build instance counts
  cudaStream_t body_stream = nullptr;  // capture stream of the captured loop's body graph
  double* d_scratch = nullptr; // global fallback for replay vectors
  size_t scratch_floats = 0;   // per instance (doubles)
  int generation = -1;         // cache stamp (single-generation API); -1 = none
  std::vector<int> gen_host;   // per-instance stamp for the batched API
  bool cache_valid = false;
  bool admm_prebuilt = false;  // gsls_admm_build_cache ran: the next ADMM solve skips its first build
  void* sls = nullptr;         // SLS workspace (sls.cu), allocated on first use
  int sls_j0 = 0, sls_j1 = -1; // SLS disturbance-column shard [j0, j1) (-1: N), gsls_sls_set_columns
  // CVF plan variants for the LQR tree: [0] factored combines where C has low rank, [1] all
  // dense.  A factored combine that meets an indefinite P raises GSLS_ERR_LOWRANK; the
  // context then switches to the dense variant for good and the scan is re-run.
  const int4* cvf_ops_v[2] = {nullptr, nullptr};
  const int* cvf_leaf_v[2] = {nullptr, nullptr};
  bool lqr_dense = false;
};

// Matrix half of the CVF combine on an explicit slot space (lqr.cu); shared by
// the LQR factorization (with aux record) and the SLS grid scan (without).
struct CombineArgs {
  int n;
  const int4* ops;
  int op_base;                 // global op index of ops[0] (record offset)
  float *Ps, *As, *Cs, *ATs;
  long long inst_stride;       // floats between instances in Ps/As/Cs/ATs
  float* rec;                  // nullptr: no record
  long long rec_inst_stride;   // floats between instances in rec
  const int* list;
  ErrSlot* err;
  float rel_tol;
  int label;                   // GSLS_ERR_LOWRANK label: 0 LQR tree, 1 SLS tree
  const int* count = nullptr;  // device-side instance count (graph-captured loop), see DevLqr
};
int launch_combine(const CombineArgs& a, int nops, int count, cudaStream_t st);
int combine_threads(int n);
int matmul_threads(int n);
enum { PLAN_CVF = 0, PLAN_CVF_REC = 1, PLAN_OTHER = 2 };  // upload_plan dead-output analysis
int upload_plan(Ctx* c, const ScanPlan& p, const int4** ops, const int** out, const int** loff, int kind,
                const int** leaf_dead = nullptr, const std::vector<int>* leaf_rank = nullptr, int rmax = 0);
// Largest C-factor rank the factored combine carries for state dimension n in the
// LQR (tree 0) or SLS (tree 1) scan; 0: off.  GSLS_LOWRANK=0 / sls / lqr restricts it.
int factor_rmax(int n, int tree);
void sls_destroy(Ctx* c);

void* dev_alloc(Ctx* c, size_t bytes);
int build_cache(Ctx* c, const gsls_qp_t* qp, const double* d_rho, const int* d_list, int count,
                cudaStream_t st);
int check_errors(Ctx* c, cudaStream_t st, const char* what);
void sls_use_dense(Ctx* c);  // SLS tree: switch to the all-dense plan variant (sls.cu)

// replay-kernel launch (admm.cu)
struct ReplayArgs;
size_t replay_smem_floats(const Ctx* c);

}  // namespace gsls
