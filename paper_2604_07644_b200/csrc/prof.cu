#include <mutex>
#include <vector>

#include "../../include/gsls.h"
#include "prof.h"

namespace gsls {

namespace {
struct Pending {
  int id;
  cudaEvent_t a, b;
  double units;
};
std::mutex mu;
bool enabled = false;
std::vector<cudaEvent_t> pool;
std::vector<Pending> pending;
cudaEvent_t open_ev[P_COUNT];
double acc_ms[P_COUNT], acc_units[P_COUNT];
long long acc_n[P_COUNT];

cudaEvent_t take() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void prof_begin(int id, cudaStream_t st) {
  std::lock_guard<std::mutex> g(mu);
  if (!enabled) return;
  open_ev[id] = take();
  cudaEventRecord(open_ev[id], st);
}

void prof_end(int id, cudaStream_t st, double units) {
  std::lock_guard<std::mutex> g(mu);
  if (!enabled || !open_ev[id]) return;
  cudaEvent_t b = take();
  cudaEventRecord(b, st);
  pending.push_back({id, open_ev[id], b, units});
  open_ev[id] = nullptr;
}

}  // namespace gsls

using namespace gsls;

extern "C" {

int gsls_prof_enable(int32_t on) {
  std::lock_guard<std::mutex> g(mu);
  enabled = on != 0;
  return GSLS_OK;
}

int gsls_prof_read(double* ms, double* units, int64_t* launches, int32_t max_ids) {
  std::lock_guard<std::mutex> g(mu);
  for (auto& p : pending) {
    cudaEventSynchronize(p.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, p.a, p.b);
    acc_ms[p.id] += t;
    acc_units[p.id] += p.units;
    acc_n[p.id] += 1;
    pool.push_back(p.a);
    pool.push_back(p.b);
  }
  pending.clear();
  const int n = max_ids < P_COUNT ? max_ids : P_COUNT;
  for (int i = 0; i < n; ++i) {
    if (ms) ms[i] = acc_ms[i];
    if (units) units[i] = acc_units[i];
    if (launches) launches[i] = acc_n[i];
    acc_ms[i] = acc_units[i] = 0.0;
    acc_n[i] = 0;
  }
  return P_COUNT;
}

}  // extern "C"
