// Host-side scan schedule: the reference's balanced combine tree, flattened.
//
// A scan over `length` elements (scan.py:141-234) is turned into layers of
// independent combine ops (dst, earlier, later) on value slots.  Slots
// [0, length) are the leaves in time order; every real combine writes a new
// slot, so no value is ever overwritten (the replay of recorded aux reads the
// same slots, lqr.py:419-454).  Identity operands — the power-of-two padding
// (scan.py:175-177) and SLS neutral elements (sls.py:269-273) — are resolved
// symbolically: combining with an identity is exact in the reference, so the
// op is elided and the other operand's slot is aliased.  "earlier"/"later"
// are in time order, i.e. the reference's inner(left, right) operands after
// its reverse-scan operand swap (scan.py:169-173).
#pragma once

#include <algorithm>
#include <vector>

namespace gsls {

struct ScanOp {
  int dst, earlier, later;
};

struct ScanPlan {
  int length = 0;
  int nslots = 0;               // leaves + combine results
  int layers = 0;               // == scan_depth(length), counting elided/skipped layers
  std::vector<int> layer_off;   // size layers+1, offsets into ops
  std::vector<ScanOp> ops;
  std::vector<int> out;         // output slot per time position (-1: identity)
};

inline int next_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

inline int scan_depth(int length) {
  int p = next_pow2(length), d = 0;
  while (p > 1) { p >>= 1; ++d; }
  return 2 * d;
}

// neutral: optional per-time-position flag (true = identity element).
inline ScanPlan make_scan_plan(int length, bool reverse, const std::vector<char>& neutral = {},
                               int first_slot = 0) {
  ScanPlan pl;
  pl.length = length;
  const int width = next_pow2(length);
  int next_slot = first_slot + length;
  // tree index t <-> time position
  auto time_of = [&](int t) { return reverse ? length - 1 - t : t; };
  std::vector<int> leaf(width, -1);
  for (int t = 0; t < length; ++t) {
    int pos = time_of(t);
    bool id = !neutral.empty() && neutral[pos];
    leaf[t] = id ? -1 : first_slot + pos;
  }
  std::vector<std::vector<int>> lay;  // per layer ops appended to pl.ops
  std::vector<ScanOp> cur_ops;
  auto combine = [&](int tl, int tr) -> int {
    // tree-order operands -> time order
    int e = reverse ? tr : tl;
    int l = reverse ? tl : tr;
    if (e < 0) return l;
    if (l < 0) return e;
    int d = next_slot++;
    cur_ops.push_back({d, e, l});
    return d;
  };
  auto flush_layer = [&]() {
    pl.layer_off.push_back((int)pl.ops.size());
    for (auto& o : cur_ops) pl.ops.push_back(o);
    cur_ops.clear();
    pl.layers++;
  };
  pl.layer_off.clear();
  std::vector<std::vector<int>> levels;
  levels.push_back(leaf);
  while (levels.back().size() > 1) {
    const auto& c = levels.back();
    std::vector<int> nxt(c.size() / 2);
    for (size_t i = 0; i < nxt.size(); ++i) nxt[i] = combine(c[2 * i], c[2 * i + 1]);
    flush_layer();
    levels.push_back(nxt);
  }
  std::vector<int> acc = levels.back();
  for (int lv = (int)levels.size() - 2; lv >= 0; --lv) {
    const auto& lvl = levels[lv];
    const int w = (int)acc.size();
    std::vector<int> head(w);
    head[0] = lvl[0];
    for (int i = 1; i < w; ++i) head[i] = combine(acc[i - 1], lvl[2 * i]);
    flush_layer();
    std::vector<int> merged(2 * w);
    for (int i = 0; i < w; ++i) {
      merged[2 * i] = head[i];
      merged[2 * i + 1] = acc[i];
    }
    acc.swap(merged);
  }
  pl.layer_off.push_back((int)pl.ops.size());
  pl.out.assign(length, -1);
  for (int t = 0; t < length; ++t) pl.out[time_of(t)] = acc[t];
  pl.nslots = next_slot - first_slot;
  return pl;
}

// Within every layer, moves the ops whose result no later op reads (the scan's
// final outputs, read only through out[]) behind the others, keeping both groups in
// order; ops of one layer are independent, so the values are unchanged.  Returns the
// per-layer count of ops whose result is read again.  The CVF replay uses it: of a
// combine's affine outputs (p, b), b is read only by later combines, so the
// unread ops skip their b half ([Psi -Y], half the op's replay operator bytes).
inline std::vector<int> partition_unread_last(ScanPlan& p) {
  std::vector<char> rd(std::max(p.nslots, 1), 0);
  for (const ScanOp& q : p.ops) {
    if (q.earlier >= 0) rd[q.earlier] = 1;
    if (q.later >= 0) rd[q.later] = 1;
  }
  std::vector<int> live(p.layers, 0);
  for (int l = 0; l < p.layers; ++l) {
    auto b = p.ops.begin() + p.layer_off[l], e = p.ops.begin() + p.layer_off[l + 1];
    auto mid = std::stable_partition(b, e, [&](const ScanOp& q) { return rd[q.dst] != 0; });
    live[l] = (int)(mid - b);
  }
  return live;
}

// Physical slots for the replay vectors: interval colouring of slot lifetimes.
// Leaves are defined at time 0; the ops of layer l read their operands and
// define their result at time l + 1 (a result may not share storage with
// anything read in the same layer); output slots stay live to the end.
// Returns the number of physical slots; phys[s] is the storage of slot s.
inline int compress_slots(const ScanPlan& p, std::vector<int>& phys) {
  const int S = p.nslots;
  const int INF = 1 << 30;
  std::vector<int> def(S, 0), last(S, 0);
  for (int l = 0; l < p.layers; ++l)
    for (int o = p.layer_off[l]; o < p.layer_off[l + 1]; ++o) {
      const ScanOp& op = p.ops[o];
      def[op.dst] = l + 1;
      last[op.dst] = std::max(last[op.dst], l + 1);
      last[op.earlier] = std::max(last[op.earlier], l + 1);
      last[op.later] = std::max(last[op.later], l + 1);
    }
  for (int t : p.out)
    if (t >= 0) last[t] = INF;
  std::vector<int> order(S);
  for (int i = 0; i < S; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return def[a] < def[b]; });
  phys.assign(S, -1);
  std::vector<int> owner;  // phys id -> slot currently holding it (-1 free)
  for (int s : order) {
    int pick = -1;
    for (int q = 0; q < (int)owner.size(); ++q) {
      const int o = owner[q];
      if (o < 0 || last[o] < def[s]) { pick = q; break; }
    }
    if (pick < 0) { pick = (int)owner.size(); owner.push_back(-1); }
    owner[pick] = s;
    phys[s] = pick;
  }
  return (int)owner.size();
}

}  // namespace gsls
