// Adaptive n_crit octree build + 2:1 balance.
#include "tree.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <memory>
#include <omp.h>
#include <parallel/algorithm>
#include <string>

#include "common.hpp"
#include "parallel.hpp"

namespace kifmm {

uint32_t fine_cell(double x, double origin, double side) {
  const double v = (x - origin) * (double(kFineCells) / side);
  if (!(v >= 0.0) || v > double(kFineCells))
    throw InvalidArgument("point outside domain: coordinate " + std::to_string(x));
  int64_t c = static_cast<int64_t>(std::floor(v));
  if (c >= int64_t(kFineCells)) c = kFineCells - 1;  // closed upper face
  return static_cast<uint32_t>(c);
}

namespace {

struct Range {
  int64_t s, e;
};

// Particle range of `key` within the sorted fine codes.
Range key_range(const std::vector<uint64_t>& codes, uint64_t key) {
  const int l = key_level(key);
  const uint64_t lo = key_code(key);
  const uint64_t hi = lo + (uint64_t(1) << (3 * (kMaxLevel - l)));
  const auto b = std::lower_bound(codes.begin(), codes.end(), lo);
  const auto e = std::lower_bound(b, codes.end(), hi);
  return {int64_t(b - codes.begin()), int64_t(e - codes.begin())};
}

Range sub_range(const std::vector<uint64_t>& codes, Range r, uint64_t key) {
  const int l = key_level(key);
  const uint64_t lo = key_code(key);
  const uint64_t hi = lo + (uint64_t(1) << (3 * (kMaxLevel - l)));
  const auto base = codes.begin();
  const auto b = std::lower_bound(base + r.s, base + r.e, lo);
  const auto e = std::lower_bound(b, base + r.e, hi);
  return {int64_t(b - base), int64_t(e - base)};
}

}  // namespace

void build_tree(Tree& t, const double* pos, int64_t n, int n_crit, const double* domain,
                bool balance, int threads) {
  if (n < 1) throw InvalidArgument("build_tree: N must be >= 1");
  if (n_crit < 1) throw InvalidArgument("build_tree: n_crit must be >= 1");
  if (!pos) throw InvalidArgument("build_tree: null positions");
  threads = resolve_threads(threads);
  t = Tree{};
  t.n = n;
  // phase timing (KIFMM_TREE_TIMING=1)
  const bool tt = std::getenv("KIFMM_TREE_TIMING") != nullptr;
  auto tt0 = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!tt) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "tree %-26s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tt0).count());
    tt0 = now;
  };

  // ---- domain: tight bounding cube, 1e-10 relative margin per side
  if (domain) {
    if (!(domain[3] > 0.0)) throw InvalidArgument("domain side must be > 0");
    for (int d = 0; d < 3; ++d) t.origin[d] = domain[d];
    t.side = domain[3];
  } else {
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::numeric_limits<double>::infinity();
      hi[d] = -std::numeric_limits<double>::infinity();
    }
    for (int64_t i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) {
        const double v = pos[3 * i + d];
        if (!std::isfinite(v)) throw InvalidArgument("non-finite particle coordinate");
        lo[d] = std::min(lo[d], v);
        hi[d] = std::max(hi[d], v);
      }
    double ext = 0.0;
    for (int d = 0; d < 3; ++d) ext = std::max(ext, hi[d] - lo[d]);
    if (ext <= 0.0) ext = 1.0;
    const double side = ext * (1.0 + 2e-10);
    for (int d = 0; d < 3; ++d) t.origin[d] = 0.5 * (lo[d] + hi[d]) - 0.5 * side;
    t.side = side;
  }

  tick("domain");
  // ---- fine codes and the Morton permutation
  // (code, index) pairs without value-initialisation (first touched by the parallel loop below)
  using CI = std::pair<uint64_t, int64_t>;
  std::unique_ptr<CI[]> ci(new CI[size_t(n)]);
  std::atomic<bool> bad{false};
  std::string bad_msg;
  parallel_for(size_t(n), threads, [&](size_t i) {
    try {
      const uint32_t cx = fine_cell(pos[3 * i + 0], t.origin[0], t.side);
      const uint32_t cy = fine_cell(pos[3 * i + 1], t.origin[1], t.side);
      const uint32_t cz = fine_cell(pos[3 * i + 2], t.origin[2], t.side);
      ci[i] = {fine_code(cx, cy, cz), int64_t(i)};
    } catch (const InvalidArgument& e) {
      if (!bad.exchange(true)) bad_msg = e.what();
    }
  });
  if (bad) throw InvalidArgument(bad_msg);
  tick("fine codes");
  if (threads > 1 && n > 100000) {
    // parallel bucket sort: 4096 buckets on the top 12 bits of the 45-bit fine code (counting pass,
    // scatter, then each bucket sorted independently); equal to a full sort of the (code, index) pairs
    constexpr int kB = 4096, kShift = 45 - 12;
    std::vector<int64_t> cnt(size_t(threads) * kB, 0);
    const int64_t per = (n + threads - 1) / threads;
#pragma omp parallel num_threads(threads)
    {
      const int th = omp_get_thread_num();
      const int64_t a = std::min<int64_t>(n, th * per), b = std::min<int64_t>(n, a + per);
      int64_t* c = cnt.data() + size_t(th) * kB;
      for (int64_t i = a; i < b; ++i) ++c[ci[i].first >> kShift];
    }
    std::vector<int64_t> start(kB + 1, 0);
    {
      int64_t acc = 0;
      for (int k = 0; k < kB; ++k) {
        start[k] = acc;
        for (int th = 0; th < threads; ++th) {
          const int64_t v = cnt[size_t(th) * kB + k];
          cnt[size_t(th) * kB + k] = acc;  // becomes this thread's write cursor in bucket k
          acc += v;
        }
      }
      start[kB] = acc;
    }
    std::unique_ptr<CI[]> tmp(new CI[size_t(n)]);
#pragma omp parallel num_threads(threads)
    {
      const int th = omp_get_thread_num();
      const int64_t a = std::min<int64_t>(n, th * per), b = std::min<int64_t>(n, a + per);
      int64_t* c = cnt.data() + size_t(th) * kB;
      for (int64_t i = a; i < b; ++i) tmp[c[ci[i].first >> kShift]++] = ci[i];
    }
#pragma omp parallel for schedule(dynamic, 8) num_threads(threads)
    for (int k = 0; k < kB; ++k) std::sort(tmp.get() + start[k], tmp.get() + start[k + 1]);
    ci.swap(tmp);
  } else {
    std::sort(ci.get(), ci.get() + n);
  }
  tick("sort");
  t.codes.resize(n);
  t.original_index.resize(n);
  t.positions.resize(3 * n);
  parallel_for(size_t(n), threads, [&](size_t i) {
    t.codes[i] = ci[i].first;
    t.original_index[i] = ci[i].second;
    for (int d = 0; d < 3; ++d) t.positions[3 * i + d] = pos[3 * ci[i].second + d];
  });
  ci.reset();

  tick("codes+sort+permute");
  // ---- unbalanced adaptive leaves: depth-first in octant order => ascending raw
  struct Item {
    uint64_t key;
    Range r;
  };
  std::vector<Item> stack;
  stack.push_back({make_key(0, 0, 0, 0), {0, n}});
  std::vector<uint64_t> leaves;
  while (!stack.empty()) {
    const Item it = stack.back();
    stack.pop_back();
    const int l = key_level(it.key);
    if (it.r.e - it.r.s <= n_crit || l == kMaxLevel) {
      leaves.push_back(it.key);
      continue;
    }
    for (int o = 7; o >= 0; --o) {
      const uint64_t ck = key_child(it.key, o);
      const Range cr = sub_range(t.codes, it.r, ck);
      if (cr.e > cr.s) stack.push_back({ck, cr});
    }
  }

  tick("adaptive split");
  // ---- 2:1 balance (design 190): split every leaf that has an
  // adjacent leaf more than one level finer, until a fixed point.  A coarser leaf
  // K adjacent to leaf A always covers one of A's 26 same-level neighbour boxes,
  // so it is found as the nearest existing ancestor of that box.
  while (balance) {
    KeyMap leafset(leaves.size());
    for (size_t i = 0; i < leaves.size(); ++i) leafset.insert(leaves[i], int64_t(i));
    KeyMap internal(leaves.size() * 2);
    for (uint64_t k : leaves)
      for (int l = key_level(k) - 1; l >= 0; --l) {
        const uint64_t a = key_ancestor(k, l);
        if (internal.contains(a)) break;
        internal.insert(a, 1);
      }
    std::vector<char> mark(leaves.size(), 0);
    parallel_for(leaves.size(), threads, [&](size_t i) {
      const uint64_t a = leaves[i];
      const int la = key_level(a);
      if (la < 2) return;
      uint64_t nb[26];
      const int cnt = key_neighbors(a, nb);
      for (int j = 0; j < cnt; ++j) {
        for (int l = la; l >= 0; --l) {
          const uint64_t k = key_ancestor(nb[j], l);
          const int64_t li = leafset.find(k);
          if (li >= 0) {
            if (l < la - 1) mark[li] = 1;
            break;
          }
          if (internal.contains(k)) break;
        }
      }
    });
    bool any = false;
    for (char m : mark) any |= (m != 0);
    if (!any) break;
    std::vector<uint64_t> next;
    next.reserve(leaves.size() + 64);
    for (size_t i = 0; i < leaves.size(); ++i) {
      if (!mark[i]) {
        next.push_back(leaves[i]);
        continue;
      }
      if (key_level(leaves[i]) >= kMaxLevel) throw InvalidArgument("balance: refinement past MAX_LEVEL");
      const Range r = key_range(t.codes, leaves[i]);
      for (int o = 0; o < 8; ++o) {
        const uint64_t ck = key_child(leaves[i], o);
        const Range cr = sub_range(t.codes, r, ck);
        if (cr.e > cr.s) next.push_back(ck);
      }
    }
    leaves.swap(next);
  }

  tick("balance");
  // ---- leaf particle ranges
  t.leaves = leaves;
  const int64_t nl = int64_t(leaves.size());
  t.leaf_ptr.assign(nl + 1, 0);
  parallel_for(size_t(nl), threads, [&](size_t i) {
    const Range r = key_range(t.codes, leaves[i]);
    t.leaf_ptr[i] = r.s;
    if (i + 1 == size_t(nl)) t.leaf_ptr[nl] = r.e;
  });
  for (int64_t i = 0; i < nl; ++i) {
    const int l = key_level(leaves[i]);
    const int64_t cnt = (i + 1 < nl ? t.leaf_ptr[i + 1] : t.leaf_ptr[nl]) - t.leaf_ptr[i];
    if (l == kMaxLevel && cnt > n_crit) ++t.n_overfull;
  }

  tick("leaf ranges");
  // ---- nodes: leaves and all their ancestors, level-major
  int depth = 0;
  for (uint64_t k : leaves) depth = std::max(depth, key_level(k));
  t.depth = depth;
  std::vector<std::vector<uint64_t>> per_level(depth + 1);
  {
    KeyMap seen(leaves.size() * 2);
    for (uint64_t k : leaves) {
      for (int l = key_level(k); l >= 0; --l) {
        const uint64_t a = key_ancestor(k, l);
        if (seen.contains(a)) break;
        seen.insert(a, 1);
        per_level[l].push_back(a);
      }
    }
  }
  t.level_ptr.assign(depth + 2, 0);
  for (int l = 0; l <= depth; ++l) {
    std::sort(per_level[l].begin(), per_level[l].end());
    t.level_ptr[l + 1] = t.level_ptr[l] + int64_t(per_level[l].size());
  }
  const int64_t nn = t.level_ptr[depth + 1];
  t.node_key.resize(nn);
  for (int l = 0; l <= depth; ++l)
    std::copy(per_level[l].begin(), per_level[l].end(), t.node_key.begin() + t.level_ptr[l]);
  t.node_map.reserve(size_t(nn));
  for (int64_t i = 0; i < nn; ++i) t.node_map.insert(t.node_key[i], i);

  t.node_parent.assign(nn, -1);
  t.node_children.assign(nn * 8, -1);
  t.node_leaf.assign(nn, -1);
  t.leaf_node.assign(nl, -1);
  parallel_for(size_t(nn), threads, [&](size_t i) {
    const uint64_t k = t.node_key[i];
    if (key_level(k) > 0) t.node_parent[i] = t.node_map.find(key_parent(k));
    if (key_level(k) < kMaxLevel)
      for (int o = 0; o < 8; ++o) t.node_children[8 * i + o] = t.node_map.find(key_child(k, o));
  });
  for (int64_t i = 0; i < nl; ++i) {
    const int64_t ni = t.node_map.find(leaves[i]);
    t.leaf_node[i] = ni;
    t.node_leaf[ni] = i;
  }
  tick("nodes");
}

}  // namespace kifmm
