// U/V/W/X interaction lists, stored as CSR.
//
// Definitions followed (members always sorted by ascending raw key):
//  U(A), leaf A : every leaf adjacent to A, plus A.
//  V(B), level>=2: existing children of the same-level neighbours of parent(B)
//                 that are not adjacent to B.
//  W(A), leaf A : existing nodes whose parent is adjacent to A, that are strictly
//                 finer than A and not adjacent to A (SPEC.md:239-247 `post`).
//                 On a pruned tree such nodes can sit more than one level below
//                 A (an internal neighbour whose A-side children are empty), so
//                 the one-level restriction of SPEC.md:267 is not applied; see
//                 DESIGN.md "SPEC pins".
//  X(B), any node: { A : B in W(A) } -- the dual, defined on all nodes so that
//                 P2L can target non-leaf nodes.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <vector>

#include "common.hpp"
#include "parallel.hpp"
#include "tree.hpp"

namespace kifmm {

namespace {
struct TvTable {
  std::vector<std::array<int, 3>> vecs;
  int id[343];
  TvTable() {
    for (int i = 0; i < 343; ++i) id[i] = -1;
    for (int dx = -3; dx <= 3; ++dx)
      for (int dy = -3; dy <= 3; ++dy)
        for (int dz = -3; dz <= 3; ++dz) {
          const int m = std::max(std::abs(dx), std::max(std::abs(dy), std::abs(dz)));
          if (m < 2) continue;
          id[(dx + 3) * 49 + (dy + 3) * 7 + (dz + 3)] = int(vecs.size());
          vecs.push_back({dx, dy, dz});
        }
  }
};
const TvTable& tv_table() {
  static const TvTable t;
  return t;
}

// Packs per-node vectors into CSR.
template <class T>
void to_csr(const std::vector<std::vector<T>>& lists, std::vector<int64_t>& ptr, std::vector<T>& idx) {
  ptr.assign(lists.size() + 1, 0);
  for (size_t i = 0; i < lists.size(); ++i) ptr[i + 1] = ptr[i] + int64_t(lists[i].size());
  idx.resize(ptr.back());
  for (size_t i = 0; i < lists.size(); ++i) std::copy(lists[i].begin(), lists[i].end(), idx.begin() + ptr[i]);
}
}  // namespace

int transfer_vector_id(int dx, int dy, int dz) {
  if (dx < -3 || dx > 3 || dy < -3 || dy > 3 || dz < -3 || dz > 3) return -1;
  return tv_table().id[(dx + 3) * 49 + (dy + 3) * 7 + (dz + 3)];
}

const std::vector<std::array<int, 3>>& transfer_vector_table() { return tv_table().vecs; }

void build_lists(Tree& t, int threads) {
  threads = resolve_threads(threads);
  const int64_t nl = t.n_leaves(), nn = t.n_nodes();
  auto is_leaf = [&](int64_t node) { return t.node_leaf[node] >= 0; };

  // ---------------- U
  std::vector<std::vector<int64_t>> u(nl);
  parallel_for_dynamic(size_t(nl), threads, [&](size_t li) {
    const uint64_t a = t.leaves[li];
    std::vector<uint64_t> mem{a};
    uint64_t nb[26];
    const int cnt = key_neighbors(a, nb);
    std::vector<int64_t> stack;
    for (int j = 0; j < cnt; ++j) {
      const int64_t ni = t.node_map.find(nb[j]);
      if (ni >= 0) {
        if (is_leaf(ni)) {
          mem.push_back(nb[j]);
          continue;
        }
        stack.assign(1, ni);
        while (!stack.empty()) {
          const int64_t d = stack.back();
          stack.pop_back();
          for (int o = 0; o < 8; ++o) {
            const int64_t c = t.node_children[8 * d + o];
            if (c < 0 || !keys_adjacent(t.node_key[c], a)) continue;
            if (is_leaf(c))
              mem.push_back(t.node_key[c]);
            else
              stack.push_back(c);
          }
        }
      } else {
        // nearest existing ancestor: a coarser leaf covering the box, or an
        // internal node (then the box is empty space)
        for (int l = key_level(nb[j]) - 1; l >= 0; --l) {
          const int64_t ai = t.node_map.find(key_ancestor(nb[j], l));
          if (ai < 0) continue;
          if (is_leaf(ai)) mem.push_back(t.node_key[ai]);
          break;
        }
      }
    }
    std::sort(mem.begin(), mem.end());
    mem.erase(std::unique(mem.begin(), mem.end()), mem.end());
    auto& out = u[li];
    out.reserve(mem.size());
    for (uint64_t k : mem) out.push_back(t.node_leaf[t.node_map.find(k)]);
  });
  to_csr(u, t.u_ptr, t.u_idx);
  std::vector<std::vector<int64_t>>().swap(u);

  // ---------------- V
  std::vector<std::vector<int64_t>> v(nn);
  std::vector<std::vector<int32_t>> vt(nn);
  parallel_for_dynamic(size_t(nn), threads, [&](size_t bi) {
    const uint64_t b = t.node_key[bi];
    if (key_level(b) < 2) return;
    const auto ab = key_anchor(b);
    uint64_t nb[26];
    const int cnt = key_neighbors(key_parent(b), nb);
    std::vector<std::pair<uint64_t, int64_t>> mem;
    for (int j = 0; j < cnt; ++j) {
      const int64_t qi = t.node_map.find(nb[j]);
      if (qi < 0 || is_leaf(qi)) continue;
      for (int o = 0; o < 8; ++o) {
        const int64_t c = t.node_children[8 * qi + o];
        if (c < 0 || keys_adjacent(t.node_key[c], b)) continue;
        mem.push_back({t.node_key[c], c});
      }
    }
    std::sort(mem.begin(), mem.end());
    auto& out = v[bi];
    auto& tv = vt[bi];
    out.reserve(mem.size());
    tv.reserve(mem.size());
    for (auto& m : mem) {
      const auto as = key_anchor(m.first);
      const int id = transfer_vector_id(int(as[0]) - int(ab[0]), int(as[1]) - int(ab[1]),
                                        int(as[2]) - int(ab[2]));
      if (id < 0) throw InvalidArgument("v_list: transfer vector outside [-3,3]^3");
      out.push_back(m.second);
      tv.push_back(id);
    }
  });
  to_csr(v, t.v_ptr, t.v_idx);
  {
    std::vector<int64_t> dummy;
    to_csr(vt, dummy, t.v_tv);
  }
  std::vector<std::vector<int64_t>>().swap(v);
  std::vector<std::vector<int32_t>>().swap(vt);

  // ---------------- W
  std::vector<std::vector<int64_t>> w(nl);
  parallel_for_dynamic(size_t(nl), threads, [&](size_t li) {
    const uint64_t a = t.leaves[li];
    uint64_t nb[26];
    const int cnt = key_neighbors(a, nb);
    std::vector<std::pair<uint64_t, int64_t>> mem;
    std::vector<int64_t> stack;
    for (int j = 0; j < cnt; ++j) {
      const int64_t ni = t.node_map.find(nb[j]);
      if (ni < 0 || is_leaf(ni)) continue;
      stack.assign(1, ni);
      while (!stack.empty()) {
        const int64_t d = stack.back();
        stack.pop_back();
        for (int o = 0; o < 8; ++o) {
          const int64_t c = t.node_children[8 * d + o];
          if (c < 0) continue;
          if (keys_adjacent(t.node_key[c], a)) {
            if (!is_leaf(c)) stack.push_back(c);
          } else {
            mem.push_back({t.node_key[c], c});
          }
        }
      }
    }
    std::sort(mem.begin(), mem.end());
    auto& out = w[li];
    out.reserve(mem.size());
    for (auto& m : mem) out.push_back(m.second);
  });
  to_csr(w, t.w_ptr, t.w_idx);
  std::vector<std::vector<int64_t>>().swap(w);

  // ---------------- X = dual of W (on all nodes)
  t.x_ptr.assign(nn + 1, 0);
  for (int64_t li = 0; li < nl; ++li)
    for (int64_t e = t.w_ptr[li]; e < t.w_ptr[li + 1]; ++e) ++t.x_ptr[t.w_idx[e] + 1];
  for (int64_t i = 0; i < nn; ++i) t.x_ptr[i + 1] += t.x_ptr[i];
  t.x_idx.assign(t.x_ptr[nn], -1);
  {
    std::vector<int64_t> fill(t.x_ptr.begin(), t.x_ptr.end() - 1);
    // leaves ascend in raw key, so filling in leaf order keeps each X sorted
    for (int64_t li = 0; li < nl; ++li)
      for (int64_t e = t.w_ptr[li]; e < t.w_ptr[li + 1]; ++e) t.x_idx[fill[t.w_idx[e]]++] = li;
  }
}

}  // namespace kifmm
