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
#include <chrono>
#include <cstdio>
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
  const bool tt = std::getenv("KIFMM_TREE_TIMING") != nullptr;
  auto tt0 = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!tt) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "lists %-25s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tt0).count());
    tt0 = now;
  };
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

  tick("U");
  // ---------------- V: two passes straight into CSR (count, then fill).  Members come out in
  // ascending raw key without a sort: the parent's neighbours are visited in ascending key order and
  // the children of one parent in octant order, which is ascending key, and the children of a smaller
  // parent all precede those of a larger one.
  // node anchors decoded once; same-level adjacency is then max |anchor difference| <= 1
  std::vector<std::array<int32_t, 3>> anc(nn);
  parallel_for(size_t(nn), threads, [&](size_t i) {
    const auto a = key_anchor(t.node_key[i]);
    anc[i] = {int32_t(a[0]), int32_t(a[1]), int32_t(a[2])};
  });
  std::array<int16_t, 343> tv_of;  // (dx+3)*49 + (dy+3)*7 + (dz+3) -> transfer-vector id
  for (int i = 0; i < 343; ++i) tv_of[i] = int16_t(transfer_vector_id(i / 49 - 3, (i / 7) % 7 - 3, i % 7 - 3));
  // per parent: its colleagues (same-level neighbours that exist and are internal), sorted by key,
  // shared by its (up to 8) children
  auto colleagues = [&](int64_t pi, int64_t* out) {
    uint64_t nb[26];
    const int cnt = key_neighbors(t.node_key[pi], nb);
    std::sort(nb, nb + cnt);
    int m = 0;
    for (int j = 0; j < cnt; ++j) {
      const int64_t qi = t.node_map.find(nb[j]);
      if (qi >= 0 && !is_leaf(qi)) out[m++] = qi;
    }
    return m;
  };
  auto v_child = [&](int64_t bi, const int64_t* col, int m, auto&& emit) {
    const auto& ab = anc[bi];
    for (int j = 0; j < m; ++j)
      for (int o = 0; o < 8; ++o) {
        const int64_t c = t.node_children[8 * col[j] + o];
        if (c < 0) continue;
        const int dx = anc[c][0] - ab[0], dy = anc[c][1] - ab[1], dz = anc[c][2] - ab[2];
        if (std::abs(dx) <= 1 && std::abs(dy) <= 1 && std::abs(dz) <= 1) continue;  // adjacent (same level)
        emit(c, (dx + 3) * 49 + (dy + 3) * 7 + (dz + 3));
      }
  };
  t.v_ptr.assign(nn + 1, 0);
  parallel_for_dynamic(size_t(nn), threads, [&](size_t pi) {
    if (is_leaf(int64_t(pi)) || key_level(t.node_key[pi]) < 1) return;  // parents of level >= 2 nodes
    int64_t col[26];
    const int m = colleagues(int64_t(pi), col);
    for (int o = 0; o < 8; ++o) {
      const int64_t bi = t.node_children[8 * pi + o];
      if (bi < 0) continue;
      int64_t k = 0;
      v_child(bi, col, m, [&](int64_t, int) { ++k; });
      t.v_ptr[bi + 1] = k;
    }
  });
  for (int64_t i = 0; i < nn; ++i) t.v_ptr[i + 1] += t.v_ptr[i];
  t.v_idx.resize(t.v_ptr[nn]);
  t.v_tv.resize(t.v_ptr[nn]);
  parallel_for_dynamic(size_t(nn), threads, [&](size_t pi) {
    if (is_leaf(int64_t(pi)) || key_level(t.node_key[pi]) < 1) return;
    int64_t col[26];
    const int m = colleagues(int64_t(pi), col);
    for (int o = 0; o < 8; ++o) {
      const int64_t bi = t.node_children[8 * pi + o];
      if (bi < 0) continue;
      int64_t e = t.v_ptr[bi];
      v_child(bi, col, m, [&](int64_t c, int code) {
        const int id = tv_of[code];
        if (id < 0) throw InvalidArgument("v_list: transfer vector outside [-3,3]^3");
        t.v_idx[e] = c;
        t.v_tv[e] = id;
        ++e;
      });
    }
  });

  tick("V");
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

  tick("W");
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
  tick("X");
}

}  // namespace kifmm
