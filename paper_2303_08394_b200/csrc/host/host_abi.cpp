// extern "C" entry points of the host modules (include/kifmm.h).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "common.hpp"
#include "morton.hpp"
#include "operators.hpp"
#include "parallel.hpp"
#include "tree.hpp"

struct kifmm_tree {
  kifmm::Tree t;
};
struct kifmm_operators {
  kifmm::Operators o;
};

namespace kifmm {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
void clear_last_error() { g_last_error.clear(); }
}  // namespace kifmm

using namespace kifmm;

extern "C" {

const char* kifmm_last_error(void) { return g_last_error.c_str(); }
const char* kifmm_version(void) { return "kifmm_b200 0.1.0 (sm_100a)"; }

// ------------------------------------------------------------------ morton
kifmm_status kifmm_morton_encode(const uint32_t anchor[3], int32_t level, uint64_t* out) {
  return guard([&] {
    if (level < 0 || level > kMaxLevel) throw InvalidArgument("encode: level out of range");
    for (int d = 0; d < 3; ++d)
      if (anchor[d] >= (1u << level)) throw InvalidArgument("encode: anchor out of range");
    *out = make_key(anchor[0], anchor[1], anchor[2], level);
  });
}

kifmm_status kifmm_morton_decode(uint64_t key, uint32_t anchor[3], int32_t* level) {
  return guard([&] {
    const int l = key_level(key);
    const uint64_t code = key_code(key);
    if (code >> (3 * kMaxLevel)) throw InvalidArgument("decode: bits above the anchor field set");
    if (code & ((uint64_t(1) << (3 * (kMaxLevel - l))) - 1))
      throw InvalidArgument("decode: anchor bits below the level set");
    const auto a = key_anchor(key);
    for (int d = 0; d < 3; ++d) anchor[d] = a[d];
    *level = l;
  });
}

kifmm_status kifmm_morton_parent(uint64_t key, uint64_t* out) {
  return guard([&] {
    if (key_level(key) < 1) throw InvalidArgument("parent: root has no parent");
    *out = key_parent(key);
  });
}

kifmm_status kifmm_morton_children(uint64_t key, uint64_t out[8]) {
  return guard([&] {
    if (key_level(key) >= kMaxLevel) throw InvalidArgument("children: level 15 node");
    for (int o = 0; o < 8; ++o) out[o] = key_child(key, o);
  });
}

int32_t kifmm_morton_neighbors(uint64_t key, uint64_t out[26]) { return key_neighbors(key, out); }

int32_t kifmm_morton_is_adjacent(uint64_t a, uint64_t b) { return keys_adjacent(a, b) ? 1 : 0; }

void kifmm_morton_node_bounds(uint64_t key, const double origin[3], double side, double center[3],
                              double* half_side) {
  const int l = key_level(key);
  const auto a = key_anchor(key);
  const double w = side / double(uint64_t(1) << l);
  for (int d = 0; d < 3; ++d) center[d] = origin[d] + (double(a[d]) + 0.5) * w;
  *half_side = side / double(uint64_t(1) << (l + 1));
}

// ------------------------------------------------------------------ kernel
double kifmm_laplace(const double x[3], const double y[3]) {
  return laplace(x[0], x[1], x[2], y[0], y[1], y[2]);
}

void kifmm_kernel_matrix(const double* sources, int64_t m, const double* targets, int64_t k, double* out) {
  kernel_matrix(sources, m, targets, k, out);
}

// ----------------------------------------------------------------- surface
int32_t kifmm_surface_count(int32_t p) { return surface_count(p); }

kifmm_status kifmm_surface_grid(int32_t p, double* out) {
  return guard([&] {
    const auto g = surface_grid(p);
    std::memcpy(out, g.data(), g.size() * sizeof(double));
  });
}

// -------------------------------------------------------------------- tree
kifmm_status kifmm_tree_build(const double* positions, int64_t n, int32_t n_crit, const double* domain,
                              int32_t balance, int32_t threads, kifmm_tree** out) {
  return guard([&] {
    if (!out) throw InvalidArgument("tree_build: null out");
    auto t = std::make_unique<kifmm_tree>();
    build_tree(t->t, positions, n, n_crit, domain, balance != 0, threads);
    build_lists(t->t, threads);
    *out = t.release();
  });
}

kifmm_status kifmm_tree_get_view(const kifmm_tree* tree, kifmm_tree_view* v) {
  return guard([&] {
    if (!tree || !v) throw InvalidArgument("tree_get_view: null argument");
    const Tree& t = tree->t;
    std::memset(v, 0, sizeof(*v));
    v->n_particles = t.n;
    v->depth = t.depth;
    v->n_overfull = t.n_overfull;
    v->n_leaves = t.n_leaves();
    v->n_nodes = t.n_nodes();
    for (int d = 0; d < 3; ++d) v->origin[d] = t.origin[d];
    v->side = t.side;
    v->positions = t.positions.data();
    v->original_index = t.original_index.data();
    v->node_key = t.node_key.data();
    v->level_ptr = t.level_ptr.data();
    v->node_parent = t.node_parent.data();
    v->node_children = t.node_children.data();
    v->node_leaf = t.node_leaf.data();
    v->leaf_node = t.leaf_node.data();
    v->leaf_ptr = t.leaf_ptr.data();
    v->u_ptr = t.u_ptr.data();
    v->u_idx = t.u_idx.data();
    v->v_ptr = t.v_ptr.data();
    v->v_idx = t.v_idx.data();
    v->v_tv = t.v_tv.data();
    v->w_ptr = t.w_ptr.data();
    v->w_idx = t.w_idx.data();
    v->x_ptr = t.x_ptr.data();
    v->x_idx = t.x_idx.data();
  });
}

void kifmm_tree_destroy(kifmm_tree* tree) { delete tree; }

int32_t kifmm_transfer_vectors(int32_t out[316 * 3]) {
  const auto& tab = transfer_vector_table();
  for (size_t i = 0; i < tab.size(); ++i)
    for (int d = 0; d < 3; ++d) out[3 * i + d] = tab[i][d];
  return int32_t(tab.size());
}

// Contiguous Z-order leaf ranges, cost-balanced, aligned to level-`cut` boxes.
namespace {
// estimated evaluate cost of every leaf: P2P pairs (near + L2P / M2P surfaces) x flops + its M2L
std::vector<double> leaf_costs(const kifmm_tree_view* tv, int n_e, bool gradient) {
  const int64_t nl = tv->n_leaves;
  const double pair_flops = gradient ? 19.0 : 11.0;
  std::vector<double> cost(nl, 0.0);
  for (int64_t l = 0; l < nl; ++l) {
    const int64_t nt = tv->leaf_ptr[l + 1] - tv->leaf_ptr[l];
    int64_t src = 0;
    for (int64_t e = tv->u_ptr[l]; e < tv->u_ptr[l + 1]; ++e) {
      const int64_t s = tv->u_idx[e];
      src += tv->leaf_ptr[s + 1] - tv->leaf_ptr[s];
    }
    src += n_e * (1 + (tv->w_ptr[l + 1] - tv->w_ptr[l]));
    const int64_t node = tv->leaf_node[l];
    const int64_t nv = tv->v_ptr[node + 1] - tv->v_ptr[node];
    cost[l] = pair_flops * double(nt) * double(src) + 2.0 * n_e * n_e * double(nv) + 11.0 * nt * n_e;
  }
  return cost;
}
// ranges for one cut level; returns the largest rank cost over the mean
double split_at_cut(const kifmm_tree_view* tv, const std::vector<double>& cost, int world, int cut,
                    int64_t* leaf_begin) {
  const int64_t nl = tv->n_leaves;
  // groups = runs of leaves sharing the level-`cut` ancestor (coarser leaves are their own group)
  std::vector<int64_t> gstart;
  uint64_t prev = ~uint64_t(0);
  for (int64_t l = 0; l < nl; ++l) {
    const uint64_t k = tv->node_key[tv->leaf_node[l]];
    const uint64_t g = key_level(k) >= cut ? key_ancestor(k, cut) : k;
    if (g != prev) gstart.push_back(l);
    prev = g;
  }
  gstart.push_back(nl);
  const int64_t ng = int64_t(gstart.size()) - 1;
  std::vector<double> prefix(ng + 1, 0.0);
  for (int64_t g = 0; g < ng; ++g) {
    double gc = 0;
    for (int64_t l = gstart[g]; l < gstart[g + 1]; ++l) gc += cost[l];
    prefix[g + 1] = prefix[g] + gc;
  }
  const double total = prefix[ng];
  leaf_begin[0] = 0;
  int64_t b = 0;
  std::vector<int64_t> gb(world + 1, 0);
  for (int r = 1; r < world; ++r) {
    const double target = total * double(r) / double(world);
    while (b < ng && std::abs(prefix[b + 1] - target) <= std::abs(prefix[b] - target)) ++b;
    gb[r] = b;
    leaf_begin[r] = gstart[b];
  }
  gb[world] = ng;
  leaf_begin[world] = nl;
  double worst = 0;
  for (int r = 0; r < world; ++r) worst = std::max(worst, prefix[gb[r + 1]] - prefix[gb[r]]);
  return total > 0 ? worst / (total / world) : 1.0;
}
}  // namespace

kifmm_status kifmm_partition_leaves(const kifmm_tree_view* tv, int32_t n_e, int32_t gradient,
                                    int32_t world_size, int32_t cut_level, int64_t* leaf_begin) {
  return guard([&] {
    if (!tv || !leaf_begin || world_size < 1 || n_e < 1 || cut_level < 0)
      throw InvalidArgument("partition: bad argument");
    const std::vector<double> cost = leaf_costs(tv, n_e, gradient != 0);
    if (cut_level > 0) {
      split_at_cut(tv, cost, world_size, cut_level, leaf_begin);
      return;
    }
    // auto: the coarsest cut level >= 2 whose ranges are within 5 % of the mean cost (clustered clouds
    // put most leaves under few level-2 boxes), else the best balanced one
    std::vector<int64_t> best(world_size + 1), cur(world_size + 1);
    double best_imb = 1e300;
    for (int cut = 2; cut <= std::max(2, tv->depth); ++cut) {
      const double imb = split_at_cut(tv, cost, world_size, cut, cur.data());
      if (imb < best_imb - 1e-12) {
        best_imb = imb;
        best = cur;
      }
      if (imb <= 1.05) break;
    }
    std::copy(best.begin(), best.end(), leaf_begin);
  });
}

// --------------------------------------------------------------- operators
kifmm_status kifmm_precompute(int32_t p, double alpha_inner, double alpha_outer, double svd_cutoff,
                              double domain_side, int32_t threads, kifmm_operators** out) {
  return guard([&] {
    if (!out) throw InvalidArgument("precompute: null out");
    auto o = std::make_unique<kifmm_operators>();
    precompute(o->o, p, alpha_inner, alpha_outer, svd_cutoff, domain_side, threads);
    *out = o.release();
  });
}

kifmm_status kifmm_operators_get_view(const kifmm_operators* ops, kifmm_operator_view* v) {
  return guard([&] {
    if (!ops || !v) throw InvalidArgument("operators_get_view: null argument");
    const Operators& o = ops->o;
    std::memset(v, 0, sizeof(*v));
    v->p = o.p;
    v->n_e = o.n_e;
    v->n_c = o.n_c;
    v->reference_level = o.reference_level;
    v->alpha_inner = o.alpha_inner;
    v->alpha_outer = o.alpha_outer;
    v->svd_cutoff = o.svd_cutoff;
    v->domain_side = o.domain_side;
    v->ref_half_side = o.ref_half_side;
    v->surface = o.surface.data();
    v->uc2e_rank = o.uc2e_rank;
    v->uc2e_u = o.uc2e_u.data();
    v->uc2e_s = o.uc2e_s.data();
    v->uc2e_v = o.uc2e_v.data();
    v->dc2e_rank = o.dc2e_rank;
    v->dc2e_u = o.dc2e_u.data();
    v->dc2e_s = o.dc2e_s.data();
    v->dc2e_v = o.dc2e_v.data();
    v->m2m = o.m2m.data();
    v->l2l = o.l2l.data();
    v->n_m2l = int32_t(o.m2l.size() / (size_t(o.n_c) * o.n_e));
    v->m2l = o.m2l.data();
    v->fingerprint = o.fingerprint;
  });
}

void kifmm_operators_destroy(kifmm_operators* ops) { delete ops; }

kifmm_status kifmm_operators_save(const kifmm_operators* ops, const char* path) {
  return guard([&] {
    if (!ops || !path) throw InvalidArgument("save: null argument");
    save_operators(ops->o, path);
  });
}

kifmm_status kifmm_operators_load(const char* path, uint64_t expected_fingerprint, kifmm_operators** out) {
  return guard([&] {
    if (!out || !path) throw InvalidArgument("load: null argument");
    auto o = std::make_unique<kifmm_operators>();
    load_operators(o->o, path, expected_fingerprint);
    *out = o.release();
  });
}

kifmm_status kifmm_svd(const double* a, int32_t m, int32_t n, double* u, double* s, double* v) {
  return guard([&] { jacobi_svd(a, m, n, u, s, v, resolve_threads(0)); });
}

}  // extern "C"
