// Multi-GPU halo tables.
//
// Ranks own contiguous Z-order leaf ranges aligned to level-`cut` boxes (kifmm_partition_leaves; cut 0:
// the coarsest level >= 2 that balances the ranks' estimated cost within 5 %).  A node whose leaves all
// lie in one rank's range -- every leaf, every node at or below the cut -- is owned by that rank, which
// computes its multipole (P2M / M2M).  The few nodes above the cut that span ranks are recomputed by
// every rank from the gathered rows of their children.  The downward pass of rank r reads multipoles of
//   V(b) for every target node b at level >= 2 with an owned leaf below it (M2L),
//   W(a) for every owned leaf a (M2P),
//   the children of every redundantly computed top node at level >= 2 (M2M above the cut).
// Rows another rank owns are the halo.  Because V is symmetric and X is the dual of W,
// a row n owned by s is read by some other rank iff
//   some b in V(n) has a leaf outside s's range, or
//   some leaf a in X(n) lies outside s's range, or
//   n's parent is a redundantly computed top node (level >= 2),
// which is what rank s exports in the all-gather -- computed here in one pass over the lists, for all
// ranks at once (every rank needs every slot's layout).  tests/test_halo.py checks the tables against
// the direct definition of each rank's reads.
#include "halo.hpp"

#include <algorithm>
#include <memory>
#include <string>

#include "common.hpp"
#include "morton.hpp"

namespace kifmm {

void build_halo_plan(HaloPlan& h, const kifmm_tree_view& t, int n_e, bool gradient, int world, int cut) {
  if (world < 1) throw InvalidArgument("halo: world_size must be >= 1");
  if (cut < 0) throw InvalidArgument("halo: cut_level must be >= 0 (0 = auto)");
  const int64_t nn = t.n_nodes, nl = t.n_leaves;
  h.world = world;
  h.cut = cut;
  h.leaf_begin.assign(world + 1, 0);
  h.leaf_begin[world] = nl;
  if (world > 1) {
    const kifmm_status st = kifmm_partition_leaves(&t, n_e, gradient ? 1 : 0, world, cut, h.leaf_begin.data());
    if (st != KIFMM_OK) throw InvalidArgument(std::string("partition: ") + kifmm_last_error());
  }
  // leaf range under every node (leaves ascend in raw key = spatial Z-order)
  h.leaf_lo.assign(nn, INT64_MAX);
  h.leaf_hi.assign(nn, -1);
  for (int64_t l = 0; l < nl; ++l)
    for (int64_t n = t.leaf_node[l]; n >= 0; n = t.node_parent[n]) {
      h.leaf_lo[n] = std::min(h.leaf_lo[n], l);
      h.leaf_hi[n] = std::max(h.leaf_hi[n], l + 1);
    }
  auto rank_of_leaf = [&](int64_t l) {
    return int(std::upper_bound(h.leaf_begin.begin(), h.leaf_begin.end(), l) - h.leaf_begin.begin()) - 1;
  };
  h.up_owner.assign(nn, world == 1 ? 0 : -1);
  h.export_ptr.assign(world + 1, 0);
  h.export_idx.clear();
  h.max_export = 0;
  if (world == 1) return;
  for (int64_t n = 0; n < nn; ++n) {  // owner = the rank whose range holds every leaf below the node
    const int r = rank_of_leaf(h.leaf_lo[n]);
    if (h.leaf_hi[n] <= h.leaf_begin[r + 1]) h.up_owner[n] = r;
  }
  std::vector<std::vector<int64_t>> exp(world);
  for (int64_t n = 0; n < nn; ++n) {
    const int s = h.up_owner[n];
    if (s < 0) continue;
    const int64_t lb = h.leaf_begin[s], le = h.leaf_begin[s + 1];
    bool out = false;
    if (key_level(t.node_key[n]) >= 2)
      for (int64_t e = t.v_ptr[n]; e < t.v_ptr[n + 1] && !out; ++e) {
        const int64_t b = t.v_idx[e];
        out = h.leaf_lo[b] < lb || h.leaf_hi[b] > le;
      }
    for (int64_t e = t.x_ptr[n]; e < t.x_ptr[n + 1] && !out; ++e) {
      const int64_t a = t.x_idx[e];
      out = a < lb || a >= le;
    }
    const int64_t par = t.node_parent[n];
    if (!out && par >= 0 && h.up_owner[par] < 0 && key_level(t.node_key[par]) >= 2) out = true;
    if (out) exp[s].push_back(n);
  }
  for (int r = 0; r < world; ++r) {
    h.export_ptr[r + 1] = h.export_ptr[r] + int64_t(exp[r].size());
    h.export_idx.insert(h.export_idx.end(), exp[r].begin(), exp[r].end());
    h.max_export = std::max<int64_t>(h.max_export, int64_t(exp[r].size()));
  }
}

}  // namespace kifmm

// ---------------------------------------------------------------------- ABI
struct kifmm_halo {
  kifmm::HaloPlan h;
};

extern "C" {

kifmm_status kifmm_halo_plan(const kifmm_tree_view* tree, int32_t n_e, int32_t gradient, int32_t world_size,
                             int32_t cut_level, kifmm_halo** out) {
  return kifmm::guard([&] {
    if (!tree || !out || n_e < 1) throw kifmm::InvalidArgument("halo_plan: bad argument");
    auto p = std::make_unique<kifmm_halo>();
    kifmm::build_halo_plan(p->h, *tree, n_e, gradient != 0, world_size, cut_level);
    *out = p.release();
  });
}

kifmm_status kifmm_halo_get_view(const kifmm_halo* halo, kifmm_halo_view* v) {
  return kifmm::guard([&] {
    if (!halo || !v) throw kifmm::InvalidArgument("halo_get_view: null argument");
    const kifmm::HaloPlan& h = halo->h;
    v->world_size = h.world;
    v->cut_level = h.cut;
    v->n_nodes = int64_t(h.up_owner.size());
    v->leaf_begin = h.leaf_begin.data();
    v->up_owner = h.up_owner.data();
    v->export_ptr = h.export_ptr.data();
    v->export_idx = h.export_idx.data();
    v->max_export = h.max_export;
  });
}

void kifmm_halo_destroy(kifmm_halo* halo) { delete halo; }

}  // extern "C"
