// Multi-GPU partition and halo-exchange tables.  Host C++, no device code: the GPU plan
// builds its exchange from these tables, and the CPU tests check them against the definitions.
#pragma once

#include <cstdint>
#include <vector>

#include "kifmm.h"

namespace kifmm {

struct HaloPlan {
  int world = 1, cut = 0;  // partition alignment level (0 = auto)
  std::vector<int64_t> leaf_begin;   // world + 1: rank r owns leaves [leaf_begin[r], leaf_begin[r+1])
  std::vector<int32_t> up_owner;     // n_nodes: rank that computes the multipole in its upward pass;
                                     // -1 = computed redundantly by every rank (nodes spanning ranks)
  std::vector<int64_t> leaf_lo, leaf_hi;  // n_nodes: leaf range [lo, hi) under the node
  // All-gather layout: rank r ships export_idx[export_ptr[r] .. export_ptr[r+1]) (ascending node index),
  // exactly the rows it owns that another rank reads; every rank's slot holds max_export rows.
  std::vector<int64_t> export_ptr, export_idx;
  int64_t max_export = 0;
};

// Partition (kifmm_partition_leaves) + owners + halo export sets.  world == 1: every node owned by
// rank 0, nothing exported.
void build_halo_plan(HaloPlan& h, const kifmm_tree_view& t, int n_e, bool gradient, int world, int cut);

}  // namespace kifmm
