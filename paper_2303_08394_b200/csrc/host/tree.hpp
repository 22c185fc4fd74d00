// Linear 2:1-balanced octree and interaction lists.
#pragma once

#include <cstdint>
#include <vector>

#include "keymap.hpp"
#include "morton.hpp"

namespace kifmm {

struct Tree {
  int64_t n = 0;
  int depth = 0;
  int n_overfull = 0;
  double origin[3] = {0, 0, 0};
  double side = 1.0;

  std::vector<double> positions;         // N x 3 reordered
  std::vector<int64_t> original_index;   // N
  std::vector<uint64_t> codes;           // fine cell code per reordered particle

  std::vector<uint64_t> leaves;          // ascending raw key
  std::vector<int64_t> leaf_ptr;         // n_leaves + 1

  std::vector<uint64_t> node_key;        // level-major
  std::vector<int64_t> level_ptr;        // depth + 2
  std::vector<int64_t> node_parent;
  std::vector<int64_t> node_children;    // n_nodes x 8
  std::vector<int64_t> node_leaf;
  std::vector<int64_t> leaf_node;
  KeyMap node_map;

  std::vector<int64_t> u_ptr, u_idx;
  std::vector<int64_t> v_ptr, v_idx;
  std::vector<int32_t> v_tv;
  std::vector<int64_t> w_ptr, w_idx;
  std::vector<int64_t> x_ptr, x_idx;

  int64_t n_leaves() const { return static_cast<int64_t>(leaves.size()); }
  int64_t n_nodes() const { return static_cast<int64_t>(node_key.size()); }
};

// Transfer-vector id of offset (dx,dy,dz) in [-3,3]^3 with Chebyshev norm >= 2, else -1.
int transfer_vector_id(int dx, int dy, int dz);
// Table of the 316 offsets, id order.
const std::vector<std::array<int, 3>>& transfer_vector_table();

// Fine-grid cell of a coordinate (half-open cells, closed upper domain face;
// SPEC.md:188).  Throws InvalidArgument for points outside the domain.
uint32_t fine_cell(double x, double origin, double side);

// Builds leaves, nodes and the particle permutation.  domain may be null.
void build_tree(Tree& t, const double* positions, int64_t n, int n_crit, const double* domain,
                bool balance, int threads);
// Fills u/v/w/x CSR lists.
void build_lists(Tree& t, int threads);

}  // namespace kifmm
