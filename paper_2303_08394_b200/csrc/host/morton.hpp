// Morton keys for the linear octree.
//
// Layout (bit positions pinned per SPEC.md:125):
//   raw = (interleave(anchor << (MAX_LEVEL - level)) << 4) | level
// with x in bit 3i, y in 3i+1, z in 3i+2 of the interleave.  Because the
// anchor is stored on the MAX_LEVEL grid, ascending raw order is Z-order at a
// fixed level *and* spatial order across levels with ancestors
// before descendants -- the cross-level comparator SURVEY Appendix C3 asks for.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>

namespace kifmm {

constexpr int kMaxLevel = 15;
constexpr uint32_t kFineCells = 1u << kMaxLevel;  // cells per axis at MAX_LEVEL

inline uint64_t spread3(uint32_t v) {
  uint64_t x = v & 0x1fffffu;
  x = (x | (x << 32)) & 0x1f00000000ffffULL;
  x = (x | (x << 16)) & 0x1f0000ff0000ffULL;
  x = (x | (x << 8)) & 0x100f00f00f00f00fULL;
  x = (x | (x << 4)) & 0x10c30c30c30c30c3ULL;
  x = (x | (x << 2)) & 0x1249249249249249ULL;
  return x;
}

inline uint32_t compact3(uint64_t x) {
  x &= 0x1249249249249249ULL;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ULL;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00fULL;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffULL;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffULL;
  x = (x ^ (x >> 32)) & 0x1fffffULL;
  return static_cast<uint32_t>(x);
}

// Interleaved code of fine-grid cell coordinates (each < 2^15).
inline uint64_t fine_code(uint32_t x, uint32_t y, uint32_t z) {
  return spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
}

inline int key_level(uint64_t key) { return static_cast<int>(key & 0xfu); }
inline uint64_t key_code(uint64_t key) { return key >> 4; }

// Unchecked encode: anchor on the node's own level grid.
inline uint64_t make_key(uint32_t ax, uint32_t ay, uint32_t az, int level) {
  const int sh = kMaxLevel - level;
  return (fine_code(ax << sh, ay << sh, az << sh) << 4) | static_cast<uint64_t>(level);
}

// Key of the level-`level` ancestor-or-self of fine cell code `code`.
inline uint64_t key_from_code(uint64_t code, int level) {
  const int sh = 3 * (kMaxLevel - level);
  return (((code >> sh) << sh) << 4) | static_cast<uint64_t>(level);
}

inline std::array<uint32_t, 3> key_anchor(uint64_t key) {
  const int sh = kMaxLevel - key_level(key);
  const uint64_t c = key_code(key);
  return {compact3(c) >> sh, compact3(c >> 1) >> sh, compact3(c >> 2) >> sh};
}

inline uint64_t key_parent(uint64_t key) { return key_from_code(key_code(key), key_level(key) - 1); }

inline uint64_t key_ancestor(uint64_t key, int level) { return key_from_code(key_code(key), level); }

// Octant of a node within its parent: dx + 2 dy + 4 dz.
inline int key_octant(uint64_t key) {
  const int l = key_level(key);
  return static_cast<int>((key_code(key) >> (3 * (kMaxLevel - l))) & 7u);
}

inline uint64_t key_child(uint64_t key, int octant) {
  const int l = key_level(key) + 1;
  const uint64_t c = key_code(key) | (static_cast<uint64_t>(octant) << (3 * (kMaxLevel - l)));
  return (c << 4) | static_cast<uint64_t>(l);
}

// Closed fine-grid extent [lo, hi] per axis (hi = lo + 2^(MAX-level)).
inline void key_extent(uint64_t key, int64_t lo[3], int64_t hi[3]) {
  const auto a = key_anchor(key);
  const int64_t w = int64_t(1) << (kMaxLevel - key_level(key));
  for (int d = 0; d < 3; ++d) {
    lo[d] = int64_t(a[d]) * w;
    hi[d] = lo[d] + w;
  }
}

// closed cubes share at least a point, and neither contains the other.
inline bool keys_adjacent(uint64_t a, uint64_t b) {
  int64_t alo[3], ahi[3], blo[3], bhi[3];
  key_extent(a, alo, ahi);
  key_extent(b, blo, bhi);
  bool a_in_b = true, b_in_a = true;
  for (int d = 0; d < 3; ++d) {
    if (alo[d] > bhi[d] || blo[d] > ahi[d]) return false;
    if (!(alo[d] >= blo[d] && ahi[d] <= bhi[d])) a_in_b = false;
    if (!(blo[d] >= alo[d] && bhi[d] <= ahi[d])) b_in_a = false;
  }
  return !(a_in_b || b_in_a);
}

// Same-level neighbours, ascending raw order.  Returns the count.
inline int key_neighbors(uint64_t key, uint64_t out[26]) {
  const int l = key_level(key);
  const auto a = key_anchor(key);
  const int64_t n = int64_t(1) << l;
  int cnt = 0;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz) {
        if (!dx && !dy && !dz) continue;
        const int64_t x = int64_t(a[0]) + dx, y = int64_t(a[1]) + dy, z = int64_t(a[2]) + dz;
        if (x < 0 || y < 0 || z < 0 || x >= n || y >= n || z >= n) continue;
        out[cnt++] = make_key(uint32_t(x), uint32_t(y), uint32_t(z), l);
      }
  std::sort(out, out + cnt);
  return cnt;
}

}  // namespace kifmm
