// Open-addressing hash map MortonKey -> dense index (the SPEC's `key_index`,
// SPEC.md:134).  Immutable after construction, so concurrent lookups are safe.
#pragma once

#include <cstdint>
#include <vector>

namespace kifmm {

class KeyMap {
 public:
  KeyMap() = default;
  explicit KeyMap(std::size_t expected) { reserve(expected); }

  void reserve(std::size_t expected) {
    std::size_t cap = 16;
    while (cap < expected * 2 + 16) cap <<= 1;
    keys_.assign(cap, kEmpty);
    vals_.assign(cap, -1);
    mask_ = cap - 1;
    size_ = 0;
  }

  void insert(uint64_t key, int64_t val) {
    if ((size_ + 1) * 2 > keys_.size()) grow();
    std::size_t h = hash(key) & mask_;
    while (keys_[h] != kEmpty && keys_[h] != key) h = (h + 1) & mask_;
    if (keys_[h] == kEmpty) ++size_;
    keys_[h] = key;
    vals_[h] = val;
  }

  int64_t find(uint64_t key) const {
    if (keys_.empty()) return -1;
    std::size_t h = hash(key) & mask_;
    while (true) {
      const uint64_t k = keys_[h];
      if (k == key) return vals_[h];
      if (k == kEmpty) return -1;
      h = (h + 1) & mask_;
    }
  }

  bool contains(uint64_t key) const { return find(key) >= 0; }
  std::size_t size() const { return size_; }

 private:
  static constexpr uint64_t kEmpty = ~uint64_t(0);
  static uint64_t hash(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ULL;
    k ^= k >> 33;
    return k;
  }
  void grow() {
    std::vector<uint64_t> ok = std::move(keys_);
    std::vector<int64_t> ov = std::move(vals_);
    reserve(ok.size());
    for (std::size_t i = 0; i < ok.size(); ++i)
      if (ok[i] != kEmpty) insert(ok[i], ov[i]);
  }
  std::vector<uint64_t> keys_;
  std::vector<int64_t> vals_;
  std::size_t mask_ = 0;
  std::size_t size_ = 0;
};

}  // namespace kifmm
