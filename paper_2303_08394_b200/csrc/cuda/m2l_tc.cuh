// tcgen05 3xTF32 M2L (placeholder until the tensor-core path lands).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace kifmm {
namespace gpu {

inline bool m2l_tc_available() { return false; }

struct M2LTcPlan {
  template <class Tree, class Ops>
  void build(const Tree&, const std::vector<std::vector<int64_t>>&, int, const Ops&, size_t*) {
    throw InvalidArgument("tcgen05 M2L backend not built");
  }
  void launch(const float*, float*, int, cudaStream_t) {}
  int launches() const { return 0; }
};

}  // namespace gpu
}  // namespace kifmm
