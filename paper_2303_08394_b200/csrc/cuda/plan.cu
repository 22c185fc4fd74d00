// GPU evaluate plan: upload of tree/lists/operators, work-list construction,
// the evaluate launch sequence, CUDA-graph capture, the NCCL
// multipole exchange, and the kifmm_gpu_* C ABI.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"
#include "gemm.cuh"
#include <chrono>
#include <cstdio>

#include "halo.hpp"
#include "m2l_tc.cuh"
#include "morton.hpp"
#include "p2p.cuh"
#include "near_ws.cuh"
#include "m2l_oz.cuh"

namespace kifmm {
namespace gpu {

// ------------------------------------------------------------ device memory
struct DevMem {
  void* p = nullptr;
  size_t bytes = 0;
  DevMem() = default;
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  ~DevMem() {
    if (p) cudaFree(p);
  }
  void alloc(size_t b, size_t* total) {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = b;
    if (b) KIFMM_CUDA(cudaMalloc(&p, b));
    if (total) *total += b;
  }
  template <class T>
  void upload(const std::vector<T>& v, size_t* total) {
    alloc(v.size() * sizeof(T), total);
    if (!v.empty()) KIFMM_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Segmented gather-GEMM work description (see gemm.cuh).
struct TileSpec {
  std::vector<int> out;                                 // BM rows (-1 pad)
  std::vector<std::pair<int, std::vector<int>>> segs;   // (matrix, BM input rows)
};

struct GemmTiles {
  int n_tiles = 0, n_segs = 0, bm = 0;
  int64_t slots = 0;  // sum over segments of BM (computed rows incl. zero rows)
  DevMem out, seg_ptr, seg_mat, seg_in;
  void build(const std::vector<TileSpec>& tiles, int bm_, size_t* total) {
    bm = bm_;
    n_tiles = int(tiles.size());
    std::vector<int> o, sp{0}, sm, si;
    for (const auto& t : tiles) {
      o.insert(o.end(), t.out.begin(), t.out.end());
      for (const auto& s : t.segs) {
        sm.push_back(s.first);
        si.insert(si.end(), s.second.begin(), s.second.end());
      }
      sp.push_back(int(sm.size()));
    }
    n_segs = int(sm.size());
    slots = int64_t(n_segs) * bm;
    out.upload(o, total);
    seg_ptr.upload(sp, total);
    seg_mat.upload(sm, total);
    seg_in.upload(si, total);
  }
};

template <class T>
struct KC_;
template <>
struct KC_<float> {
  static constexpr int v = 32;
};
template <>
struct KC_<double> {
  static constexpr int v = 16;
};

// fp64 64-row tiles run on the DMMA kernel (KIFMM_DMMA=0: the SIMT DFMA kernel)
inline bool use_dmma() {  // read per launch (a captured graph keeps the choice of its capture)
  const char* e = std::getenv("KIFMM_DMMA");
  return !(e && std::atoi(e) == 0);
}

template <class T, int N, int BM, int TM>
void launch_gemm_n(const GemmTiles& t, const GemmArgs<T>& a, cudaStream_t s, int col_blocks = 1) {
  if constexpr (sizeof(T) == 8 && BM == 64 && N % 32 == 0) {
    if (use_dmma()) {
      auto kern = gather_dmma_kernel<N>;
      static bool attr = false;
      if (!attr) {
        KIFMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(DmmaShape<N>::SMEM)));
        attr = true;
      }
      kern<<<dim3(t.n_tiles, col_blocks), DmmaShape<N>::NT, DmmaShape<N>::SMEM, s>>>(a);
      KIFMM_LAUNCH_CHECK();
      return;
    }
  }
  constexpr int KC = KC_<T>::v;
  using S = GemmShape<T, N, BM, TM, 8, KC, 3>;
  auto kern = gather_gemm_kernel<T, N, BM, TM, 8, KC, 3>;
  static bool attr = false;
  if (!attr) {
    KIFMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::SMEM)));
    attr = true;
  }
  kern<<<dim3(t.n_tiles, col_blocks), S::NT, S::SMEM, s>>>(a);
  KIFMM_LAUNCH_CHECK();
}

template <class T, int BM, int TM>
void launch_gemm(int np, const GemmTiles& t, GemmArgs<T> a, cudaStream_t s) {
  if (t.n_tiles == 0) return;
  a.tile_out = t.out.as<int>();
  a.tile_seg = t.seg_ptr.as<int>();
  a.seg_mat = t.seg_mat.as<int>();
  a.seg_in = t.seg_in.as<int>();
  switch (np) {
    case 32: return launch_gemm_n<T, 32, BM, TM>(t, a, s);
    case 64: return launch_gemm_n<T, 64, BM, TM>(t, a, s);
    case 128: return launch_gemm_n<T, 128, BM, TM>(t, a, s);
    case 160: return launch_gemm_n<T, 160, BM, TM>(t, a, s);
    case 224: return launch_gemm_n<T, 224, BM, TM>(t, a, s);
    // p = 8, 9, 10: column blocks of an instantiated width (blockIdx.y; W row stride a.ldw = np)
    case 320: return launch_gemm_n<T, 160, BM, TM>(t, a, s, 2);
    case 448: return launch_gemm_n<T, 224, BM, TM>(t, a, s, 2);
    case 512: return launch_gemm_n<T, 128, BM, TM>(t, a, s, 4);
    default: throw InvalidArgument("gemm: unsupported padded width " + std::to_string(np));
  }
}

// SIMT M2L-shaped GEMM tiles (rows per tile / fp64 rows per thread); experiment overrides
#ifndef KIFMM_M2L_SIMT_BM
#define KIFMM_M2L_SIMT_BM 64
#endif
#ifndef KIFMM_M2L_SIMT_TM64
#define KIFMM_M2L_SIMT_TM64 8
#endif

// ------------------------------------------------------------------- NCCL
// libnccl is opened lazily so single-GPU use has no NCCL dependency.
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  static Nccl& get() {
    static Nccl n;
    if (!n.h) {
      n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!n.h) throw DeviceError(KIFMM_E_NCCL, "cannot dlopen libnccl.so.2");
      n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(dlsym(n.h, "ncclGetUniqueId"));
      n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(dlsym(n.h, "ncclCommInitRank"));
      n.allGather = reinterpret_cast<decltype(n.allGather)>(dlsym(n.h, "ncclAllGather"));
      n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(dlsym(n.h, "ncclCommDestroy"));
      n.getErrorString = reinterpret_cast<decltype(n.getErrorString)>(dlsym(n.h, "ncclGetErrorString"));
      if (!n.getUniqueId || !n.commInitRank || !n.allGather || !n.commDestroy)
        throw DeviceError(KIFMM_E_NCCL, "libnccl.so.2 lacks required symbols");
    }
    return n;
  }
  void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
      throw DeviceError(KIFMM_E_NCCL, std::string(what) + ": " + (getErrorString ? getErrorString(r) : "nccl error"));
  }
};

// Row gather / scatter for the multipole exchange.
template <class T>
__global__ void gather_rows_kernel(const T* __restrict__ src, int ld, const int* __restrict__ rows, int n,
                                   T* __restrict__ dst) {
  const int r = blockIdx.x;
  if (r >= n) return;
  for (int j = threadIdx.x; j < ld; j += blockDim.x) dst[size_t(r) * ld + j] = src[size_t(rows[r]) * ld + j];
}
// dst[rows[k]] = src[slot[k]] for the k-th received row (slot = rank * x_max + position in its export list)
template <class T>
__global__ void scatter_rows_kernel(const T* __restrict__ src, int ld, const int* __restrict__ rows,
                                    const int* __restrict__ slot, int n, T* __restrict__ dst) {
  const int k = blockIdx.x;
  if (k >= n) return;
  const T* a = src + size_t(slot[k]) * ld;
  T* b = dst + size_t(rows[k]) * ld;
  for (int j = threadIdx.x; j < ld; j += blockDim.x) b[j] = a[j];
}
// fp32 tcgen05 path: warp per received row, also writes the row's fp16 split (M2L A operand)
template <int W>
__global__ void scatter_rows_split_kernel(const float* __restrict__ src, const int* __restrict__ rows,
                                          const int* __restrict__ slot, int n, float* __restrict__ dst,
                                          __half* __restrict__ hi, __half* __restrict__ lo, float* __restrict__ un) {
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= n) return;
  const float* a = src + size_t(slot[k]) * W;
  const size_t row = size_t(rows[k]);
  float v[W / 32];
#pragma unroll
  for (int c = 0; c < W / 32; ++c) {
    v[c] = a[lane + 32 * c];
    dst[row * W + lane + 32 * c] = v[c];
  }
  split_row_warp<W>(v, lane, row, hi, lo, un);
}

template <class T>
void launch_check(int np, int n, const P2PParams<T>& pp, const CheckWork* works, const int2* ranges, const int* lvl,
                  int ref, T alpha, T* out, cudaStream_t s, const TcSplit* split = nullptr, bool half_warp = false) {
  const int blocks = int(ceil_div(n, kCheckWarps));
  if constexpr (sizeof(T) == 4) {
    // p = 4, 5, 6 (np = 64, 128, 160): packed fp32 kernels, which also write the fp16 split of the check row
    // for the tcgen05 solve -- half a warp per work (works sorted by source count), or a warp per work
    if (tc_np_supported(np)) {
      tc_dispatch_np(np, [&](auto w) {
        constexpr int K = decltype(w)::value / 32;
        if (half_warp)
          check_hw_kernel<K><<<int(ceil_div(n, 2 * kCheckWarps)), kCheckWarps * 32, 0, s>>>(
              pp, works, n, ranges, ref, alpha, out, np, split ? split->hi : nullptr, split ? split->lo : nullptr,
              split ? split->un : nullptr);
        else
          check_f2_kernel<K><<<blocks, kCheckWarps * 32, 0, s>>>(pp, works, n, ranges, ref, alpha, out, np,
                                                                 split ? split->hi : nullptr,
                                                                 split ? split->lo : nullptr,
                                                                 split ? split->un : nullptr);
      });
      KIFMM_LAUNCH_CHECK();
      return;
    }
  }
  switch ((np + 31) / 32) {
    case 1: check_kernel<T, 1><<<blocks, kCheckWarps * 32, 0, s>>>(pp, works, n, ranges, lvl, ref, alpha, out, np); break;
    case 2: check_kernel<T, 2><<<blocks, kCheckWarps * 32, 0, s>>>(pp, works, n, ranges, lvl, ref, alpha, out, np); break;
    case 4: check_kernel<T, 4><<<blocks, kCheckWarps * 32, 0, s>>>(pp, works, n, ranges, lvl, ref, alpha, out, np); break;
    case 5: check_kernel<T, 5><<<blocks, kCheckWarps * 32, 0, s>>>(pp, works, n, ranges, lvl, ref, alpha, out, np); break;
    case 7: check_kernel<T, 7><<<blocks, kCheckWarps * 32, 0, s>>>(pp, works, n, ranges, lvl, ref, alpha, out, np); break;
    case 10: check_kernel<T, 10><<<blocks, kCheckWarps * 32, 0, s>>>(pp, works, n, ranges, lvl, ref, alpha, out, np); break;
    case 14: check_kernel<T, 14><<<blocks, kCheckWarps * 32, 0, s>>>(pp, works, n, ranges, lvl, ref, alpha, out, np); break;
    case 16: check_kernel<T, 16><<<blocks, kCheckWarps * 32, 0, s>>>(pp, works, n, ranges, lvl, ref, alpha, out, np); break;
    default: throw InvalidArgument("check kernel: unsupported width");
  }
  KIFMM_LAUNCH_CHECK();
}

#ifdef KIFMM_EXPERIMENTS
// Experiments only (KIFMM_CORUN_DUMMY): a co-running load of one kind -- 0 FFMA chains, 1 LDS.128
// broadcasts, 2 MUFU.RSQ -- for `iters` rounds, to see which resource slows the tensor-core kernels.
__global__ void __launch_bounds__(128) dummy_load_kernel(int kind, int iters, float* out) {
  __shared__ float4 sh[256];
  sh[threadIdx.x] = make_float4(threadIdx.x, 1.f, 2.f, 3.f);
  sh[threadIdx.x + 128] = make_float4(threadIdx.x, 1.f, 2.f, 3.f);
  __syncthreads();
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
    if (kind == 0) {
#pragma unroll
      for (int u = 0; u < 16; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 0.999f, 0.001f);
    } else if (kind == 1) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float4 v = sh[(it * 16 + u) & 255];
        a[u & 7] += v.x + v.y;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 16; ++u) a[u & 7] = rsqrtf(a[u & 7] + 1.f);
    }
  }
  float t = 0.f;
  for (int i = 0; i < 8; ++i) t += a[i];
  if (t == -1.f) out[0] = t;
}
#endif

// M2M split over octants: partial products land in scratch rows (slot*8 + octant)
// and are summed here in fixed octant order (deterministic, no atomics).
template <class T>
__global__ void m2m_reduce_kernel(const T* __restrict__ scratch, const int* __restrict__ parents,
                                  const int* __restrict__ masks, int n, int ld, T* __restrict__ M) {
  const int s = blockIdx.x;
  if (s >= n) return;
  const int mask = masks[s];
  for (int c = threadIdx.x; c < ld; c += blockDim.x) {
    T acc = T(0);
#pragma unroll
    for (int o = 0; o < 8; ++o)
      if ((mask >> o) & 1) acc += scratch[(size_t(s) * 8 + o) * ld + c];
    M[size_t(parents[s]) * ld + c] = acc;
  }
}

// fp32 tcgen05 variant (warp per parent, same fixed octant order) that also writes the fp16 split of the
// parent row for the next tcgen05 GEMM (M2M of the level above, M2L)
template <int W>
__global__ void m2m_reduce_split_kernel(const float* __restrict__ scratch, const int* __restrict__ parents,
                                        const int* __restrict__ masks, int n, float* __restrict__ M,
                                        __half* __restrict__ hi, __half* __restrict__ lo, float* __restrict__ un) {
  pdl_trigger();
  pdl_wait();
  const int s = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (s >= n) return;
  const int mask = masks[s];
  float v[W / 32];
#pragma unroll
  for (int k = 0; k < W / 32; ++k) {
    float acc = 0.f;
#pragma unroll
    for (int o = 0; o < 8; ++o)
      if ((mask >> o) & 1) acc += scratch[(size_t(s) * 8 + o) * W + lane + 32 * k];
    v[k] = acc;
  }
  const size_t row = size_t(parents[s]);
#pragma unroll
  for (int k = 0; k < W / 32; ++k) M[row * W + lane + 32 * k] = v[k];
  split_row_warp<W>(v, lane, row, hi, lo, un);
}

// Y[out(r)] += sum over a tile's pieces (fixed order) of partial[slot][r]   (rows x ld per piece)
template <class T>
__global__ void reduce_partials_kernel(const T* __restrict__ partial, const int* __restrict__ tile_out,
                                       const int* __restrict__ tile_slot, int rows, int ld, T* __restrict__ Y) {
  const int tile = blockIdx.x;
  const int s0 = tile_slot[tile], s1 = tile_slot[tile + 1];
  for (int idx = threadIdx.x; idx < rows * ld; idx += blockDim.x) {
    const int r = idx / ld, col = idx % ld;
    const int out = tile_out[size_t(tile) * rows + r];
    if (out < 0) continue;
    T acc = Y[size_t(out) * ld + col];
    for (int sl = s0; sl < s1; ++sl) acc += partial[(size_t(sl) * rows + r) * ld + col];
    Y[size_t(out) * ld + col] = acc;
  }
}

struct LeafPlan {
  DevMem works, rounds, items;
  int n = 0;
};

struct M2MLevel {
  int level = 0;    // parent level
  GemmTiles tiles;  // one tile per (64 parents, octant)   [SIMT]
  TcGemm tc;        // one tile per (128 parents, octant), or per 128 parents with 8 octant taps (direct)
  bool direct = false;
  int r0 = 0, r1 = 0;  // child rows to split before the tcgen05 GEMM
  DevMem parents, masks;
  int n = 0;
};

struct L2LLevel {
  GemmTiles tiles;
  TcGemm tc;
  int r0 = 0, r1 = 0;  // parent rows (level l) to split
};

}  // namespace gpu
}  // namespace kifmm

using namespace kifmm;
using namespace kifmm::gpu;

struct kifmm_gpu_plan {
  kifmm_gpu_options opt{};
  int device = 0;
  int precision = 32;
  bool leaf_packed = false;
  // warp-specialised persistent near-field kernel (bit-identical results): KIFMM_NEAR_WS=0 never, 1 (default) for
  // the queue-mode side / drain launches of the captured evaluate (config 2: 1.33 vs 1.35 ms), 2 also for the
  // standalone launch of the serialized timed run (there 2-5 % slower than one leaf_eval_f2 block per leaf)
  int near_ws = 1;
  int near_ws_bps = 2;
  int near_ws_blocks = 6;  // resident blocks per SM of the standalone / drain launch (occupancy query)   // its side blocks per SM next to the tcgen05 kernels (smem: 2 x 37 KB + stages)
  int near_pause = 0;  // side blocks sleep during M2L: 1 all, 2 half (KIFMM_NEAR_PAUSE; 1 measured slower)
  int near_bps = 3;  // queue mode: near-field blocks per SM next to the tree passes (KIFMM_NEAR_BPS, 0 = off)
  bool m2m_parent_tiles = false;  // KIFMM_M2M=parent: 8-tap parent tiles, direct (measured slower)
  DevMem near_counter;  // queue mode work counter [, counter at the drain launch (KIFMM_NEAR_DEBUG)]
  bool near_debug = false, near_skip = false, far_as_leaf = false, near_corun = false;
  int near_fork_at = 0;  // 0: at the start of the evaluate, 1: just before M2L, 2: after the P2M check, 3: after M2M
  bool check_hw = true;     // fp32 p = 6 check potentials: half-warp kernel (KIFMM_CHECK_HW=0: warp per work)
  bool near_pair64 = false;  // fp64 near field: two targets per thread (leaf_eval_pair_kernel; KIFMM_NEAR_PAIR64)
  bool near_serial = false;  // near field on the plan stream after L2L instead of a side stream (KIFMM_NEAR_SERIAL;
                             // default for fp64)
  bool grad = false;
  int64_t N = 0, nl = 0, nn = 0;
  int depth = 0, ne = 0, nc = 0, np = 0, ref_level = 2;
  int world = 1, rank = 0;
  int64_t lb = 0, le = 0, pb = 0, pe = 0;  // owned leaves / particles
  int m2l_backend = 1;
  double alpha_in = 1.05, alpha_out = 2.95;
  size_t dev_bytes = 0;
  cudaStream_t stream = nullptr, side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_done = nullptr;  // end of the last evaluate (any entry point, any stream)
  cudaEvent_t ev_half[2] = {nullptr, nullptr};  // device span of an upward / downward half (exchange = 1)
  std::array<cudaEvent_t, 16> ev{};
  kifmm_gpu_plan_info info{};
  kifmm_gpu_timings last{};

  // static data
  DevMem pos4, perm, node_geom, node_lo, node_level, surface;
  DevMem w_us_u, w_vt_u, w_us_d, w_vt_d, w_m2m, w_l2l, w_m2l;
  // per-evaluate buffers
  DevMem q_in, src4, pot, grad_buf, pot_out, grad_out;
  DevMem M, L, check_up, check_dn, tmp;
  // work lists
  DevMem p2m_works, p2m_ranges, p2l_works, p2l_ranges;
  LeafPlan leaf_near, leaf_far;
  DevMem far_works, far_surfaces, leaf_ptr_dev;  // far_works: int4 (scalar kernel) or FarWork (packed)
  int n_far = 0;
  int far_chunk = 0, n_far_groups = 0;  // surface chunking of long half-warp far works (see build)
  DevMem far_part, far_groups;
  bool far_packed = false;  // fp32 packed far kernels (fused output write); else the scalar chunked far_kernel
  bool far_hw = false;  // half-warp far kernel (every work has at most one surface; KIFMM_FAR_HW=0: off)
  int n_p2m = 0, n_p2l = 0;
  GemmTiles solve_up1, solve_up2, solve_dn1, solve_dn2, m2l;
  std::vector<std::unique_ptr<M2MLevel>> m2m_levels, m2m_top;
  std::vector<std::unique_ptr<L2LLevel>> l2l_levels;
  // fp32 solves / M2M / L2L on tcgen05 (kind::f16 3-term split) -- see TcGemm
  bool gemm_tc = false;
  TcSplit sp_cu, sp_tmp, sp_M, sp_cd, sp_L;
  TcGemm tg_up1, tg_up2, tg_dn1, tg_dn2;
  // split downward chain (tcgen05 path): second solve GEMM for the levels above the deepest one, then the
  // L2L chain into those levels on side2, concurrent with the deepest level's second solve on the plan
  // stream (run on the fewest CTAs with the same makespan, leaving SMs to the chain); joined before the
  // last L2L level.  KIFMM_DN_SPLIT=0: one second-solve GEMM, then the L2L levels in order.
  bool dn_split = false;
  int dn_split_level = 0;  // child level of the last L2L level (the deepest)
  TcGemm tg_dn2_up, tg_dn2_lo;
  cudaStream_t side2 = nullptr;
  cudaEvent_t ev_dn_fork = nullptr, ev_dn_join = nullptr;
  // P2L (MUFU-bound check potentials) on side2 next to the tensor-core M2L kernel, which neither reads nor
  // writes the check rows; the M2L reduction joins them (KIFMM_P2L_OVERLAP=0: serial)
  bool p2l_overlap = true;
  cudaEvent_t ev_p2l_fork = nullptr, ev_p2l_join = nullptr;
  DevMem dn_extra;  // down-check rows with P2L but no M2L (split after M2L)
  int n_dn_extra = 0;
  DevMem m2m_scratch;
  DevMem m2l_red_out, m2l_red_slot, m2l_partial;
  int m2l_red_tiles = 0;
  int64_t m2m_scratch_rows = 0;
  M2LTcPlan m2l_tc;
  M2LOzPlan m2l_oz;  // fp64 M2L on the int8 tensor cores (m2l_backend 4)
  // exchange
  void* comm = nullptr;
  DevMem x_send, x_recv, x_rows, x_rank /* source slot of each received row */, x_my_rows;
  int x_max = 0, x_total = 0, x_mine = 0;
  bool host_phase_input_order = true;  // exchange = 1: the input_order of the pending upward half
  // graphs
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  // evaluate_many: copy-in / copy-out streams and double-buffered device staging (created on first use)
  struct Pipe {
    cudaStream_t cin = nullptr, cout = nullptr;
    cudaEvent_t in_ready[2]{}, in_free[2]{}, out_ready[2]{}, out_free[2]{};
    DevMem q[2], pot[2], grad[2];
  };
  std::unique_ptr<Pipe> pipe;

  ~kifmm_gpu_plan() {
    for (auto& g : graph)
      if (g) cudaGraphExecDestroy(g);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    if (side) cudaStreamDestroy(side);
    if (side2) cudaStreamDestroy(side2);
    if (ev_dn_fork) cudaEventDestroy(ev_dn_fork);
    if (ev_dn_join) cudaEventDestroy(ev_dn_join);
    if (ev_p2l_fork) cudaEventDestroy(ev_p2l_fork);
    if (ev_p2l_join) cudaEventDestroy(ev_p2l_join);
    if (pipe) {
      if (pipe->cin) cudaStreamDestroy(pipe->cin);
      if (pipe->cout) cudaStreamDestroy(pipe->cout);
      for (int b = 0; b < 2; ++b)
        for (cudaEvent_t e : {pipe->in_ready[b], pipe->in_free[b], pipe->out_ready[b], pipe->out_free[b]})
          if (e) cudaEventDestroy(e);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_done) cudaEventDestroy(ev_done);
    for (auto& e : ev_half)
      if (e) cudaEventDestroy(e);
    if (comm) Nccl::get().commDestroy(static_cast<ncclComm_t>(comm));
  }

  size_t esz() const { return precision == 32 ? 4 : 8; }
  void build(const kifmm_gpu_options& o, const kifmm_tree_view& t, const kifmm_operator_view& ops);
  template <class T>
  void upload_static(const kifmm_tree_view& t, const kifmm_operator_view& ops);
  template <class T>
  // phase 1: upward pass (+ the export rows of a multi-rank plan into x_send); 2: exchange import +
  // downward pass + leaves; 3: both, with the NCCL all-gather between them
  void run(cudaStream_t s, bool input_order, bool timed, int phase = 3);
  void gather_exports(cudaStream_t s);
  void allgather(cudaStream_t s);
  void scatter_imports(cudaStream_t s);
  void evaluate_device(const void* q, void* pot_dst, void* grad_dst, bool input_order, cudaStream_t user, bool timed);
  // the captured evaluate graph of this output order (captured on the plan stream on first use, with the
  // capture always ended -- also when a launch throws -- so the stream never stays in capture mode),
  // launched on `s`
  void launch_graph(bool input_order, cudaStream_t s) {
    const int gi = input_order ? 1 : 0;
    if (!graph[gi]) {
      cudaGraph_t g;
      KIFMM_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      try {
        if (precision == 32)
          run<float>(stream, input_order, false);
        else
          run<double>(stream, input_order, false);
      } catch (...) {
        cudaStreamEndCapture(stream, &g);
        throw;
      }
      KIFMM_CUDA(cudaStreamEndCapture(stream, &g));
      const cudaError_t e = cudaGraphInstantiateWithFlags(&graph[gi], g, cudaGraphInstantiateFlagUseNodePriority);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) {
        graph[gi] = nullptr;
        KIFMM_CUDA(e);
      }
    }
    KIFMM_CUDA(cudaGraphLaunch(graph[gi], s));
  }
  // Every evaluate entry point orders itself after the previous evaluate of this plan, whichever stream
  // that one ran on (the plan's buffers -- q_in, src4, M, L, check rows, outputs, the near-field counter --
  // are shared by all of them): wait on `ev_done` first, record it last.
  void begin(cudaStream_t s) { KIFMM_CUDA(cudaStreamWaitEvent(s, ev_done, 0)); }
  void require_single_call() const {
    if (world > 1 && opt.exchange == 1)
      throw InvalidArgument("evaluate: a host-exchange plan runs as kifmm_gpu_evaluate_upward + _downward");
  }
  // results (input order: the full vector, other ranks' entries zero; reordered: this rank's range) -> dst
  void copy_out(void* pot_dst, void* grad_dst, bool input_order, cudaStream_t s) {
    const size_t es = esz();
    const void* ps = input_order ? pot_out.p : pot.p;
    const void* gs = input_order ? grad_out.p : grad_buf.p;
    if (input_order || world == 1) {
      if (pot_dst) KIFMM_CUDA(cudaMemcpyAsync(pot_dst, ps, size_t(N) * es, cudaMemcpyDefault, s));
      if (grad && grad_dst) KIFMM_CUDA(cudaMemcpyAsync(grad_dst, gs, size_t(N) * 3 * es, cudaMemcpyDefault, s));
    } else {
      const size_t off = size_t(pb) * es, cnt = size_t(pe - pb) * es;
      if (pot_dst && cnt)
        KIFMM_CUDA(cudaMemcpyAsync(static_cast<char*>(pot_dst) + off, static_cast<const char*>(ps) + off, cnt,
                                   cudaMemcpyDefault, s));
      if (grad && grad_dst && cnt)
        KIFMM_CUDA(cudaMemcpyAsync(static_cast<char*>(grad_dst) + 3 * off, static_cast<const char*>(gs) + 3 * off,
                                   3 * cnt, cudaMemcpyDefault, s));
    }
  }
  void finish(cudaStream_t s) { KIFMM_CUDA(cudaEventRecord(ev_done, s)); }
  void evaluate_many(int n_rhs, const void* const* charges, void* const* potentials, void* const* gradients,
                     bool input_order);
};

namespace {

int round_up(int x, int m) { return (x + m - 1) / m * m; }

template <class T>
std::vector<T> to_t(const std::vector<double>& v) {
  return std::vector<T>(v.begin(), v.end());
}

}  // namespace

template <class T>
void kifmm_gpu_plan::upload_static(const kifmm_tree_view& t, const kifmm_operator_view& ops) {
  // positions (x, y, z, 0)
  std::vector<T> p4(size_t(N) * 4);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    for (int d = 0; d < 3; ++d) p4[4 * i + d] = T(t.positions[3 * i + d]);
    p4[4 * i + 3] = T(0);
  }
  pos4.upload(p4, &dev_bytes);
  std::vector<int> pm(N);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) pm[i] = int(t.original_index[i]);
  perm.upload(pm, &dev_bytes);
  // node geometry (center, half side) computed in fp64 then rounded
  std::vector<T> g(size_t(nn) * 4), glo(size_t(nn) * 4, T(0));  // glo: centre - T(centre) (fp32 node-local geometry)
  std::vector<int> lv(nn);
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < nn; ++n) {
    const uint64_t k = t.node_key[n];
    const auto a = key_anchor(k);
    const int l = key_level(k);
    const double w = t.side / double(uint64_t(1) << l);
    for (int d = 0; d < 3; ++d) {
      const double c = t.origin[d] + (double(a[d]) + 0.5) * w;
      g[4 * n + d] = T(c);
      glo[4 * n + d] = T(c - double(T(c)));
    }
    g[4 * n + 3] = T(t.side / double(uint64_t(1) << (l + 1)));
    lv[n] = l;
  }
  node_geom.upload(g, &dev_bytes);
  node_lo.upload(glo, &dev_bytes);
  node_level.upload(lv, &dev_bytes);
  surface.upload(to_t<T>(std::vector<double>(ops.surface, ops.surface + 3 * ne)), &dev_bytes);

  // factored pinvs as two GEMM operands: W1 = U diag(1/s) (nc x k), W2 = V^T (k x ne), zero padded to np x np
  auto factored = [&](const double* U, const double* S, const double* V, int k, DevMem& w1, DevMem& w2) {
    std::vector<double> a(size_t(np) * np, 0.0), b(size_t(np) * np, 0.0);
    for (int i = 0; i < nc; ++i)
      for (int j = 0; j < k; ++j) a[size_t(i) * np + j] = U[size_t(i) * k + j] / S[j];
    for (int j = 0; j < k; ++j)
      for (int e = 0; e < ne; ++e) b[size_t(j) * np + e] = V[size_t(e) * k + j];
    w1.upload(to_t<T>(a), &dev_bytes);
    w2.upload(to_t<T>(b), &dev_bytes);
  };
  factored(ops.uc2e_u, ops.uc2e_s, ops.uc2e_v, ops.uc2e_rank, w_us_u, w_vt_u);
  factored(ops.dc2e_u, ops.dc2e_s, ops.dc2e_v, ops.dc2e_rank, w_us_d, w_vt_d);
  // W[k][n] = A[n][k] for m2m / l2l / m2l (out_n = sum_k A[n][k] in_k)
  auto transposed = [&](const double* A, int count, int rows, int cols, DevMem& w) {
    std::vector<T> out(size_t(count) * np * np, T(0));
    for (int c = 0; c < count; ++c)
      for (int n = 0; n < rows; ++n)
        for (int k = 0; k < cols; ++k)
          out[size_t(c) * np * np + size_t(k) * np + n] = T(A[size_t(c) * rows * cols + size_t(n) * cols + k]);
    w.upload(out, &dev_bytes);
  };
  transposed(ops.m2m, 8, ne, ne, w_m2m);
  transposed(ops.l2l, 8, ne, ne, w_l2l);
  transposed(ops.m2l, ops.n_m2l, nc, ne, w_m2l);
}

void kifmm_gpu_plan::build(const kifmm_gpu_options& o, const kifmm_tree_view& t, const kifmm_operator_view& ops) {
  // plan-creation phase timing (KIFMM_PLAN_TIMING=1 prints host wall times per phase)
  const bool ptime = std::getenv("KIFMM_PLAN_TIMING") != nullptr;
  auto pt0 = std::chrono::steady_clock::now();
  auto ptick = [&](const char* what) {
    if (!ptime) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "plan %-22s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - pt0).count());
    pt0 = now;
  };
  opt = o;
  device = o.device;
  precision = o.precision;
  grad = o.gradient != 0;
  world = std::max(1, o.world_size);
  rank = o.rank;
  if (precision != 32 && precision != 64) throw InvalidArgument("gpu: precision must be 32 or 64");
  if (rank < 0 || rank >= world) throw InvalidArgument("gpu: rank out of range");
  if (ops.n_e != ops.n_c) throw InvalidArgument("gpu: n_c != n_e is not supported");
  if (ops.n_e > 512) throw InvalidArgument("gpu: expansion order above p=10 (n_e > 512) is not supported");
  if (t.n_particles >= (int64_t(1) << 31)) throw InvalidArgument("gpu: N >= 2^31");
  if (ops.n_m2l != 316) throw InvalidArgument("gpu: operator cache must hold 316 M2L matrices");
  KIFMM_CUDA(cudaSetDevice(device));
  N = t.n_particles;
  nl = t.n_leaves;
  nn = t.n_nodes;
  depth = t.depth;
  ne = ops.n_e;
  nc = ops.n_c;
  np = round_up(ne, 32);
  if (np == 96 || np == 192) np += 32;  // instantiated widths: 32, 64, 128, 160, 224
  // p = 8, 9, 10 (n_e = 296, 386, 488 -> 320, 448, 512): column blocks of the 160 / 224 / 128-wide GEMM
  // kernels, chunked far-field staging
  if (np == 416) np = 448;
  ref_level = ops.reference_level;
  alpha_in = ops.alpha_inner;
  alpha_out = ops.alpha_outer;
  const double expect_half = t.side / double(1 << (ref_level + 1));
  if (std::fabs(ops.ref_half_side - expect_half) > 1e-12 * expect_half)
    throw InvalidArgument("gpu: operator cache was built for another domain side");
  {
    int lo = 0, hi = 0;  // numerically lower = higher priority
    KIFMM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    KIFMM_CUDA(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, hi));
    KIFMM_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo));
    KIFMM_CUDA(cudaStreamCreateWithPriority(&side2, cudaStreamNonBlocking, hi));
    KIFMM_CUDA(cudaEventCreateWithFlags(&ev_dn_fork, cudaEventDisableTiming));
    KIFMM_CUDA(cudaEventCreateWithFlags(&ev_dn_join, cudaEventDisableTiming));
    KIFMM_CUDA(cudaEventCreateWithFlags(&ev_p2l_fork, cudaEventDisableTiming));
    KIFMM_CUDA(cudaEventCreateWithFlags(&ev_p2l_join, cudaEventDisableTiming));
    if (const char* e = std::getenv("KIFMM_P2L_OVERLAP")) p2l_overlap = std::atoi(e) != 0;
    KIFMM_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    KIFMM_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    KIFMM_CUDA(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
    for (auto& e : ev_half) KIFMM_CUDA(cudaEventCreate(&e));
  }
  for (auto& e : ev) KIFMM_CUDA(cudaEventCreate(&e));
  check_hw = precision == 32 && tc_np_supported(np);
  if (const char* e = std::getenv("KIFMM_CHECK_HW")) check_hw = check_hw && std::atoi(e) != 0;

  ptick("setup");
  // ---- partition, owners, halo export tables (csrc/host/halo.cpp)
  HaloPlan halo;
  build_halo_plan(halo, t, ne, grad, world, std::max(0, o.cut_level));
  const std::vector<int64_t>& lbeg = halo.leaf_begin;
  lb = lbeg[rank];
  le = lbeg[rank + 1];
  pb = t.leaf_ptr[lb];
  pe = t.leaf_ptr[le];
  auto node_lvl = [&](int64_t n) { return key_level(t.node_key[n]); };
  auto is_leaf = [&](int64_t n) { return t.node_leaf[n] >= 0; };
  // owner rank of a node's multipole in the upward pass (-1: every rank recomputes it after the exchange)
  const std::vector<int32_t>& up_owner = halo.up_owner;
  // downward-active nodes: ancestors-or-self of owned leaves
  std::vector<char> active(nn, 0);
  for (int64_t l = lb; l < le; ++l)
    for (int64_t n = t.leaf_node[l]; n >= 0 && !active[n]; n = t.node_parent[n]) active[n] = 1;

  if (precision == 32)
    upload_static<float>(t, ops);
  else
    upload_static<double>(t, ops);

  const size_t es = esz();
  q_in.alloc(size_t(N) * es, &dev_bytes);
  src4.alloc(size_t(N) * 4 * es, &dev_bytes);
  pot.alloc(size_t(N) * es, &dev_bytes);
  pot_out.alloc(size_t(N) * es, &dev_bytes);
  if (grad) {
    grad_buf.alloc(size_t(N) * 3 * es, &dev_bytes);
    grad_out.alloc(size_t(N) * 3 * es, &dev_bytes);
  }
  M.alloc(size_t(nn) * np * es, &dev_bytes);
  L.alloc(size_t(nn) * np * es, &dev_bytes);
  KIFMM_CUDA(cudaMemset(M.p, 0, M.bytes));
  KIFMM_CUDA(cudaMemset(L.p, 0, L.bytes));
  check_dn.alloc(size_t(nn) * np * es, &dev_bytes);

  const int bm_m2l = 64;
  {
    const char* e = std::getenv("KIFMM_TC_GEMM");
    gemm_tc = precision == 32 && tc_np_supported(np) && o.m2l_backend != 1 && m2l_tc_available() &&
              !(e && std::string(e) == "0");
  }
  // solves / L2L: 64-row tiles on the SIMT path (2 CTAs per SM; K = 160 only), 128 on tcgen05
  const int ld_tiles = gemm_tc ? tc::BM : 64;
  // fp64 B operands of the tcgen05 GEMMs: B[m][j][k], j = output column, k = reduction index
  auto factored_b = [&](const double* U, const double* S, const double* V, int k, std::vector<double>& b1,
                        std::vector<double>& b2) {
    b1.assign(size_t(np) * np, 0.0);
    b2.assign(size_t(np) * np, 0.0);
    for (int i = 0; i < nc; ++i)
      for (int j = 0; j < k; ++j) b1[size_t(j) * np + i] = U[size_t(i) * k + j] / S[j];
    for (int j = 0; j < k; ++j)
      for (int e = 0; e < ne; ++e) b2[size_t(e) * np + j] = V[size_t(e) * k + j];
  };
  auto octant_b = [&](const double* A) {  // 8 x (ne x ne) -> 8 x np x np
    std::vector<double> b(size_t(8) * np * np, 0.0);
    for (int m = 0; m < 8; ++m)
      for (int j = 0; j < ne; ++j)
        for (int k = 0; k < ne; ++k) b[(size_t(m) * np + j) * np + k] = A[(size_t(m) * ne + j) * ne + k];
    return b;
  };

  ptick("partition+static upload");
  // ---- P2M: one check work per owned leaf, solve rows = slots
  {
    std::vector<CheckWork> w;
    std::vector<int2> rg;
    for (int64_t l = lb; l < le; ++l) {
      const int64_t ln = t.leaf_node[l];
      w.push_back({int(ln), int(l - lb), int(rg.size()), int(rg.size()) + 1, int(t.leaf_ptr[l]),
                   int(t.leaf_ptr[l + 1] - t.leaf_ptr[l]), node_lvl(ln), 0});
      rg.push_back(make_int2(int(t.leaf_ptr[l]), int(t.leaf_ptr[l + 1] - t.leaf_ptr[l])));
      info.p2m_pairs += (t.leaf_ptr[l + 1] - t.leaf_ptr[l]) * ne;
    }
    n_p2m = int(w.size());
    if (check_hw) {  // half-warp check kernel: pair works of similar source counts in a warp
      auto srcs = [&](const CheckWork& c) {
        int64_t n = 0;
        for (int r = c.range_begin; r < c.range_end; ++r) n += rg[r].y;
        return n;
      };
      std::vector<std::pair<int64_t, int>> key(w.size());
      for (size_t i = 0; i < w.size(); ++i) key[i] = {-srcs(w[i]), int(i)};
      std::stable_sort(key.begin(), key.end());
      std::vector<CheckWork> sorted(w.size());
      for (size_t i = 0; i < w.size(); ++i) sorted[i] = w[key[i].second];
      w.swap(sorted);
    }
    p2m_works.upload(w, &dev_bytes);
    p2m_ranges.upload(rg, &dev_bytes);
    check_up.alloc(size_t(std::max<int64_t>(1, le - lb)) * np * es, &dev_bytes);
    std::vector<TileSpec> a, b;
    for (int64_t s0 = 0; s0 < le - lb; s0 += ld_tiles) {
      TileSpec x, y;
      std::vector<int> slots(ld_tiles, -1), nodes(ld_tiles, -1);
      for (int r = 0; r < ld_tiles && s0 + r < le - lb; ++r) {
        slots[r] = int(s0 + r);
        nodes[r] = int(t.leaf_node[lb + s0 + r]);
      }
      x.out = slots;
      x.segs.push_back({0, slots});
      y.out = nodes;
      y.segs.push_back({0, slots});
      a.push_back(x);
      b.push_back(y);
    }
    if (gemm_tc) {
      std::vector<double> b1, b2;
      factored_b(ops.uc2e_u, ops.uc2e_s, ops.uc2e_v, ops.uc2e_rank, b1, b2);
      tg_up1.build(a, b1, 1, np, &dev_bytes);
      tg_up2.build(b, b2, 1, np, &dev_bytes);
      sp_cu.alloc(int(std::max<int64_t>(1, le - lb)), np, &dev_bytes);
    } else {
      solve_up1.build(a, ld_tiles, &dev_bytes);
      solve_up2.build(b, ld_tiles, &dev_bytes);
    }
  }

  ptick("P2M + up solves");
  // ---- M2M per level (owned internal nodes), then the redundant top levels
  const std::vector<double> b_m2m = gemm_tc ? octant_b(ops.m2m) : std::vector<double>();
  if (const char* e = std::getenv("KIFMM_M2M")) m2m_parent_tiles = std::string(e) == "parent";
  auto m2m_tiles = [&](std::vector<int64_t>& parents) {
    const int BMS = gemm_tc ? tc::BM : 64;
    std::vector<TileSpec> tiles;
    std::vector<int> par, msk;
    for (size_t s0 = 0; s0 < parents.size(); s0 += BMS) {
      for (int o = 0; o < 8; ++o) {
        TileSpec ts;
        ts.out.assign(BMS, -1);
        std::vector<int> in(BMS, -1);
        bool any = false;
        for (int r = 0; r < BMS && s0 + r < parents.size(); ++r) {
          const int64_t ch = t.node_children[8 * parents[s0 + r] + o];
          if (ch < 0) continue;
          ts.out[r] = int((s0 + r) * 8 + o);
          in[r] = int(ch);
          any = true;
        }
        if (!any) continue;
        ts.segs.push_back({o, in});
        tiles.push_back(std::move(ts));
      }
    }
    for (int64_t pn : parents) {
      int m = 0;
      for (int o = 0; o < 8; ++o)
        if (t.node_children[8 * pn + o] >= 0) m |= 1 << o;
      par.push_back(int(pn));
      msk.push_back(m);
    }
    auto g = std::make_unique<M2MLevel>();
    if (gemm_tc && m2m_parent_tiles) {
      // parent-major tiles: 128 parents x up to 8 octant taps accumulate in the epilogue and are written
      // straight into M (+ split) -- no scratch rows, no reduction launch
      std::vector<TileSpec> pt;
      for (size_t s0 = 0; s0 < parents.size(); s0 += tc::BM) {
        TileSpec ts;
        ts.out.assign(tc::BM, -1);
        for (int r = 0; r < tc::BM && s0 + r < parents.size(); ++r) ts.out[r] = int(parents[s0 + r]);
        for (int o = 0; o < 8; ++o) {
          std::vector<int> in(tc::BM, -1);
          bool any = false;
          for (int r = 0; r < tc::BM && s0 + r < parents.size(); ++r) {
            const int64_t ch = t.node_children[8 * parents[s0 + r] + o];
            if (ch >= 0) {
              in[r] = int(ch);
              any = true;
            }
          }
          if (any) ts.segs.push_back({o, in});
        }
        pt.push_back(std::move(ts));
      }
      g->tc.build(pt, b_m2m, 8, np, &dev_bytes);
      g->direct = true;
    } else if (gemm_tc) {
      g->tc.build(tiles, b_m2m, 8, np, &dev_bytes);
      int64_t lo = INT64_MAX, hi = -1;  // child rows (one level: contiguous node range)
      for (int64_t pn : parents)
        for (int o = 0; o < 8; ++o) {
          const int64_t ch = t.node_children[8 * pn + o];
          if (ch >= 0) {
            lo = std::min(lo, ch);
            hi = std::max(hi, ch + 1);
          }
        }
      g->r0 = int(lo == INT64_MAX ? 0 : lo);
      g->r1 = int(std::max<int64_t>(hi, g->r0));
    } else {
      g->tiles.build(tiles, BMS, &dev_bytes);
    }
    g->parents.upload(par, &dev_bytes);
    g->masks.upload(msk, &dev_bytes);
    g->n = int(parents.size());
    g->level = parents.empty() ? 0 : node_lvl(parents[0]);
    m2m_scratch_rows = std::max<int64_t>(m2m_scratch_rows, int64_t(parents.size()) * 8);
    return g;
  };
  // parents above level 2 get no M2M: V / W members are all at level >= 2, so multipoles of levels 0-1
  // feed no operator (the reference's M2M loop computes them, without observable effect)
  for (int l = depth - 1; l >= 2; --l) {
    std::vector<int64_t> parents;
    for (int64_t n = t.level_ptr[l]; n < t.level_ptr[l + 1]; ++n)
      if (!is_leaf(n) && up_owner[n] == rank) parents.push_back(n);
    if (!parents.empty()) m2m_levels.push_back(m2m_tiles(parents));
  }
  if (world > 1) {
    // the nodes spanning ranks, recomputed by every rank after the exchange (children first)
    for (int l = depth - 1; l >= 2; --l) {
      std::vector<int64_t> parents;
      for (int64_t n = t.level_ptr[l]; n < t.level_ptr[l + 1]; ++n)
        if (!is_leaf(n) && up_owner[n] < 0) parents.push_back(n);
      if (!parents.empty()) m2m_top.push_back(m2m_tiles(parents));
    }
    // all-gather layout: every rank ships its export rows in a slot of x_max rows; this rank scatters the
    // other ranks' rows into M (and, on the tcgen05 path, their fp16 split)
    x_max = int(halo.max_export);
    std::vector<int> mine, rows, src;
    for (int r = 0; r < world; ++r)
      for (int64_t i = halo.export_ptr[r]; i < halo.export_ptr[r + 1]; ++i) {
        if (r == rank) {
          mine.push_back(int(halo.export_idx[i]));
        } else {
          rows.push_back(int(halo.export_idx[i]));
          src.push_back(r * x_max + int(i - halo.export_ptr[r]));
        }
      }
    x_mine = int(mine.size());
    x_total = int(rows.size());
    x_my_rows.upload(mine, &dev_bytes);
    x_rows.upload(rows, &dev_bytes);
    x_rank.upload(src, &dev_bytes);
    x_send.alloc(size_t(std::max(1, x_max)) * np * es, &dev_bytes);
    x_recv.alloc(size_t(std::max(1, x_max)) * np * es * world, &dev_bytes);
    KIFMM_CUDA(cudaMemset(x_recv.p, 0, x_recv.bytes));  // a host-exchange plan's warm-up imports zeros
    info.halo_rows_max = x_max;
    info.halo_rows_mine = x_mine;
    if (o.exchange == 0) {
      if (!o.nccl_unique_id) throw InvalidArgument("gpu: world_size > 1 needs nccl_unique_id (or exchange = 1)");
      ncclUniqueId id;
      std::memcpy(&id, o.nccl_unique_id, sizeof(id));
      ncclComm_t c;
      Nccl& nc_ = Nccl::get();
      nc_.check(nc_.commInitRank(&c, world, id, rank), "ncclCommInitRank");
      comm = c;
    } else if (o.exchange != 1) {
      throw InvalidArgument("gpu: exchange must be 0 (NCCL) or 1 (host)");
    }
  }

  m2m_scratch.alloc(size_t(std::max<int64_t>(1, m2m_scratch_rows)) * np * es, &dev_bytes);

  ptick("M2M");
  // ---- P2L check works: active nodes with X members
  {
    std::vector<CheckWork> w;
    std::vector<int2> rg;
    for (int64_t n = 0; n < nn; ++n) {
      if (!active[n] || t.x_ptr[n] == t.x_ptr[n + 1]) continue;
      const int r0 = int(rg.size());
      for (int64_t e = t.x_ptr[n]; e < t.x_ptr[n + 1]; ++e) {
        const int64_t a = t.x_idx[e];
        rg.push_back(make_int2(int(t.leaf_ptr[a]), int(t.leaf_ptr[a + 1] - t.leaf_ptr[a])));
        info.p2l_pairs += (t.leaf_ptr[a + 1] - t.leaf_ptr[a]) * ne;
      }
      w.push_back({int(n), int(n), r0, int(rg.size()), rg[r0].x, rg[r0].y, node_lvl(n), 0});
    }
    n_p2l = int(w.size());
    if (check_hw) {  // half-warp check kernel: pair works of similar source counts in a warp
      auto srcs = [&](const CheckWork& c) {
        int64_t n = 0;
        for (int r = c.range_begin; r < c.range_end; ++r) n += rg[r].y;
        return n;
      };
      std::vector<std::pair<int64_t, int>> key(w.size());
      for (size_t i = 0; i < w.size(); ++i) key[i] = {-srcs(w[i]), int(i)};
      std::stable_sort(key.begin(), key.end());
      std::vector<CheckWork> sorted(w.size());
      for (size_t i = 0; i < w.size(); ++i) sorted[i] = w[key[i].second];
      w.swap(sorted);
    }
    p2l_works.upload(w, &dev_bytes);
    p2l_ranges.upload(rg, &dev_bytes);
  }

  ptick("P2L");
  // ---- M2L tiles: active targets at level >= 2 grouped by (level, octant), Z-order inside
  std::vector<std::vector<int64_t>> m2l_groups;
  {
    std::map<std::array<int, 3>, std::vector<int64_t>> groups;
    // boundary class of a target: which domain faces its parent touches (those V offsets are absent).
    // 0 = interior; else 1 + 2 a + side for the first axis a whose parent coordinate is on a face --
    // a face group collects the face rows with the edge / corner rows whose tap sets are subsets of it,
    // so its tiles need (almost) no zero rows (KIFMM_M2L_CLASSES=1; measured more padded slots at
    // config 2, 7.87 M vs 7.11 M: the extra partial tiles cost more than the tighter tap sets save)
    bool by_class = false;
    if (const char* e = std::getenv("KIFMM_M2L_CLASSES")) by_class = std::atoi(e) != 0;
    auto bclass = [&](int64_t n) {
      const int l = node_lvl(n);
      if (!by_class || l < 3) return 0;
      const auto pa = key_anchor(t.node_key[t.node_parent[n]]);
      const uint32_t hi = (uint32_t(1) << (l - 1)) - 1;
      for (int a = 0; a < 3; ++a) {
        if (pa[a] == 0) return 1 + 2 * a;
        if (pa[a] == hi) return 2 + 2 * a;
      }
      return 0;
    };
    // levels with few targets are one group (octant classes would each fill a fraction of a tile with
    // zero rows); larger levels are split by octant (shared transfer-vector sets)
    std::map<int, int64_t> per_level;
    for (int64_t n = 0; n < nn; ++n)
      if (active[n] && node_lvl(n) >= 2 && t.v_ptr[n] != t.v_ptr[n + 1]) ++per_level[node_lvl(n)];
    for (int64_t n = 0; n < nn; ++n) {
      if (!active[n] || node_lvl(n) < 2 || t.v_ptr[n] == t.v_ptr[n + 1]) continue;
      const int lvl = node_lvl(n);
      const bool small = per_level[lvl] <= 2048;
      groups[{lvl, small ? 0 : key_octant(t.node_key[n]), small ? 0 : bclass(n)}].push_back(n);
      info.m2l_pairs += t.v_ptr[n + 1] - t.v_ptr[n];
    }
    for (auto& kv : groups) m2l_groups.push_back(kv.second);
  }
  m2l_backend = 1;
  if (o.m2l_backend == 2 || (o.m2l_backend == 0 && precision == 32 && tc_m2l_np_supported(np) && m2l_tc_available())) {
    if (precision != 32) throw InvalidArgument("gpu: tcgen05 3xTF32 M2L is an fp32 path");
    m2l_tc.build(t, m2l_groups, np, ops, &dev_bytes, /*own_split=*/!gemm_tc);
    m2l_backend = m2l_tc.f16 ? 2 : 3;  // 2: kind::f16 3-term split, 3: kind::tf32 3xTF32
    info.m2l_padded_pairs = m2l_tc.slots;
  }
  if (o.m2l_backend == 4 && precision != 64) throw InvalidArgument("gpu: the int8 (Ozaki) M2L is an fp64 path");
  if (precision == 64 &&
      (o.m2l_backend == 4 || (o.m2l_backend == 0 && M2LOzPlan::supported(np) && m2l_tc_available()))) {
    if (!M2LOzPlan::supported(np)) throw InvalidArgument("gpu: the int8 (Ozaki) M2L needs n_e padded to 160 or 224");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    m2l_oz.build(t, m2l_groups, np, ops, nn, node_lvl, depth, sms, &dev_bytes);
    m2l_backend = 4;
    info.m2l_padded_pairs = m2l_oz.slots;
  }
  if (m2l_backend == 1) {
    std::vector<TileSpec> tiles;
    for (auto& grp : m2l_groups) {
      for (size_t s0 = 0; s0 < grp.size(); s0 += bm_m2l) {
        TileSpec ts;
        ts.out.assign(bm_m2l, -1);
        std::map<int, std::vector<int>> taps;
        for (int r = 0; r < bm_m2l && s0 + r < grp.size(); ++r) {
          const int64_t b = grp[s0 + r];
          ts.out[r] = int(b);
          for (int64_t e = t.v_ptr[b]; e < t.v_ptr[b + 1]; ++e) {
            auto& v = taps[t.v_tv[e]];
            if (v.empty()) v.assign(bm_m2l, -1);
            v[r] = int(t.v_idx[e]);
          }
        }
        for (auto& kv : taps) ts.segs.push_back({kv.first, kv.second});
        tiles.push_back(std::move(ts));
      }
    }
    // split each tile's taps into pieces (~8 per SM-slot in total) so small trees still fill the GPU;
    // piece partials land in scratch rows and are summed per tile in fixed order (m2l_reduce)
    int64_t total_segs = 0;
    for (auto& ts : tiles) total_segs += int64_t(ts.segs.size());
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int64_t chunk = std::max<int64_t>(8, (total_segs + 16 * sms - 1) / (16 * sms));
    std::vector<TileSpec> pieces;
    std::vector<int> red_out, red_slot{0};
    for (auto& ts : tiles) {
      const int64_t ns = int64_t(ts.segs.size());
      const int64_t np_ = std::max<int64_t>(1, (ns + chunk - 1) / chunk);
      for (int64_t pc = 0; pc < np_; ++pc) {
        TileSpec piece;
        const int64_t a = ns * pc / np_, b = ns * (pc + 1) / np_;
        const int slot = int(pieces.size());
        piece.out.resize(bm_m2l);
        for (int r = 0; r < bm_m2l; ++r) piece.out[r] = slot * bm_m2l + r;
        piece.segs.assign(ts.segs.begin() + a, ts.segs.begin() + b);
        pieces.push_back(std::move(piece));
      }
      red_out.insert(red_out.end(), ts.out.begin(), ts.out.end());
      red_slot.push_back(int(pieces.size()));
    }
    // most expensive pieces first (better tail on the block scheduler); slots keep the reduction order
    std::stable_sort(pieces.begin(), pieces.end(),
                     [](const TileSpec& x, const TileSpec& y) { return x.segs.size() > y.segs.size(); });
    m2l.build(pieces, bm_m2l, &dev_bytes);
    m2l_red_tiles = int(tiles.size());
    m2l_red_out.upload(red_out, &dev_bytes);
    m2l_red_slot.upload(red_slot, &dev_bytes);
    m2l_partial.alloc(std::max<size_t>(1, pieces.size()) * bm_m2l * np * esz(), &dev_bytes);
    info.m2l_padded_pairs = m2l.slots;
  }

  ptick("M2L");
  // ---- downward solves over active nodes at level >= 2 (slots -> tmp rows)
  std::vector<int64_t> dn_nodes;
  for (int64_t n = 0; n < nn; ++n)
    if (active[n] && node_lvl(n) >= 2) dn_nodes.push_back(n);
  {
    std::vector<int> extra;  // P2L rows outside every M2L tile (M2L tiles cover exactly the nonempty V lists)
    for (int64_t n : dn_nodes)
      if (t.v_ptr[n] == t.v_ptr[n + 1] && t.x_ptr[n] != t.x_ptr[n + 1]) extra.push_back(int(n));
    n_dn_extra = int(extra.size());
    dn_extra.upload(extra, &dev_bytes);
  }
  {
    std::vector<TileSpec> a, b;
    for (size_t s0 = 0; s0 < dn_nodes.size(); s0 += ld_tiles) {
      TileSpec x, y;
      std::vector<int> slots(ld_tiles, -1), nodes(ld_tiles, -1);
      for (int r = 0; r < ld_tiles && s0 + r < dn_nodes.size(); ++r) {
        slots[r] = int(s0 + r);
        nodes[r] = int(dn_nodes[s0 + r]);
      }
      x.out = slots;
      x.segs.push_back({0, nodes});
      y.out = nodes;
      y.segs.push_back({0, slots});
      a.push_back(x);
      b.push_back(y);
    }
    if (gemm_tc) {
      std::vector<double> b1, b2;
      factored_b(ops.dc2e_u, ops.dc2e_s, ops.dc2e_v, ops.dc2e_rank, b1, b2);
      tg_dn1.build(a, b1, 1, np, &dev_bytes);
      // rows of the deepest level start at dn_nodes[k] (level-major order); tiles of the second solve are
      // cut there so the upper levels' rows finish first
      size_t k = 0;
      while (k < dn_nodes.size() && node_lvl(dn_nodes[k]) < depth) ++k;
      dn_split = depth >= 4 && k > 0 && k < dn_nodes.size();
      if (const char* e = std::getenv("KIFMM_DN_SPLIT")) dn_split = dn_split && std::atoi(e) != 0;
      if (dn_split) {
        dn_split_level = depth;
        std::vector<TileSpec> bu, bl;
        for (size_t s0 = 0; s0 < dn_nodes.size();) {
          const size_t e0 = std::min(dn_nodes.size(), s0 < k ? std::min(k, s0 + ld_tiles) : s0 + ld_tiles);
          TileSpec y;
          std::vector<int> slots(ld_tiles, -1), nodes(ld_tiles, -1);
          for (size_t r = s0; r < e0; ++r) {
            slots[r - s0] = int(r);
            nodes[r - s0] = int(dn_nodes[r]);
          }
          y.out = nodes;
          y.segs.push_back({0, slots});
          (s0 < k ? bu : bl).push_back(std::move(y));
          s0 = e0;
        }
        tg_dn2_up.build(bu, b2, 1, np, &dev_bytes);
        tg_dn2_lo.build(bl, b2, 1, np, &dev_bytes, TcGemm::min_ctas(int(bl.size())));
      } else {
        tg_dn2.build(b, b2, 1, np, &dev_bytes);
      }
    } else {
      solve_dn1.build(a, ld_tiles, &dev_bytes);
      solve_dn2.build(b, ld_tiles, &dev_bytes);
    }
  }
  const int64_t tmp_rows = std::max<int64_t>({int64_t(1), le - lb, int64_t(dn_nodes.size())});
  tmp.alloc(size_t(tmp_rows) * np * es, &dev_bytes);
  if (gemm_tc) {
    sp_tmp.alloc(int(tmp_rows), np, &dev_bytes);
    sp_M.alloc(int(nn), np, &dev_bytes);
    sp_cd.alloc(int(nn), np, &dev_bytes);
    sp_L.alloc(int(nn), np, &dev_bytes);
  }
  const std::vector<double> b_l2l = gemm_tc ? octant_b(ops.l2l) : std::vector<double>();

  ptick("down solves");
  // ---- L2L per level: active children at l+1 (l >= 2), grouped by octant
  for (int l = 2; l < depth; ++l) {
    std::vector<TileSpec> tiles;
    for (int oc = 0; oc < 8; ++oc) {
      std::vector<int64_t> ch;
      for (int64_t n = t.level_ptr[l + 1]; n < t.level_ptr[l + 2]; ++n)
        if (active[n] && key_octant(t.node_key[n]) == oc) ch.push_back(n);
      for (size_t s0 = 0; s0 < ch.size(); s0 += ld_tiles) {
        TileSpec ts;
        ts.out.assign(ld_tiles, -1);
        std::vector<int> in(ld_tiles, -1);
        for (int r = 0; r < ld_tiles && s0 + r < ch.size(); ++r) {
          ts.out[r] = int(ch[s0 + r]);
          in[r] = int(t.node_parent[ch[s0 + r]]);
        }
        ts.segs.push_back({oc, in});
        tiles.push_back(std::move(ts));
      }
    }
    if (!tiles.empty()) {
      auto g = std::make_unique<L2LLevel>();
      if (gemm_tc) {
        g->tc.build(tiles, b_l2l, 8, np, &dev_bytes);
        g->r0 = int(t.level_ptr[l]);
        g->r1 = int(t.level_ptr[l + 1]);
      } else {
        g->tiles.build(tiles, ld_tiles, &dev_bytes);
      }
      l2l_levels.push_back(std::move(g));
    }
  }

  ptick("L2L");
  // ---- leaf works, <= 128 targets per work, staged in rounds:
  //      near plan = self + U-list particles (runs on the side stream from the start),
  //      far plan  = L2P + M2P surfaces (after L2L; accumulates into the near result)
  // fp32: packed two-targets-per-thread kernel (KIFMM_P2P=scalar selects the scalar one)
  {
    const char* e = std::getenv("KIFMM_P2P");
    leaf_packed = precision == 32 && !(e && std::string(e) == "scalar");
  }
  const bool packed = leaf_packed;
  // fp64: the scalar near field slows the int8 M2L more than it gains next to it (config 4: 101 ms serial,
  // 105 ms on the side stream); fp32 keeps its queue-mode side blocks (config 2: 1.20 vs 1.46 ms serial)
  near_serial = precision == 64;
  near_pair64 = precision == 64;
  if (const char* e = std::getenv("KIFMM_NEAR_PAIR64")) near_pair64 = precision == 64 && std::atoi(e) != 0;
  if (const char* e = std::getenv("KIFMM_NEAR_SERIAL")) near_serial = std::atoi(e) != 0;
  if (packed) {
    if (const char* e = std::getenv("KIFMM_NEAR_WS")) near_ws = std::atoi(e);
    if (near_ws) near_bps = near_ws_bps;
    if (const char* e = std::getenv("KIFMM_NEAR_BPS")) near_bps = std::max(0, std::atoi(e));
    near_counter.alloc(4 * sizeof(int), &dev_bytes);
#ifdef KIFMM_EXPERIMENTS  // timing experiments only (tools/build_variant.sh); NEAR_SKIP gives wrong results
    if (const char* e = std::getenv("KIFMM_NEAR_PAUSE")) near_pause = std::atoi(e);
    near_debug = std::getenv("KIFMM_NEAR_DEBUG") != nullptr;
    near_skip = std::getenv("KIFMM_NEAR_SKIP") != nullptr;
    if (const char* e = std::getenv("KIFMM_NEAR_FORK")) {
      const std::string v(e);
      near_fork_at = v == "m2l" ? 1 : v == "check" ? 2 : v == "m2m" ? 3 : 0;
    }
    near_corun = std::getenv("KIFMM_NEAR_CORUN") != nullptr;
#endif
    // full shared-memory carveout, so an SM running near-field blocks need not drain before a tcgen05
    // CTA (which needs the maximum carveout) can start next to them
    for (const void* f : {(const void*)leaf_eval_f2_kernel<true, false, true, false>,
                          (const void*)leaf_eval_f2_kernel<false, false, true, false>,
                          (const void*)leaf_eval_f2_kernel<true, false, true, true>,
                          (const void*)leaf_eval_f2_kernel<false, false, true, true>,
                          (const void*)near_ws_kernel<true, 0>, (const void*)near_ws_kernel<true, 1>,
                          (const void*)near_ws_kernel<true, 2>, (const void*)near_ws_kernel<false, 0>,
                          (const void*)near_ws_kernel<false, 1>, (const void*)near_ws_kernel<false, 2>,
                          (const void*)leaf_eval_f2_kernel<true, false, false>,
                          (const void*)leaf_eval_f2_kernel<false, false, false>})
      KIFMM_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int nb = 0;
    KIFMM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, near_ws_kernel<true, 2>, kNearWsThreads, 0));
    near_ws_blocks = std::max(1, nb);
  }
  auto build_leaf_plan = [&](bool near_part, LeafPlan& lp) {
    struct Src {
      int kind, a, len;
    };
    // leaves in chunks built in parallel (local works / rounds / items), then concatenated in order
    struct Part {
      std::vector<LeafWork> w;
      std::vector<int4> rounds, items;
      int64_t near_pairs = 0, l2p_pairs = 0, m2p_pairs = 0;
    };
    constexpr int64_t kChunk = 2048;
    const int64_t nparts = (le - lb + kChunk - 1) / kChunk;
    std::vector<Part> parts(size_t(std::max<int64_t>(nparts, 0)));
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t pi = 0; pi < nparts; ++pi) {
    Part& P = parts[pi];
    std::vector<LeafWork>& w = P.w;
    std::vector<int4>& rounds = P.rounds;
    std::vector<int4>& items = P.items;
    for (int64_t l = lb + pi * kChunk; l < std::min(le, lb + (pi + 1) * kChunk); ++l) {
      const int64_t node = t.leaf_node[l];
      std::vector<Src> self, other;
      const int64_t ntl = t.leaf_ptr[l + 1] - t.leaf_ptr[l];
      if (near_part) {
        int64_t src_cnt = 0;
        self.push_back({kSrcSelf, int(t.leaf_ptr[l]), int(ntl)});
        int cur_b = -1, cur_e = -1;  // U ranges, merged when contiguous in the reordered buffer
        for (int64_t e = t.u_ptr[l]; e < t.u_ptr[l + 1]; ++e) {
          const int64_t s2 = t.u_idx[e];
          const int b = int(t.leaf_ptr[s2]), en = int(t.leaf_ptr[s2 + 1]);
          src_cnt += en - b;
          if (s2 == l) continue;
          if (b == cur_e) {
            cur_e = en;
          } else {
            if (cur_b >= 0) other.push_back({kSrcParticles, cur_b, cur_e - cur_b});
            cur_b = b;
            cur_e = en;
          }
        }
        if (cur_b >= 0) other.push_back({kSrcParticles, cur_b, cur_e - cur_b});
        P.near_pairs += ntl * src_cnt;
      } else {
        if (node_lvl(node) >= 2) {
          other.push_back({kSrcL2P, int(node), ne});
          P.l2p_pairs += ntl * ne;
        }
        for (int64_t e = t.w_ptr[l]; e < t.w_ptr[l + 1]; ++e) {
          other.push_back({kSrcM2P, int(t.w_idx[e]), ne});
          P.m2p_pairs += ntl * ne;
        }
        if (other.empty()) continue;
      }
      // block geometry: <= 128 targets, leaf_slices source slices, rounds of <= kP2PCap sources; two
      // targets per thread for the packed fp32 kernels and the fp64 pair kernel (near field)
      const int chunk = kP2PThreads;
      const bool pairs = packed || (near_part && near_pair64);
      for (int64_t t0 = t.leaf_ptr[l]; t0 < t.leaf_ptr[l + 1]; t0 += chunk) {
        const int nt = int(std::min<int64_t>(chunk, t.leaf_ptr[l + 1] - t0));
        const int R = leaf_slices(nt, pairs), q = leaf_unroll(pairs) * R;
        const int cap = kP2PCap - kP2PCap % q;
        const int rb = int(rounds.size());
        size_t si = 0, oi = 0;
        int soff = 0, ooff = 0;  // offsets inside the current self / other source
        while (si < self.size() || oi < other.size()) {
          const int ib = int(items.size());
          int ns = 0, no = 0;
          while (si < self.size() && ns < cap) {  // self section first
            const Src& x = self[si];
            const int take = std::min(x.len - soff, cap - ns);
            items.push_back(make_int4(x.kind, x.a + soff, take, ns));
            ns += take;
            soff += take;
            if (soff == x.len) {
              ++si;
              soff = 0;
            }
          }
          const int S = (ns + q - 1) / q * q;
          while (oi < other.size() && S + no < cap) {
            const Src& x = other[oi];
            const int take = std::min(x.len - ooff, cap - S - no);
            if (x.kind == kSrcParticles)
              items.push_back(make_int4(x.kind, x.a + ooff, take, S + no));
            else
              items.push_back(make_int4(x.kind | (ooff << 4), x.a, take, S + no));
            no += take;
            ooff += take;
            if (ooff == x.len) {
              ++oi;
              ooff = 0;
            }
          }
          const int O = (no + q - 1) / q * q;
          rounds.push_back(make_int4(ib, int(items.size()), S | (ns << 16), O | (no << 16)));
        }
        const int TT = packed ? (nt + 2 * kNearNPair - 1) / (2 * kNearNPair) : pairs ? (nt + 1) / 2 : nt;
        w.push_back({int(l), int(t0), nt, rb, int(rounds.size()), R | (TT << 8), (65536 + TT - 1) / TT,
                     (65536 + R - 1) / R});
      }
    }
    }
    std::vector<LeafWork> w;
    std::vector<int4> rounds, items;
    for (auto& P : parts) {
      const int rb = int(rounds.size()), ib = int(items.size());
      for (LeafWork x : P.w) {
        x.round_begin += rb;
        x.round_end += rb;
        w.push_back(x);
      }
      for (int4 r : P.rounds) {
        r.x += ib;
        r.y += ib;
        rounds.push_back(r);
      }
      items.insert(items.end(), P.items.begin(), P.items.end());
      info.near_pairs += P.near_pairs;
      info.l2p_pairs += P.l2p_pairs;
      info.m2p_pairs += P.m2p_pairs;
    }
    lp.n = int(w.size());
    lp.works.upload(w, &dev_bytes);
    lp.rounds.upload(rounds, &dev_bytes);
    lp.items.upload(items, &dev_bytes);
  };
  build_leaf_plan(true, leaf_near);
  ptick("near-field plan");
  if (const char* e = std::getenv("KIFMM_FAR")) far_as_leaf = packed && std::string(e) == "leaf";
  if (far_as_leaf) build_leaf_plan(false, leaf_far);  // experiments: far field on the block kernel
  // far field: one warp-work per owned leaf with any L2P / M2P surface
  far_packed = packed && ne <= kFarMaxNe;  // the packed fp32 kernels stage whole surfaces (p <= 7)
  {
    std::vector<int4> fw;
    std::vector<FarWork> fw2;
    std::vector<int2> sf;
    for (int64_t l = lb; l < le; ++l) {
      const int64_t node = t.leaf_node[l];
      const int b = int(sf.size());
      const int64_t ntl = t.leaf_ptr[l + 1] - t.leaf_ptr[l];
      if (node_lvl(node) >= 2) {
        sf.push_back(make_int2(int(node), kSrcL2P));
        info.l2p_pairs += ntl * ne;
      }
      for (int64_t e = t.w_ptr[l]; e < t.w_ptr[l + 1]; ++e) {
        sf.push_back(make_int2(int(t.w_idx[e]), kSrcM2P));
        info.m2p_pairs += ntl * ne;
      }
      // <= 32 targets per warp; the packed fp32 kernel has a work for every owned leaf (it also
      // writes the final output), the scalar kernel only for leaves with far sources
      const int chunk = 32;  // packed: 16 target pairs x 2 slices fill the warp
      const int e = int(sf.size());
      for (int64_t t0 = t.leaf_ptr[l]; t0 < t.leaf_ptr[l + 1]; t0 += chunk) {
        const int cnt = int(std::min<int64_t>(chunk, t.leaf_ptr[l + 1] - t0));
        if (far_packed)
          fw2.push_back({int(t0), cnt, b, e, e > b ? sf[b].x : 0, e > b ? sf[b].y : 0, 0, 0});
        else if (e > b)
          fw.push_back(make_int4(int(t0), b, e, cnt));
      }
    }
    far_hw = far_packed && ne <= 4 * (kFarHwSlot / 4);
    if (const char* e = std::getenv("KIFMM_FAR_HW")) far_hw = far_hw && std::atoi(e) != 0;
    // Long works (many M2P surfaces, adaptive trees) are cut into chunks of <= far_chunk surfaces: a
    // half-warp walks one work's surfaces in sequence, so the longest work bounds the kernel (config 3:
    // 41 surfaces, against 19 per resident half-warp on average).  Chunks write partial sums to far_part
    // slots (FarWork.pad0 = slot + 1); far_combine_kernel adds them in chunk order to the near field
    // and writes the output.
    // Measured (config 3): 1.312 ms unchunked, 1.217 / 1.210 / 1.213 ms with chunks of 6 / 8 / 12, 1.231 with
    // the mean surfaces per resident half-warp (19); config 5 is unchanged (118 ms).  KIFMM_FAR_CHUNK=0: off.
    far_chunk = 0;
    if (far_hw) {
      far_chunk = 12;
      if (const char* e = std::getenv("KIFMM_FAR_CHUNK")) far_chunk = std::atoi(e);
    }
    std::vector<int4> groups;  // {t0, count, first slot, n chunks}
    if (far_chunk > 0) {
      std::vector<FarWork> out;
      int slots = 0;
      for (const FarWork& w : fw2) {
        const int nsf = w.surf_end - w.surf_begin;
        if (nsf <= far_chunk) {
          out.push_back(w);
          continue;
        }
        const int nch = (nsf + far_chunk - 1) / far_chunk;
        groups.push_back(make_int4(w.t0, w.count, slots, nch));
        for (int c = 0; c < nch; ++c) {
          const int b = w.surf_begin + c * far_chunk, e = std::min(w.surf_end, b + far_chunk);
          out.push_back({w.t0, w.count, b, e, sf[b].x, sf[b].y, slots + c + 1, 0});
        }
        slots += nch;
      }
      fw2.swap(out);
      n_far_groups = int(groups.size());
      if (slots) {
        far_part.alloc(size_t(slots) * 32 * sizeof(float4), &dev_bytes);
        far_groups.upload(groups, &dev_bytes);
      }
    }
    n_far = int(far_packed ? fw2.size() : fw.size());
    // half-warp kernel: a warp's two works loop to the longer surface list -- pair works of equal
    // surface counts (stable sort by count; every work writes only its own targets, order is free)
    if (far_hw && far_packed)  // equal (surface count, source slices) in the two halves of a warp
      std::stable_sort(fw2.begin(), fw2.end(), [](const FarWork& a, const FarWork& b) {
        const int na = a.surf_end - a.surf_begin, nb = b.surf_end - b.surf_begin;
        if (na != nb) return na > nb;
        return far_hw_slices(a.count) < far_hw_slices(b.count);
      });
    if (far_packed)
      far_works.upload(fw2, &dev_bytes);
    else
      far_works.upload(fw, &dev_bytes);
    far_surfaces.upload(sf, &dev_bytes);
    std::vector<int64_t> lp(t.leaf_ptr, t.leaf_ptr + nl + 1);
    leaf_ptr_dev.upload(lp, &dev_bytes);
  }

  // call structure (SPEC acceptance #8)
  {
    std::set<int> m2m_lv, m2l_lv, l2l_lv;
    for (const auto* lvs : {&m2m_levels, &m2m_top})
      for (const auto& g : *lvs) m2m_lv.insert(g->level);
    for (const auto& g : m2l_groups)
      for (int64_t n : g) m2l_lv.insert(node_lvl(n));
    for (int l = 2; l < depth; ++l)
      for (int64_t n = t.level_ptr[l + 1]; n < t.level_ptr[l + 2]; ++n)
        if (active[n]) {
          l2l_lv.insert(l + 1);
          break;
        }
    info.m2m_levels = int(m2m_lv.size());
    info.m2l_levels = int(m2l_lv.size());
    info.m2l_launch_levels = m2l_lv.empty() ? 0 : 1;  // every M2L level in one batched launch
    info.l2l_levels = int(l2l_lv.size());
    info.p2m_leaves = n_p2m;
    info.p2l_nodes = n_p2l;
    for (int64_t l = lb; l < le; ++l) {
      ++info.near_leaves;
      info.l2p_leaves += node_lvl(t.leaf_node[l]) >= 2;
      info.m2p_leaves += t.w_ptr[l + 1] != t.w_ptr[l];
    }
  }
  info.n_particles = N;
  info.n_leaves = nl;
  info.n_nodes = nn;
  info.owned_leaf_begin = lb;
  info.owned_leaf_end = le;
  info.owned_particle_begin = pb;
  info.owned_particle_end = pe;
  info.n_e = ne;
  info.n_c = nc;
  info.ne_pad = np;
  info.m2l_backend = m2l_backend;
  ptick("far-field plan");
  KIFMM_CUDA(cudaDeviceSynchronize());
  ptick("device sync");
  info.device_bytes = int64_t(dev_bytes);
}

// Multi-GPU exchange: this rank's export rows -> x_send; all-gather (NCCL, or the caller in
// host mode); the other ranks' rows x_recv -> M (+ fp16 split).
void kifmm_gpu_plan::gather_exports(cudaStream_t s) {
  if (x_mine <= 0) return;
  if (precision == 32)
    gather_rows_kernel<float><<<x_mine, 128, 0, s>>>(M.as<float>(), np, x_my_rows.as<int>(), x_mine, x_send.as<float>());
  else
    gather_rows_kernel<double><<<x_mine, 128, 0, s>>>(M.as<double>(), np, x_my_rows.as<int>(), x_mine, x_send.as<double>());
  KIFMM_LAUNCH_CHECK();
}

void kifmm_gpu_plan::allgather(cudaStream_t s) {
  Nccl& n = Nccl::get();
  n.check(n.allGather(x_send.p, x_recv.p, size_t(std::max(1, x_max)) * np,
                      precision == 32 ? ncclFloat32 : ncclFloat64, static_cast<ncclComm_t>(comm), s),
          "ncclAllGather");
}

void kifmm_gpu_plan::scatter_imports(cudaStream_t s) {
  if (x_total <= 0) return;
  if (precision == 32 && gemm_tc) {
    tc_dispatch_np(np, [&](auto w) {
      scatter_rows_split_kernel<decltype(w)::value><<<unsigned((x_total + 7) / 8), 256, 0, s>>>(
          x_recv.as<float>(), x_rows.as<int>(), x_rank.as<int>(), x_total, M.as<float>(), sp_M.hi, sp_M.lo, sp_M.un);
    });
  } else if (precision == 32) {
    scatter_rows_kernel<float><<<x_total, 128, 0, s>>>(x_recv.as<float>(), np, x_rows.as<int>(), x_rank.as<int>(),
                                                       x_total, M.as<float>());
  } else {
    scatter_rows_kernel<double><<<x_total, 128, 0, s>>>(x_recv.as<double>(), np, x_rows.as<int>(),
                                                        x_rank.as<int>(), x_total, M.as<double>());
  }
  KIFMM_LAUNCH_CHECK();
}

template <class T>
void kifmm_gpu_plan::run(cudaStream_t s, bool input_order, bool timed, int phase) {
  constexpr int BMB = sizeof(T) == 4 ? 128 : 64;
  constexpr int TMB = sizeof(T) == 4 ? 8 : 4;
  int ei = (phase & 1) ? 0 : 3;  // event slots of the phase-2 marks stay the same
  auto mark = [&]() {
    if (timed) KIFMM_CUDA(cudaEventRecord(ev[ei++], s));
  };
  int launches = 0;
  const P2PParams<T> pp{src4.as<v4_t<T>>(), node_geom.as<v4_t<T>>(), surface.as<T>(), ne, np, T(alpha_in),
                        T(alpha_out), node_lo.as<v4_t<T>>()};
  auto gemm = [&](const GemmTiles& tl, const T* X, const T* W, T* Y, bool acc, bool m2l_shape) {
    if (tl.n_tiles == 0) return;
    GemmArgs<T> a{};
    a.X = X;
    a.ldx = np;
    a.W = W;
    a.ldw = np;
    a.K = np;
    a.Y = Y;
    a.ldy = np;
    a.accumulate = acc ? 1 : 0;
    if (m2l_shape)
      launch_gemm<T, KIFMM_M2L_SIMT_BM, (sizeof(T) == 8 ? KIFMM_M2L_SIMT_TM64 : 4)>(np, tl, a, s);
    else
      launch_gemm<T, BMB, TMB>(np, tl, a, s);
    ++launches;
  };
  T* Mp = M.as<T>();
  T* Lp = L.as<T>();
  auto leaf = [&](const LeafPlan& lp, bool acc, cudaStream_t st) {
    if (!lp.n) return;
    const LeafWork* w = lp.works.as<LeafWork>();
    const int4* r = lp.rounds.as<int4>();
    const int4* it = lp.items.as<int4>();
    T* g = grad ? grad_buf.as<T>() : nullptr;
    if constexpr (sizeof(T) == 4) {
      if (leaf_packed && near_ws >= 2 && &lp == &leaf_near && !acc) {  // standalone persistent near field
        int* qc = near_counter.as<int>();
        KIFMM_CUDA(cudaMemsetAsync(qc, 0, 4 * sizeof(int), st));
        const int grid = std::min(lp.n, near_ws_blocks * sm_count());
        if (grad)
          near_ws_kernel<true, 0><<<grid, kNearWsThreads, 0, st>>>(pp, w, r, it, pot.as<T>(), g, lp.n, qc);
        else
          near_ws_kernel<false, 0><<<grid, kNearWsThreads, 0, st>>>(pp, w, r, it, pot.as<T>(), g, lp.n, qc);
        KIFMM_LAUNCH_CHECK();
        ++launches;
        return;
      }
      if (leaf_packed) {
        if (grad && acc)
          leaf_eval_f2_kernel<true, true><<<lp.n, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pot.as<T>(), g);
        else if (grad)
          leaf_eval_f2_kernel<true, false><<<lp.n, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pot.as<T>(), g);
        else if (acc)
          leaf_eval_f2_kernel<false, true><<<lp.n, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pot.as<T>(), g);
        else
          leaf_eval_f2_kernel<false, false><<<lp.n, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pot.as<T>(), g);
        KIFMM_LAUNCH_CHECK();
        ++launches;
        return;
      }
    }
    if (near_pair64 && &lp == &leaf_near && !acc) {  // fp64 near field, two targets per thread
      if (grad)
        leaf_eval_pair_kernel<T, true, false><<<lp.n, kP2PThreads, 0, st>>>(pp, w, r, it, pot.as<T>(), g);
      else
        leaf_eval_pair_kernel<T, false, false><<<lp.n, kP2PThreads, 0, st>>>(pp, w, r, it, pot.as<T>(), g);
      KIFMM_LAUNCH_CHECK();
      ++launches;
      return;
    }
    if (grad && acc)
      leaf_eval_kernel<T, true, true><<<lp.n, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pot.as<T>(), g);
    else if (grad)
      leaf_eval_kernel<T, true, false><<<lp.n, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pot.as<T>(), g);
    else if (acc)
      leaf_eval_kernel<T, false, true><<<lp.n, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pot.as<T>(), g);
    else
      leaf_eval_kernel<T, false, false><<<lp.n, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pot.as<T>(), g);
    KIFMM_LAUNCH_CHECK();
    ++launches;
  };

  const bool up = (phase & 1) != 0, down = (phase & 2) != 0;
  if (up) {
    mark();  // 0
    // zero the down-check rows here, not just before P2L / M2L: a memset between the M2M and M2L kernels
    // would break their programmatic (PDL) launch edge
    if (!(gemm_tc && m2l_backend == 2 && !n_p2l && world == 1))  // else nothing reads the fp32 check rows
      KIFMM_CUDA(cudaMemsetAsync(check_dn.p, 0, check_dn.bytes, s));
    pack_sources_kernel<T><<<int(ceil_div(N, 256)), 256, 0, s>>>(pos4.as<v4_t<T>>(), q_in.as<T>(),
                                                                 input_order ? perm.as<int>() : nullptr, int(N),
                                                                 src4.as<v4_t<T>>());
    KIFMM_LAUNCH_CHECK();
    ++launches;
  }
  // near field has no dependency on the tree passes: fork it onto the low-priority side stream --
  // either all of it, or (queue mode, fp32) a few blocks per SM that run next to the tensor-core tree
  // kernels and take works from a shared counter, drained by a full launch after L2L
  // (KIFMM_NEAR_CORUN: experiments -- the timed run co-runs the near field with M2L to time M2L under load)
  const bool corun = timed && near_corun && leaf_packed;
  const bool queue_mode = (!timed || corun) && !near_serial && leaf_packed && near_bps > 0 && leaf_near.n && !near_skip;
  auto near_queue = [&](cudaStream_t st, int grid, bool drain) {
    if constexpr (sizeof(T) == 4) {
      const LeafWork* w = leaf_near.works.as<LeafWork>();
      const int4* r = leaf_near.rounds.as<int4>();
      const int4* it = leaf_near.items.as<int4>();
      float* g = grad ? grad_buf.as<float>() : nullptr;
      int* qc = near_counter.as<int>();
      float* pt = pot.as<float>();
      const int n = leaf_near.n;
      if (near_ws) {
        if (grad && drain)
          near_ws_kernel<true, 2><<<grid, kNearWsThreads, 0, st>>>(pp, w, r, it, pt, g, n, qc);
        else if (grad)
          near_ws_kernel<true, 1><<<grid, kNearWsThreads, 0, st>>>(pp, w, r, it, pt, g, n, qc);
        else if (drain)
          near_ws_kernel<false, 2><<<grid, kNearWsThreads, 0, st>>>(pp, w, r, it, pt, g, n, qc);
        else
          near_ws_kernel<false, 1><<<grid, kNearWsThreads, 0, st>>>(pp, w, r, it, pt, g, n, qc);
        KIFMM_LAUNCH_CHECK();
        ++launches;
        return;
      }
      if (grad && drain)
        leaf_eval_f2_kernel<true, false, true, true><<<grid, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pt, g, n, qc);
      else if (grad)
        leaf_eval_f2_kernel<true, false, true, false><<<grid, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pt, g, n, qc);
      else if (drain)
        leaf_eval_f2_kernel<false, false, true, true><<<grid, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pt, g, n, qc);
      else
        leaf_eval_f2_kernel<false, false, true, false><<<grid, kP2PThreads, 0, st>>>(pp, w, r, it, Mp, Lp, pt, g, n, qc);
      KIFMM_LAUNCH_CHECK();
      ++launches;
    }
  };
  const bool near_fork = (!timed || corun) && !near_serial;  // near field on the side stream
  auto fork_near = [&]() {
    if (near_fork && leaf_near.n && !near_skip) {
      if (queue_mode) KIFMM_CUDA(cudaMemsetAsync(near_counter.p, 0, 4 * sizeof(int), s));
      KIFMM_CUDA(cudaEventRecord(ev_fork, s));
      KIFMM_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
      if (queue_mode)
        near_queue(side, std::min(leaf_near.n, near_bps * sm_count()), false);
      else
        leaf(leaf_near, false, side);
      KIFMM_CUDA(cudaEventRecord(ev_join, side));
    }
  };
  if (up && near_fork_at == 0 && !corun) fork_near();
  // upward: P2M check -> factored solve
  if (up && n_p2m) {
    launch_check<T>(np, n_p2m, pp, p2m_works.as<CheckWork>(), p2m_ranges.as<int2>(), node_level.as<int>(),
                    ref_level, T(alpha_out), check_up.as<T>(), s, gemm_tc ? &sp_cu : nullptr, check_hw);
    KIFMM_LAUNCH_CHECK();
    ++launches;
  }
  if (up && near_fork_at == 2 && !corun) fork_near();
  // tcgen05 GEMM: split the fp32 source rows, then dst (=/+=) A . B^T
  // tcgen05 GEMMs: the A rows arrive already split by their producer (check kernel, previous GEMM's
  // epilogue, M2M / M2L reductions); the epilogue writes the fp32 rows (Y, may be null) and their split
  auto tgemm = [&](const TcGemm& g, const TcSplit& a, T* Y, bool acc, const TcSplit* out_split) {
    if constexpr (sizeof(T) == 4) {
      if (!g.n_tiles) return;
      g.run(a, Y, acc, s, out_split);
      ++launches;
    }
  };
  if (up) {
    if (gemm_tc) {
      tgemm(tg_up1, sp_cu, nullptr, false, &sp_tmp);
      tgemm(tg_up2, sp_tmp, Mp, false, &sp_M);
    } else {
      gemm(solve_up1, check_up.as<T>(), w_us_u.as<T>(), tmp.as<T>(), false, true);
      gemm(solve_up2, tmp.as<T>(), w_vt_u.as<T>(), Mp, false, true);
    }
    mark();  // 1
  }
  // M2M, levels d-1 .. floor
  auto m2m_level = [&](const M2MLevel& lv) {
    if (gemm_tc && lv.direct) {
      tgemm(lv.tc, sp_M, Mp, false, &sp_M);
      return;
    }
    if (gemm_tc) {
      if constexpr (sizeof(T) == 4) {
        tgemm(lv.tc, sp_M, m2m_scratch.as<T>(), false, nullptr);
        tc_dispatch_np(np, [&](auto w) {
          launch_pdl(m2m_reduce_split_kernel<decltype(w)::value>, dim3(unsigned((lv.n + 7) / 8)), dim3(256), 0, s,
                     (const float*)m2m_scratch.as<float>(), (const int*)lv.parents.as<int>(),
                     (const int*)lv.masks.as<int>(), lv.n, Mp, sp_M.hi, sp_M.lo, sp_M.un);
        });
      }
    } else {
      gemm(lv.tiles, Mp, w_m2m.as<T>(), m2m_scratch.as<T>(), false, true);
      m2m_reduce_kernel<T><<<lv.n, 128, 0, s>>>(m2m_scratch.as<T>(), lv.parents.as<int>(), lv.masks.as<int>(), lv.n,
                                               np, Mp);
    }
    KIFMM_LAUNCH_CHECK();
    ++launches;
  };
  if (up) {
    for (auto& lv : m2m_levels) m2m_level(*lv);
    mark();  // 2
  }
  if (up && near_fork_at == 3 && !corun) fork_near();
  // multipole exchange (multi-GPU): export rows -> all-gather -> import rows (+ their fp16 split), then the
  // nodes spanning ranks, recomputed by every rank
  if (world > 1) {
    if (up) {
      gather_exports(s);
      launches += x_mine > 0;
      if (phase == 3 && opt.exchange == 0) {
        allgather(s);
        ++launches;
      }
    }
    if (down) {
      scatter_imports(s);
      launches += x_total > 0;
      for (auto& lv : m2m_top) m2m_level(*lv);
    }
  }
  if (!down) return;
  mark();  // 3
  // downward: P2L check into the down-check buffer (zeroed at the start of the evaluate)
  const bool p2l_side = !timed && n_p2l && p2l_overlap && gemm_tc && m2l_backend == 2 && sizeof(T) == 4;
  if (p2l_side) {
    KIFMM_CUDA(cudaEventRecord(ev_p2l_fork, s));
    KIFMM_CUDA(cudaStreamWaitEvent(side2, ev_p2l_fork, 0));
  }
  if (n_p2l) {
    launch_check<T>(np, n_p2l, pp, p2l_works.as<CheckWork>(), p2l_ranges.as<int2>(), node_level.as<int>(),
                    ref_level, T(alpha_in), check_dn.as<T>(), p2l_side ? side2 : s, nullptr, check_hw);
    KIFMM_LAUNCH_CHECK();
    ++launches;
  }
  if (p2l_side) KIFMM_CUDA(cudaEventRecord(ev_p2l_join, side2));
  mark();  // 4
#ifdef KIFMM_EXPERIMENTS
  if (const char* e = std::getenv("KIFMM_CORUN_DUMMY"); e && timed) {  // experiments: a dummy load next to M2L
    KIFMM_CUDA(cudaEventRecord(ev_fork, s));
    KIFMM_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
    dummy_load_kernel<<<2 * sm_count(), 128, 0, side>>>(std::atoi(e), 20000, pot.as<float>());
    KIFMM_CUDA(cudaEventRecord(ev_join, side));
  }
#endif
  if (near_fork_at == 1 || corun) fork_near();  // experiments (KIFMM_NEAR_FORK=m2l): near field next to M2L only
  if (queue_mode && near_pause)  // side near-field blocks sleep while M2L runs
    KIFMM_CUDA(cudaMemsetAsync(near_counter.as<int>() + 3, near_pause, 1, s));
  // M2L over all levels at once, accumulated as reference-level check potentials
  if (m2l_backend == 4) {
    if constexpr (sizeof(T) == 8) {
      m2l_oz.run(Mp, node_level.as<int>(), check_dn.as<T>(), s);
      launches += m2l_oz.launches();
    }
  } else if (m2l_backend >= 2) {
    if constexpr (sizeof(T) == 4) {
      if (gemm_tc && m2l_backend == 2) {  // multipoles already split; the reduce splits the check rows
        // no P2L rows: the fp32 check rows are never read (only their split) -- skip them entirely
        m2l_tc.launch_presplit_main(sp_M, s);
        if (p2l_side) KIFMM_CUDA(cudaStreamWaitEvent(s, ev_p2l_join, 0));
        m2l_tc.launch_presplit_reduce(n_p2l ? check_dn.as<float>() : nullptr, &sp_cd, s);
        launches += 2;
        if (n_dn_extra) {  // P2L-only check rows (no V list): split them here
          tc_dispatch_np(np, [&](auto w) {
            tc::split_f16_list_kernel<decltype(w)::value><<<unsigned((n_dn_extra + 7) / 8), 256, 0, s>>>(
                check_dn.as<float>(), dn_extra.as<int>(), n_dn_extra, sp_cd.hi, sp_cd.lo, sp_cd.un);
          });
          KIFMM_LAUNCH_CHECK();
          ++launches;
        }
      } else {
        m2l_tc.launch(Mp, check_dn.as<float>(), np, s);
        launches += m2l_tc.launches();
        if (gemm_tc) {
          sp_cd.split(check_dn.as<float>(), 0, int(nn), s);
          ++launches;
        }
      }
    }
  } else {
    gemm(m2l, Mp, w_m2l.as<T>(), m2l_partial.as<T>(), false, true);
    if (m2l_red_tiles) {
      reduce_partials_kernel<T><<<m2l_red_tiles, 256, 0, s>>>(m2l_partial.as<T>(), m2l_red_out.as<int>(),
                                                             m2l_red_slot.as<int>(), 64, np, check_dn.as<T>());
      KIFMM_LAUNCH_CHECK();
      ++launches;
    }
  }
  if (queue_mode && near_pause) KIFMM_CUDA(cudaMemsetAsync(near_counter.as<int>() + 3, 0, sizeof(int), s));
#ifdef KIFMM_EXPERIMENTS
  if (queue_mode && near_debug && std::getenv("KIFMM_NEAR_DEBUG_M2L"))  // experiments: snapshot after M2L
    KIFMM_CUDA(cudaMemcpyAsync(near_counter.as<int>() + 2, near_counter.as<int>(), sizeof(int),
                               cudaMemcpyDeviceToDevice, s));
#endif
  mark();  // 5
  // factored downward solve (dc2e at the reference level; M2L/P2L level factors folded)
  bool l2l_done = false;
  if (gemm_tc && dn_split) {
    if constexpr (sizeof(T) == 4) {
      tgemm(tg_dn1, sp_cd, nullptr, false, &sp_tmp);
      tgemm(tg_dn2_up, sp_tmp, Lp, false, &sp_L);
      // L2L into the upper levels on side2, next to the deepest level's second solve
      KIFMM_CUDA(cudaEventRecord(ev_dn_fork, s));
      KIFMM_CUDA(cudaStreamWaitEvent(side2, ev_dn_fork, 0));
      const size_t nl2l = l2l_levels.size();
      for (size_t i = 0; i + 1 < nl2l; ++i) {
        l2l_levels[i]->tc.run(sp_L, Lp, true, side2, &sp_L);
        ++launches;
      }
      KIFMM_CUDA(cudaEventRecord(ev_dn_join, side2));
      tgemm(tg_dn2_lo, sp_tmp, Lp, false, &sp_L);
      mark();  // 6
      KIFMM_CUDA(cudaStreamWaitEvent(s, ev_dn_join, 0));
      if (nl2l) tgemm(l2l_levels[nl2l - 1]->tc, sp_L, Lp, true, &sp_L);
      mark();  // 7
      l2l_done = true;
    }
  }
  if (!l2l_done) {
    if (gemm_tc) {
      tgemm(tg_dn1, sp_cd, nullptr, false, &sp_tmp);
      tgemm(tg_dn2, sp_tmp, Lp, false, &sp_L);
    } else {
      gemm(solve_dn1, check_dn.as<T>(), w_us_d.as<T>(), tmp.as<T>(), false, true);
      gemm(solve_dn2, tmp.as<T>(), w_vt_d.as<T>(), Lp, false, true);
    }
    mark();  // 6
    // L2L top-down
    for (auto& lv : l2l_levels) {
      if (gemm_tc)
        tgemm(lv->tc, sp_L, Lp, true, &sp_L);  // reads parent rows (level l), writes child rows (l + 1)
      else
        gemm(lv->tiles, Lp, w_l2l.as<T>(), Lp, true, true);
    }
    mark();  // 7
  }
  // leaves: near field (side stream, or here when timed) then L2P + M2P
  if (!near_fork) leaf(leaf_near, false, s);
#ifdef KIFMM_EXPERIMENTS
  if (queue_mode && near_debug && !std::getenv("KIFMM_NEAR_DEBUG_M2L"))  // experiments: works taken by now
    KIFMM_CUDA(cudaMemcpyAsync(near_counter.as<int>() + 2, near_counter.as<int>(), sizeof(int),
                               cudaMemcpyDeviceToDevice, s));
#endif
  // drain the works the side-stream blocks did not take (persistent: at most 8 blocks per SM, so an
  // empty queue costs one short wave instead of a block per leaf)
  if (queue_mode)
    near_queue(s,
               std::min(leaf_near.n, (near_ws ? near_ws_blocks : 8) * sm_count()),
               true);
  if (near_fork && leaf_near.n && !near_skip) KIFMM_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
  bool fused_out = false;  // the packed far kernel wrote the final (input-order) output
  if (far_as_leaf) leaf(leaf_far, true, s);
  if constexpr (sizeof(T) == 4) {
    if (far_packed && n_far && !far_as_leaf) {
      if (input_order && world > 1) {
        KIFMM_CUDA(cudaMemsetAsync(pot_out.p, 0, pot_out.bytes, s));
        if (grad) KIFMM_CUDA(cudaMemsetAsync(grad_out.p, 0, grad_out.bytes, s));
      }
      const int blocks = int(ceil_div(n_far, kFarWarps));
      float* g = grad ? grad_buf.as<float>() : nullptr;
      const int* pm = input_order ? perm.as<int>() : nullptr;
      float* go = grad ? grad_out.as<float>() : nullptr;
      const int hw_blocks = int(ceil_div(n_far, 2 * kFarWarps));
      float4* part = n_far_groups ? far_part.as<float4>() : nullptr;
      if (far_hw && grad)
        far_hw_kernel<true><<<hw_blocks, kFarWarps * 32, 0, s>>>(pp, far_works.as<FarWork>(), n_far,
                                                                 far_surfaces.as<int2>(), Mp, Lp, pot.as<float>(), g,
                                                                 pm, pot_out.as<float>(), go, part);
      else if (far_hw)
        far_hw_kernel<false><<<hw_blocks, kFarWarps * 32, 0, s>>>(pp, far_works.as<FarWork>(), n_far,
                                                                  far_surfaces.as<int2>(), Mp, Lp, pot.as<float>(), g,
                                                                  pm, pot_out.as<float>(), go, part);
      else if (grad)
        far_f2_kernel<true><<<blocks, kFarWarps * 32, 0, s>>>(pp, far_works.as<FarWork>(), n_far, far_surfaces.as<int2>(),
                                                              Mp, Lp, pot.as<float>(), g, pm, pot_out.as<float>(), go);
      else
        far_f2_kernel<false><<<blocks, kFarWarps * 32, 0, s>>>(pp, far_works.as<FarWork>(), n_far,
                                                               far_surfaces.as<int2>(), Mp, Lp, pot.as<float>(), g, pm,
                                                               pot_out.as<float>(), go);
      if (far_hw && n_far_groups) {  // targets of the long works cut into surface chunks
        KIFMM_LAUNCH_CHECK();
        ++launches;
        if (grad)
          far_combine_kernel<true><<<unsigned(ceil_div(int64_t(n_far_groups) * 32, 256)), 256, 0, s>>>(
              far_groups.as<int4>(), n_far_groups, part, pot.as<float>(), g, pm, pot_out.as<float>(), go);
        else
          far_combine_kernel<false><<<unsigned(ceil_div(int64_t(n_far_groups) * 32, 256)), 256, 0, s>>>(
              far_groups.as<int4>(), n_far_groups, part, pot.as<float>(), g, pm, pot_out.as<float>(), go);
      }
      KIFMM_LAUNCH_CHECK();
      ++launches;
      fused_out = true;
    }
  }
  if (!fused_out && n_far && !far_as_leaf) {
    const int blocks = int(ceil_div(n_far, kFarWarps));
    T* g = grad ? grad_buf.as<T>() : nullptr;
    if (grad)
      far_kernel<T, true><<<blocks, kFarWarps * 32, 0, s>>>(pp, far_works.as<int4>(), n_far, far_surfaces.as<int2>(),
                                                           leaf_ptr_dev.as<int64_t>(), Mp, Lp, pot.as<T>(), g);
    else
      far_kernel<T, false><<<blocks, kFarWarps * 32, 0, s>>>(pp, far_works.as<int4>(), n_far, far_surfaces.as<int2>(),
                                                            leaf_ptr_dev.as<int64_t>(), Mp, Lp, pot.as<T>(), g);
    KIFMM_LAUNCH_CHECK();
    ++launches;
  }
  mark();  // 8
  if (input_order && !fused_out) {
    if (world > 1) {
      KIFMM_CUDA(cudaMemsetAsync(pot_out.p, 0, pot_out.bytes, s));
      if (grad) KIFMM_CUDA(cudaMemsetAsync(grad_out.p, 0, grad_out.bytes, s));
    }
    const int cnt = int(pe - pb);
    if (cnt > 0) {
      unpermute_kernel<T><<<int(ceil_div(cnt, 256)), 256, 0, s>>>(pot.as<T>(), perm.as<int>(), int(pb), int(pe), 1,
                                                                  pot_out.as<T>());
      ++launches;
      if (grad) {
        unpermute_kernel<T><<<int(ceil_div(cnt, 256)), 256, 0, s>>>(grad_buf.as<T>(), perm.as<int>(), int(pb),
                                                                    int(pe), 3, grad_out.as<T>());
        ++launches;
      }
      KIFMM_LAUNCH_CHECK();
    }
  }
  mark();  // 9
  if (phase == 3) info.kernel_launches = launches;
}

void kifmm_gpu_plan::evaluate_device(const void* q, void* pot_dst, void* grad_dst, bool input_order,
                                     cudaStream_t user, bool timed) {
  KIFMM_CUDA(cudaSetDevice(device));
  cudaStream_t s = user ? user : stream;
  const size_t es = esz();
  require_single_call();
  begin(s);
  KIFMM_CUDA(cudaMemcpyAsync(q_in.p, q, size_t(N) * es, cudaMemcpyDefault, s));
  if (!timed && opt.use_graph) {
    launch_graph(input_order, s);
  } else {
    if (precision == 32)
      run<float>(s, input_order, timed);
    else
      run<double>(s, input_order, timed);
  }
  copy_out(pot_dst, grad_dst, input_order, s);
  finish(s);
}

namespace {
template <class T>
void direct_impl(int device, const T* pos, const T* q, int64_t n, const int64_t* targets, int64_t m, T* pot, T* grad) {
  KIFMM_CUDA(cudaSetDevice(device));
  std::vector<T> s4(size_t(n) * 4);
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < 3; ++d) s4[4 * i + d] = pos[3 * i + d];
    s4[4 * i + 3] = q[i];
  }
  std::vector<int64_t> tg(targets, targets + m);
  size_t dummy = 0;
  DevMem d_src, d_tg, d_pot, d_grad;
  d_src.upload(s4, &dummy);
  d_tg.upload(tg, &dummy);
  d_pot.alloc(size_t(m) * sizeof(T), &dummy);
  if (grad) d_grad.alloc(size_t(m) * 3 * sizeof(T), &dummy);
  const int blocks = int(ceil_div(m, kP2PThreads));
  if (grad)
    direct_kernel<T, true><<<blocks, kP2PThreads>>>(d_src.as<v4_t<T>>(), n, d_tg.as<int64_t>(), m, d_pot.as<T>(),
                                                    d_grad.as<T>());
  else
    direct_kernel<T, false><<<blocks, kP2PThreads>>>(d_src.as<v4_t<T>>(), n, d_tg.as<int64_t>(), m, d_pot.as<T>(),
                                                     nullptr);
  KIFMM_LAUNCH_CHECK();
  KIFMM_CUDA(cudaMemcpy(pot, d_pot.p, size_t(m) * sizeof(T), cudaMemcpyDeviceToHost));
  if (grad) KIFMM_CUDA(cudaMemcpy(grad, d_grad.p, size_t(m) * 3 * sizeof(T), cudaMemcpyDeviceToHost));
}

template <class T>
double fma_peak_impl(int device) {
  KIFMM_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  KIFMM_CUDA(cudaGetDeviceProperties(&prop, device));
  DevMem out;
  size_t dummy = 0;
  out.alloc(64, &dummy);
  const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = sizeof(T) == 4 ? 16384 : 2048;
  cudaEvent_t a, b;
  KIFMM_CUDA(cudaEventCreate(&a));
  KIFMM_CUDA(cudaEventCreate(&b));
  fma_probe_kernel<T><<<blocks, threads>>>(out.as<T>(), iters / 4, T(0.999), T(1e-3));
  KIFMM_CUDA(cudaEventRecord(a));
  fma_probe_kernel<T><<<blocks, threads>>>(out.as<T>(), iters, T(0.999), T(1e-3));
  KIFMM_CUDA(cudaEventRecord(b));
  KIFMM_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  KIFMM_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return double(blocks) * threads * iters * 8 * 2 / (ms * 1e-3);
}
}  // namespace

// Many right-hand sides through one plan, software-pipelined over three streams: the H2D copy of
// charges k+1 (copy-in stream) and the D2H copy of results k-1 (copy-out stream) run under the
// evaluate of k (plan stream).  Device staging is double-buffered; the plan's own input / output
// buffers are filled and drained with device-to-device copies on the plan stream (~7 us per
// evaluate at config 2), so the captured graph is the same one evaluate() launches.
void kifmm_gpu_plan::evaluate_many(int n_rhs, const void* const* charges, void* const* potentials,
                                   void* const* gradients, bool input_order) {
  KIFMM_CUDA(cudaSetDevice(device));
  const size_t es = esz();
  if (!pipe) {
    auto P = std::make_unique<Pipe>();
    KIFMM_CUDA(cudaStreamCreateWithFlags(&P->cin, cudaStreamNonBlocking));
    KIFMM_CUDA(cudaStreamCreateWithFlags(&P->cout, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      for (cudaEvent_t* e : {&P->in_ready[b], &P->in_free[b], &P->out_ready[b], &P->out_free[b]})
        KIFMM_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      P->q[b].alloc(size_t(N) * es, &dev_bytes);
      P->pot[b].alloc(size_t(N) * es, &dev_bytes);
      if (grad) P->grad[b].alloc(size_t(N) * 3 * es, &dev_bytes);
    }
    pipe = std::move(P);
  }
  Pipe& P = *pipe;
  require_single_call();
  begin(stream);
  const bool full = input_order || world == 1;  // else: this rank's particle range (reordered order)
  const size_t off = full ? 0 : size_t(pb), cnt = full ? size_t(N) : size_t(pe - pb);
  const void* ps = input_order ? pot_out.p : pot.p;
  const void* gs = input_order ? grad_out.p : grad_buf.p;
  for (int k = 0; k < n_rhs; ++k) {
    const int b = k & 1;
    // copy-in: charges k into staging b once the evaluate of k-2 has consumed it
    if (k >= 2) KIFMM_CUDA(cudaStreamWaitEvent(P.cin, P.in_free[b], 0));
    KIFMM_CUDA(cudaMemcpyAsync(P.q[b].p, charges[k], size_t(N) * es, cudaMemcpyDefault, P.cin));
    KIFMM_CUDA(cudaEventRecord(P.in_ready[b], P.cin));
    // evaluate k on the plan stream
    KIFMM_CUDA(cudaStreamWaitEvent(stream, P.in_ready[b], 0));
    KIFMM_CUDA(cudaMemcpyAsync(q_in.p, P.q[b].p, size_t(N) * es, cudaMemcpyDeviceToDevice, stream));
    KIFMM_CUDA(cudaEventRecord(P.in_free[b], stream));
    if (opt.use_graph) {
      launch_graph(input_order, stream);
    } else if (precision == 32) {
      run<float>(stream, input_order, false);
    } else {
      run<double>(stream, input_order, false);
    }
    if (k >= 2) KIFMM_CUDA(cudaStreamWaitEvent(stream, P.out_free[b], 0));  // results k-2 have left staging b
    if (cnt) {
      KIFMM_CUDA(cudaMemcpyAsync(static_cast<char*>(P.pot[b].p) + off * es, static_cast<const char*>(ps) + off * es,
                                 cnt * es, cudaMemcpyDeviceToDevice, stream));
      if (grad && gradients && gradients[k])
        KIFMM_CUDA(cudaMemcpyAsync(static_cast<char*>(P.grad[b].p) + 3 * off * es,
                                   static_cast<const char*>(gs) + 3 * off * es, 3 * cnt * es, cudaMemcpyDeviceToDevice,
                                   stream));
    }
    KIFMM_CUDA(cudaEventRecord(P.out_ready[b], stream));
    // copy-out: results k to the caller's buffers
    KIFMM_CUDA(cudaStreamWaitEvent(P.cout, P.out_ready[b], 0));
    if (cnt) {
      KIFMM_CUDA(cudaMemcpyAsync(static_cast<char*>(potentials[k]) + off * es,
                                 static_cast<const char*>(P.pot[b].p) + off * es, cnt * es, cudaMemcpyDefault, P.cout));
      if (grad && gradients && gradients[k])
        KIFMM_CUDA(cudaMemcpyAsync(static_cast<char*>(gradients[k]) + 3 * off * es,
                                   static_cast<const char*>(P.grad[b].p) + 3 * off * es, 3 * cnt * es,
                                   cudaMemcpyDefault, P.cout));
    }
    KIFMM_CUDA(cudaEventRecord(P.out_free[b], P.cout));
  }
  KIFMM_CUDA(cudaStreamWaitEvent(stream, P.out_free[(n_rhs + 1) & 1], 0));  // the last copy-outs
  if (n_rhs > 1) KIFMM_CUDA(cudaStreamWaitEvent(stream, P.out_free[n_rhs & 1], 0));
  finish(stream);
  KIFMM_CUDA(cudaStreamSynchronize(P.cout));
  KIFMM_CUDA(cudaStreamSynchronize(stream));
}

// ====================================================================== ABI
extern "C" {

kifmm_status kifmm_gpu_plan_create(const kifmm_gpu_options* options, const kifmm_tree_view* tree,
                                   const kifmm_operator_view* ops, kifmm_gpu_plan** out) {
  return guard([&] {
    if (!options || !tree || !ops || !out) throw InvalidArgument("plan_create: null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw DeviceError(KIFMM_E_CUDA, "plan_create: no CUDA device available (the library has no CPU fallback)");
    if (options->device < 0 || options->device >= ndev) throw InvalidArgument("plan_create: bad device ordinal");
    auto p = std::make_unique<kifmm_gpu_plan>();
    p->build(*options, *tree, *ops);
    // one untimed warm-up pass (sets kernel attributes, validates every launch)
    KIFMM_CUDA(cudaMemsetAsync(p->q_in.p, 0, p->q_in.bytes, p->stream));
    if (p->precision == 32)
      p->run<float>(p->stream, false, false);
    else
      p->run<double>(p->stream, false, false);
    KIFMM_CUDA(cudaStreamSynchronize(p->stream));
    *out = p.release();
  });
}

kifmm_status kifmm_gpu_evaluate_many(kifmm_gpu_plan* p, int32_t n_rhs, const void* const* charges,
                                     void* const* potentials, void* const* gradients, int32_t input_order) {
  return guard([&] {
    if (!p || n_rhs < 0 || (n_rhs > 0 && (!charges || !potentials)))
      throw InvalidArgument("evaluate_many: null argument or negative count");
    for (int k = 0; k < n_rhs; ++k)
      if (!charges[k] || !potentials[k]) throw InvalidArgument("evaluate_many: null charges / potential buffer");
    p->evaluate_many(n_rhs, charges, potentials, gradients, input_order != 0);
  });
}

kifmm_status kifmm_gpu_evaluate(kifmm_gpu_plan* p, const void* charges, void* potential, void* gradient,
                                int32_t input_order, kifmm_gpu_timings* timings) {
  return guard([&] {
    if (!p || !charges || !potential) throw InvalidArgument("evaluate: null argument");
    p->require_single_call();
    KIFMM_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    const size_t es = p->esz();
    auto& ev = p->ev;
    p->begin(s);
    // events 10..13: H2D, compute, D2H boundaries
    KIFMM_CUDA(cudaEventRecord(ev[10], s));
    KIFMM_CUDA(cudaMemcpyAsync(p->q_in.p, charges, size_t(p->N) * es, cudaMemcpyDefault, s));
    KIFMM_CUDA(cudaEventRecord(ev[11], s));
    const bool timed = timings != nullptr;
    if (!timed && p->opt.use_graph) {
      p->launch_graph(input_order != 0, s);
    } else if (p->precision == 32) {
      p->run<float>(s, input_order != 0, timed);
    } else {
      p->run<double>(s, input_order != 0, timed);
    }
    KIFMM_CUDA(cudaEventRecord(ev[12], s));
#ifdef KIFMM_EXPERIMENTS
    if (std::getenv("KIFMM_TIMELINE")) {
      unsigned long long tl[16][2];
      KIFMM_CUDA(cudaStreamSynchronize(s));
      KIFMM_CUDA(cudaMemcpyFromSymbol(tl, g_timeline, sizeof(tl)));
      unsigned long long t0 = ~0ull;
      for (auto& r : tl)
        if (r[1]) t0 = std::min(t0, r[0]);
      const char* names[] = {"", "m2l", "tc-gemms", "near-side", "near-drain", "far", "", "", "", "", "", "", "", "",
                             "", ""};
      if (tl[9][0] > tl[8][0])
        std::fprintf(stderr, "timeline m2l CTA 0 SM clock %.0f MHz\n",
                     double(tl[9][1] - tl[8][1]) / double(tl[9][0] - tl[8][0]) * 1e3);
      for (int i = 0; i < 8; ++i)
        if (tl[i][1])
          std::fprintf(stderr, "timeline %-10s start %8.1f us  end %8.1f us\n", names[i], (tl[i][0] - t0) * 1e-3,
                       (tl[i][1] - t0) * 1e-3);
      unsigned long long init[16][2];
      for (auto& r : init) {
        r[0] = ~0ull;
        r[1] = 0;
      }
      KIFMM_CUDA(cudaMemcpyToSymbol(g_timeline, init, sizeof(init)));
      int on = 1;
      KIFMM_CUDA(cudaMemcpyToSymbol(g_timeline_on, &on, sizeof(on)));
    }
    if (p->near_debug && p->near_counter.p) {
      int c[3];
      KIFMM_CUDA(cudaMemcpyAsync(c, p->near_counter.p, sizeof(c), cudaMemcpyDeviceToHost, s));
      KIFMM_CUDA(cudaStreamSynchronize(s));
      std::fprintf(stderr, "near queue: %d of %d works taken before the drain\n", c[2], p->leaf_near.n);
    }
#endif
    p->copy_out(potential, gradient, input_order != 0, s);
    KIFMM_CUDA(cudaEventRecord(ev[13], s));
    p->finish(s);
    KIFMM_CUDA(cudaStreamSynchronize(s));
    if (timed) {
      kifmm_gpu_timings t{};
      auto el = [&](int a, int b) {
        float ms = 0;
        KIFMM_CUDA(cudaEventElapsedTime(&ms, ev[a], ev[b]));
        return ms;
      };
      t.upload_ms = el(10, 11);
      t.p2m_ms = el(0, 1);
      t.m2m_ms = el(1, 2);
      t.exchange_ms = el(2, 3);
      t.p2l_ms = el(3, 4);
      t.m2l_ms = el(4, 5);
      t.down_solve_ms = el(5, 6);
      t.l2l_ms = el(6, 7);
      t.leaf_ms = el(7, 8);
      t.total_ms = el(0, 9);
      t.download_ms = el(12, 13);
      p->last = t;
      *timings = t;
    }
  });
}

kifmm_status kifmm_gpu_evaluate_device(kifmm_gpu_plan* p, const void* d_charges, void* d_potential,
                                       void* d_gradient, int32_t input_order, void* stream) {
  return guard([&] {
    if (!p || !d_charges) throw InvalidArgument("evaluate_device: null argument");
    p->evaluate_device(d_charges, d_potential, d_gradient, input_order != 0, static_cast<cudaStream_t>(stream), false);
  });
}

kifmm_status kifmm_gpu_evaluate_upward(kifmm_gpu_plan* p, const void* charges, int32_t input_order,
                                       void* export_rows) {
  return guard([&] {
    if (!p || !charges) throw InvalidArgument("evaluate_upward: null argument");
    if (p->world < 2 || p->opt.exchange != 1)
      throw InvalidArgument("evaluate_upward: needs a multi-rank plan with exchange = 1 (host)");
    if (p->x_max > 0 && !export_rows) throw InvalidArgument("evaluate_upward: null export buffer");
    KIFMM_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    const size_t es = p->esz();
    p->begin(s);
    KIFMM_CUDA(cudaMemcpyAsync(p->q_in.p, charges, size_t(p->N) * es, cudaMemcpyDefault, s));
    p->host_phase_input_order = input_order != 0;
    KIFMM_CUDA(cudaEventRecord(p->ev_half[0], s));
    if (p->precision == 32)
      p->run<float>(s, input_order != 0, false, 1);
    else
      p->run<double>(s, input_order != 0, false, 1);
    KIFMM_CUDA(cudaEventRecord(p->ev_half[1], s));
    if (p->x_mine > 0)
      KIFMM_CUDA(cudaMemcpyAsync(export_rows, p->x_send.p, size_t(p->x_mine) * p->np * es, cudaMemcpyDefault, s));
    p->finish(s);
    KIFMM_CUDA(cudaStreamSynchronize(s));
    KIFMM_CUDA(cudaEventElapsedTime(&p->last.upward_ms, p->ev_half[0], p->ev_half[1]));
  });
}

kifmm_status kifmm_gpu_evaluate_downward(kifmm_gpu_plan* p, const void* gathered, void* potential, void* gradient) {
  return guard([&] {
    if (!p || !potential) throw InvalidArgument("evaluate_downward: null argument");
    if (p->world < 2 || p->opt.exchange != 1)
      throw InvalidArgument("evaluate_downward: needs a multi-rank plan with exchange = 1 (host)");
    if (p->x_max > 0 && !gathered) throw InvalidArgument("evaluate_downward: null gathered buffer");
    KIFMM_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    const size_t es = p->esz();
    const bool io = p->host_phase_input_order;
    p->begin(s);
    if (p->x_max > 0)
      KIFMM_CUDA(cudaMemcpyAsync(p->x_recv.p, gathered, size_t(p->world) * p->x_max * p->np * es, cudaMemcpyDefault,
                                 s));
    KIFMM_CUDA(cudaEventRecord(p->ev_half[0], s));
    if (p->precision == 32)
      p->run<float>(s, io, false, 2);
    else
      p->run<double>(s, io, false, 2);
    KIFMM_CUDA(cudaEventRecord(p->ev_half[1], s));
    p->copy_out(potential, gradient, io, s);
    p->finish(s);
    KIFMM_CUDA(cudaStreamSynchronize(s));
    KIFMM_CUDA(cudaEventElapsedTime(&p->last.downward_ms, p->ev_half[0], p->ev_half[1]));
  });
}

kifmm_status kifmm_gpu_plan_get_info(const kifmm_gpu_plan* p, kifmm_gpu_plan_info* info) {
  return guard([&] {
    if (!p || !info) throw InvalidArgument("plan_get_info: null argument");
    *info = p->info;
  });
}

kifmm_status kifmm_gpu_last_timings(kifmm_gpu_plan* p, kifmm_gpu_timings* t) {
  return guard([&] {
    if (!p || !t) throw InvalidArgument("last_timings: null argument");
    *t = p->last;
  });
}

void kifmm_gpu_plan_destroy(kifmm_gpu_plan* p) { delete p; }

kifmm_status kifmm_gpu_nccl_unique_id(void* out128) {
  return guard([&] {
    if (!out128) throw InvalidArgument("nccl_unique_id: null out");
    Nccl& n = Nccl::get();
    ncclUniqueId id;
    n.check(n.getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
  });
}

kifmm_status kifmm_gpu_direct(int32_t precision, int32_t device, const void* positions, const void* charges,
                              int64_t n, const int64_t* targets, int64_t m, void* potential, void* gradient) {
  return guard([&] {
    if (!positions || !charges || !targets || !potential || n < 1 || m < 0)
      throw InvalidArgument("gpu_direct: bad argument");
    if (m == 0) return;
    if (precision == 32)
      direct_impl<float>(device, static_cast<const float*>(positions), static_cast<const float*>(charges), n, targets,
                         m, static_cast<float*>(potential), static_cast<float*>(gradient));
    else if (precision == 64)
      direct_impl<double>(device, static_cast<const double*>(positions), static_cast<const double*>(charges), n,
                          targets, m, static_cast<double*>(potential), static_cast<double*>(gradient));
    else
      throw InvalidArgument("gpu_direct: precision must be 32 or 64");
  });
}

kifmm_status kifmm_gpu_fma_peak(int32_t device, int32_t precision, double* flops) {
  return guard([&] {
    if (!flops) throw InvalidArgument("fma_peak: null out");
    *flops = precision == 64 ? fma_peak_impl<double>(device) : fma_peak_impl<float>(device);
  });
}

}  // extern "C"
