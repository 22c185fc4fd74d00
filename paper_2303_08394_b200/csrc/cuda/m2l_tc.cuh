// M2L on the 5th-generation tensor cores: tcgen05 kind::tf32 with 3xTF32 error
// compensation (SURVEY 7.3 "M2L batching").
//
// Work: for a tile of 128 same-class target nodes and one transfer vector t,
//   D[128 x 160] += A_t[128 x 160] . K_t^T,   A_t rows = multipoles of the V-list
// sources at offset t (zero rows where absent), K_t = reference-level kernel
// matrix (n_c x n_e, K-major).  fp32 operands are split x = hi + lo with hi the
// round-to-nearest tf32 value, and D += A_hi B_hi + A_hi B_lo + A_lo B_hi keeps
// fp32-level accuracy (the dropped A_lo B_lo term is ~2^-22 relative).
//
// CTA (6 warps, one work item = tile x tap chunk, accumulator in TMEM):
//   warp 0   : TMEM alloc/dealloc; lane 0 streams B_hi/B_lo K-blocks with TMA
//              (SWIZZLE_128B, 160 rows x 128 B per operand per stage)
//   warp 1   : lane 0 issues tcgen05.mma (M=128, N=160, K=8) and commits stages
//   warps 2-5: gather A_hi/A_lo rows with cp.async into the SW128 K-major layout
//   warps 6-13: per-tap promotion -- each tap accumulates in a fresh TMEM buffer
//              (two alternate), drained with tcgen05.ld into fp32 registers; the
//              tensor-core accumulator is not IEEE round-to-nearest and its bias
//              grows with the accumulation length (measured: 1.2e-6 at 1 tap,
//              1.5e-5 at 16, 1.5e-4 at 189 taps), so only one tap (K = 160) ever
//              accumulates in TMEM.
// Stages: (tap, 32-wide K block) pairs, 3-deep mbarrier ring (72 KB each).
// Partials of the tap chunks of a tile are summed by m2l_tc_reduce_kernel in a
// fixed order (deterministic; no atomics).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "common.cuh"

namespace kifmm {
namespace gpu {

namespace tc {

constexpr int BM = 128;          // target rows per tile (UMMA M)
constexpr int NP = 160;          // check points, padded (UMMA N); p = 6 only
constexpr int KB = 32;           // fp32 elements per 128-byte K block
constexpr int NKB = NP / KB;     // K blocks per tap (K = n_e padded = 160)
constexpr int STAGES = 3;
constexpr int A_BYTES = BM * 128;  // one operand K block: 16 KB
constexpr int B_BYTES = NP * 128;  // 20 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int EPI_WARPS = 8;                 // 2 per TMEM lane quarter, 80 columns each
constexpr int EPI_COLS = NP / 2;
constexpr int THREADS = (6 + EPI_WARPS) * 32;  // TMA, MMA, 4 A-producer warps, epilogue
constexpr uint32_t TMEM_COLS = 512;            // two 160-column accumulators at 0 and 256
// instruction descriptor: D f32 (bit 4), A/B tf32 (bits 7, 10), K-major, N>>3 at 17, M>>4 at 24
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(NP >> 3) << 17) | (uint32_t(BM >> 4) << 24);

struct Item {
  int tile, seg_begin, seg_end, slot;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1u << 28)) asm volatile("trap;");
  }
}

__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}

// SM100 UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);       // start address
  d |= uint64_t(1) << 16;                      // LBO (unused for swizzled K-major) = 16 B
  d |= uint64_t(1024 >> 4) << 32;              // SBO = 1024 B
  d |= uint64_t(1) << 46;                      // version (sm100)
  d |= uint64_t(2) << 61;                      // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    m2l_tc_kernel(const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_bhi_lo,
                  const Item* __restrict__ items, const int* __restrict__ seg_mat, const int* __restrict__ seg_in,
                  const float* __restrict__ m_hi, const float* __restrict__ m_lo, float* __restrict__ partial) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  // bars: [0,S) full, [S,2S) empty, [2S,2S+2) tmem_full[b], [2S+2,2S+4) tmem_empty[b]; then the TMEM address
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Item it = items[blockIdx.x];
  const int ntap = it.seg_end - it.seg_begin;
  const int nstage = ntap * NKB;
  const uint32_t sbase = smem_u32(smem);
  auto a_hi = [&](int s) { return sbase + s * STAGE_BYTES; };
  auto a_lo = [&](int s) { return sbase + s * STAGE_BYTES + A_BYTES; };
  auto b_hi = [&](int s) { return sbase + s * STAGE_BYTES + 2 * A_BYTES; };
  auto b_lo = [&](int s) { return sbase + s * STAGE_BYTES + 2 * A_BYTES + B_BYTES; };
  auto full = [&](int s) { return smem_u32(&bars[s]); };
  auto empty = [&](int s) { return smem_u32(&bars[STAGES + s]); };
  auto tfull = [&](int b) { return smem_u32(&bars[2 * STAGES + b]); };
  auto tempty = [&](int b) { return smem_u32(&bars[2 * STAGES + 2 + b]); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 128 + 1);  // 128 A-producer threads + the TMA arrive (with tx bytes)
      mbar_init(empty(s), 1);       // one tcgen05.commit per stage
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);                  // tcgen05.commit after the tap's last MMA
      mbar_init(tempty(b), EPI_WARPS * 32);    // every epilogue thread after draining
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_bhi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_bhi_lo) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- B producer (TMA)
    if (lane == 0) {
      for (int i = 0; i < nstage; ++i) {
        const int s = i % STAGES, round = i / STAGES;
        mbar_wait(empty(s), (round & 1) ^ 1);
        const int seg = it.seg_begin + i / NKB, kb = i % NKB;
        const int row = seg_mat[seg] * NP;
        mbar_expect_tx(full(s), 2 * B_BYTES);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
                "r"(b_hi(s)),
            "l"(&tm_bhi), "r"(full(s)), "r"(kb * KB), "r"(row)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
                "r"(b_lo(s)),
            "l"(&tm_bhi_lo), "r"(full(s)), "r"(kb * KB), "r"(row)
            : "memory");
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: one fresh TMEM accumulator per tap (buffers alternate)
    if (lane == 0) {
      for (int j = 0; j < ntap; ++j) {
        const int b = j & 1;
        mbar_wait(tempty(b), ((j >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem_base + uint32_t(b * 256);
        for (int kb = 0; kb < NKB; ++kb) {
          const int i = j * NKB + kb;
          const int s = i % STAGES, round = i / STAGES;
          mbar_wait(full(s), round & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int k = 0; k < KB / 8; ++k) {  // 4 x (K = 8 tf32 = 32 bytes) per 128-byte block
            const uint64_t dah = make_desc(a_hi(s) + 32 * k), dal = make_desc(a_lo(s) + 32 * k);
            const uint64_t dbh = make_desc(b_hi(s) + 32 * k), dbl = make_desc(b_lo(s) + 32 * k);
            mma_tf32(d, dah, dbh, (kb > 0 || k > 0) ? 1u : 0u);
            mma_tf32(d, dah, dbl, 1u);
            mma_tf32(d, dal, dbh, 1u);
          }
          mma_commit(empty(s));
        }
        mma_commit(tfull(b));
      }
    }
  } else if (warp < 6) {
    // ---------------- A producers: thread -> (16-byte chunk c, rows r0 + 16 j)
    const int t = threadIdx.x - 64;  // 0..127
    const int c = t & 7, r0 = t >> 3;
    int src[8];
    int cur_seg = -1;
    for (int i = 0; i < nstage; ++i) {
      const int s = i % STAGES, round = i / STAGES;
      const int seg = it.seg_begin + i / NKB, kb = i % NKB;
      if (seg != cur_seg) {
        cur_seg = seg;
#pragma unroll
        for (int j = 0; j < 8; ++j) src[j] = seg_in[size_t(seg) * BM + r0 + 16 * j];
      }
      mbar_wait(empty(s), (round & 1) ^ 1);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = r0 + 16 * j;
        const uint32_t off = uint32_t((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
        const size_t g = size_t(src[j] < 0 ? 0 : src[j]) * NP + kb * KB + c * 4;
        cp_async16_zfill(a_hi(s) + off, m_hi + g, src[j] >= 0);
        cp_async16_zfill(a_lo(s) + off, m_lo + g, src[j] >= 0);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      // publish the previous stage: its copies are complete once <= 1 group is pending
      if (i > 0) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(full((i - 1) % STAGES));
      }
    }
    if (nstage > 0) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(full((nstage - 1) % STAGES));
    }
  } else {
    // ---------------- epilogue: drain each tap's accumulator into fp32 registers (IEEE RN adds)
    // warp w reads TMEM lanes 32*(w%4).. (rows) and columns [h*80, h*80+80), h = (w-6)/4
    const int q = warp & 3, h = (warp - 6) >> 2;
    const int row = q * 32 + lane;
    float acc[EPI_COLS];
#pragma unroll
    for (int k = 0; k < EPI_COLS; ++k) acc[k] = 0.f;
    for (int j = 0; j < ntap; ++j) {
      const int b = j & 1;
      mbar_wait(tfull(b), (j >> 1) & 1);
      __syncwarp();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(b * 256 + h * EPI_COLS);
#pragma unroll
      for (int cb = 0; cb < EPI_COLS / 16; ++cb) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr + uint32_t(cb * 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[cb * 16 + k] += __uint_as_float(v[k]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(tempty(b));
    }
    float4* o4 = reinterpret_cast<float4*>(partial + (size_t(it.slot) * BM + row) * NP + h * EPI_COLS);
#pragma unroll
    for (int k = 0; k < EPI_COLS / 4; ++k) o4[k] = make_float4(acc[4 * k], acc[4 * k + 1], acc[4 * k + 2], acc[4 * k + 3]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// x = hi + lo with hi = tf32(x) (round to nearest, ties away), lo exact in fp32.
__global__ void split_tf32_kernel(const float* __restrict__ x, size_t n, float* __restrict__ hi, float* __restrict__ lo) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = x[i];
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
  const float hv = __uint_as_float(h);
  hi[i] = hv;
  lo[i] = v - hv;
}

// check[out(r)] += sum over the tile's items (fixed order) of partial[slot][r]
__global__ void m2l_tc_reduce_kernel(const float* __restrict__ partial, const int* __restrict__ tile_out,
                                     const int* __restrict__ tile_slot, float* __restrict__ check) {
  const int tile = blockIdx.x;
  const int s0 = tile_slot[tile], s1 = tile_slot[tile + 1];
  for (int idx = threadIdx.x; idx < BM * NP; idx += blockDim.x) {
    const int r = idx / NP, col = idx % NP;
    const int out = tile_out[size_t(tile) * BM + r];
    if (out < 0) continue;
    float acc = check[size_t(out) * NP + col];
    for (int s = s0; s < s1; ++s) acc += partial[(size_t(s) * BM + r) * NP + col];
    check[size_t(out) * NP + col] = acc;
  }
}

}  // namespace tc

inline bool m2l_tc_available() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0;
}

// Host side: tiles/items, split operators, TMA descriptors.
struct M2LTcPlan {
  int n_items = 0, n_tiles = 0, n_segs = 0;
  size_t nn = 0;
  float *d_khi = nullptr, *d_klo = nullptr, *d_mhi = nullptr, *d_mlo = nullptr, *d_partial = nullptr;
  int *d_tile_out = nullptr, *d_tile_slot = nullptr, *d_seg_mat = nullptr, *d_seg_in = nullptr;
  tc::Item* d_items = nullptr;
  CUtensorMap tm_hi{}, tm_lo{};
  int64_t slots = 0;

  ~M2LTcPlan() {
    for (void* p : {(void*)d_khi, (void*)d_klo, (void*)d_mhi, (void*)d_mlo, (void*)d_partial, (void*)d_tile_out,
                    (void*)d_tile_slot, (void*)d_seg_mat, (void*)d_seg_in, (void*)d_items})
      if (p) cudaFree(p);
  }
  int launches() const { return n_items ? 3 : 0; }

  template <class V>
  static void up(V** dst, const std::vector<V>& v, size_t* total) {
    KIFMM_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), std::max<size_t>(1, v.size()) * sizeof(V)));
    if (!v.empty()) KIFMM_CUDA(cudaMemcpy(*dst, v.data(), v.size() * sizeof(V), cudaMemcpyHostToDevice));
    *total += v.size() * sizeof(V);
  }

  static float tf32_rna(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xFFFFE000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
  }

  template <class TreeView, class OpsView>
  void build(const TreeView& t, const std::vector<std::vector<int64_t>>& groups, int np, const OpsView& ops,
             size_t* total) {
    if (np != tc::NP) throw InvalidArgument("tcgen05 M2L: only p = 6 (n_e padded to 160) is instantiated");
    nn = size_t(t.n_nodes);
    // ---- tiles (128 same-class targets) and their tap segments
    std::vector<int> tile_out, seg_mat, seg_in, tile_seg{0};
    for (const auto& grp : groups) {
      for (size_t s0 = 0; s0 < grp.size(); s0 += tc::BM) {
        std::vector<int> out(tc::BM, -1);
        std::map<int, std::vector<int>> taps;
        for (int r = 0; r < tc::BM && s0 + r < grp.size(); ++r) {
          const int64_t b = grp[s0 + r];
          out[r] = int(b);
          for (int64_t e = t.v_ptr[b]; e < t.v_ptr[b + 1]; ++e) {
            auto& v = taps[t.v_tv[e]];
            if (v.empty()) v.assign(tc::BM, -1);
            v[r] = int(t.v_idx[e]);
          }
        }
        tile_out.insert(tile_out.end(), out.begin(), out.end());
        for (auto& kv : taps) {
          seg_mat.push_back(kv.first);
          seg_in.insert(seg_in.end(), kv.second.begin(), kv.second.end());
        }
        tile_seg.push_back(int(seg_mat.size()));
      }
    }
    n_tiles = int(tile_seg.size()) - 1;
    n_segs = int(seg_mat.size());
    slots = int64_t(n_segs) * tc::BM;
    // ---- items: split each tile's taps into balanced chunks (~4 items per SM in total)
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t target_items = int64_t(4) * sms;
    int chunk = int(std::max<int64_t>(16, (n_segs + target_items - 1) / std::max<int64_t>(1, target_items)));
    if (const char* e = std::getenv("KIFMM_TC_CHUNK")) chunk = std::max(1, std::atoi(e));
    std::vector<tc::Item> items;
    std::vector<int> tile_slot{0};
    for (int ti = 0; ti < n_tiles; ++ti) {
      const int a = tile_seg[ti], b = tile_seg[ti + 1];
      const int pieces = std::max(1, (b - a + chunk - 1) / chunk);
      for (int pc = 0; pc < pieces; ++pc) {
        const int sa = a + int(int64_t(b - a) * pc / pieces), sb = a + int(int64_t(b - a) * (pc + 1) / pieces);
        items.push_back({ti, sa, sb, int(items.size())});
      }
      tile_slot.push_back(int(items.size()));
    }
    n_items = int(items.size());
    // launch order: longest items first (slots keep the fixed reduction order)
    std::stable_sort(items.begin(), items.end(), [](const tc::Item& x, const tc::Item& y) {
      return (x.seg_end - x.seg_begin) > (y.seg_end - y.seg_begin);
    });
    up(&d_tile_out, tile_out, total);
    up(&d_tile_slot, tile_slot, total);
    up(&d_seg_mat, seg_mat, total);
    up(&d_seg_in, seg_in, total);
    up(&d_items, items, total);
    // ---- K_t split into tf32 hi / lo, padded to 160 x 160 per transfer vector
    const int ne = ops.n_e, nc = ops.n_c, nt = ops.n_m2l;
    std::vector<float> khi(size_t(nt) * tc::NP * tc::NP, 0.f), klo(khi.size(), 0.f);
    for (int v = 0; v < nt; ++v)
      for (int c = 0; c < nc; ++c)
        for (int e = 0; e < ne; ++e) {
          const float x = float(ops.m2l[(size_t(v) * nc + c) * ne + e]);
          const float h = tf32_rna(x);
          const size_t idx = (size_t(v) * tc::NP + c) * tc::NP + e;
          khi[idx] = h;
          klo[idx] = x - h;
        }
    up(&d_khi, khi, total);
    up(&d_klo, klo, total);
    KIFMM_CUDA(cudaMalloc(&d_mhi, nn * tc::NP * sizeof(float)));
    KIFMM_CUDA(cudaMalloc(&d_mlo, nn * tc::NP * sizeof(float)));
    KIFMM_CUDA(cudaMalloc(&d_partial, std::max(1, n_items) * size_t(tc::BM) * tc::NP * sizeof(float)));
    *total += 2 * nn * tc::NP * sizeof(float) + size_t(n_items) * tc::BM * tc::NP * sizeof(float);
    // ---- TMA descriptors over [nt * 160 rows][160 cols] fp32, box 32 x 160, SWIZZLE_128B
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    KIFMM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn) throw DeviceError(KIFMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {cuuint64_t(tc::NP), cuuint64_t(nt) * tc::NP};
    const cuuint64_t strides[1] = {cuuint64_t(tc::NP) * sizeof(float)};
    const cuuint32_t box[2] = {cuuint32_t(tc::KB), cuuint32_t(tc::NP)};
    const cuuint32_t estr[2] = {1, 1};
    for (int which = 0; which < 2; ++which) {
      CUresult r = reinterpret_cast<EncodeFn>(fn)(which ? &tm_lo : &tm_hi, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                                  which ? d_klo : d_khi, dims, strides, box, estr,
                                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw DeviceError(KIFMM_E_CUDA, "cuTensorMapEncodeTiled failed");
    }
    KIFMM_CUDA(cudaFuncSetAttribute(tc::m2l_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_BYTES));
  }

  // check += M2L(M): split M, run the tcgen05 items, reduce partials.
  void launch(const float* M, float* check, int np, cudaStream_t s) {
    if (!n_items) return;
    const size_t n = nn * size_t(np);
    tc::split_tf32_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(M, n, d_mhi, d_mlo);
    KIFMM_LAUNCH_CHECK();
    tc::m2l_tc_kernel<<<n_items, tc::THREADS, tc::SMEM_BYTES, s>>>(tm_hi, tm_lo, d_items, d_seg_mat, d_seg_in, d_mhi,
                                                                   d_mlo, d_partial);
    KIFMM_LAUNCH_CHECK();
    tc::m2l_tc_reduce_kernel<<<n_tiles, 256, 0, s>>>(d_partial, d_tile_out, d_tile_slot, check);
    KIFMM_LAUNCH_CHECK();
  }
};

}  // namespace gpu
}  // namespace kifmm
