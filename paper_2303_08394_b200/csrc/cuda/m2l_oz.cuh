// fp64 M2L on the int8 tensor cores: the Ozaki scheme (error-free splitting into int8
// digit slices, exact int32 products and sums) with tcgen05.mma kind::i8.
//
// check[target] += sum_taps M[src(target, t)] . K_t^T, in fp64 (config 4: p = 7, n_e = 218 -> 224).
// B200's fp64 paths top out at 37 TFLOP/s (DMMA and DFMA alike, tools/ubench/dmma_rate.cu), so the
// DMMA kernel (gemm.cuh) needs ~134 ms for config 4's 5e12 useful flop at best; the int8 tensor cores
// run at 4.5 POPS.  Operands are split into S signed 7-bit digits:
//   M[row][k] = 2^E(l) sum_i d_i 2^-7i        (E(l): one exponent per tree level, |M| 2^-E < 1/2)
//   K_t[n][k] = 2^F    sum_j e_j 2^-7j        (F: one exponent for all 316 operators)
// with |d|, |e| <= 64, so  M K^T = 2^(E+F) sum_g 2^-7g sum_{i+j=g} D_i E_j^T  and every D_i E_j^T is an
// exact int8 x int8 -> int32 product.  Digit sums g = i + j <= S + 1 are kept (Ozaki's triangular
// truncation; the dropped terms and the digit residue are ~2^-50 relative to the level maximum).
// Because E is per level (a tile's rows, and all its sources, are one level) and F is global, all taps
// of a tile share one scale: the int32 accumulators run over the whole tap list (|sum| <= S products x
// NP x 64 x 64 per tap: up to 292 taps for S = 8, NP = 224; longer lists drain in two units) and are
// converted to fp64 once per tile -- no per-tap promotion.  S = 8 (36 products, 8 groups): the int8 path
// agrees with the fp64 DMMA kernel to 3e-15 (S = 7: 1e-13 on signed charges, 10 % faster).
//
// Work item = (tile of 128 target rows, output half h: columns [h NH, h NH + NH), NH = NP / 2).  Each
// item runs two passes over its taps with different digit-sum groups in TMEM (int32, NH columns each):
//   pass 0: g = 2..5 (10 products, digits 1..4)     pass 1: g = 6..S+1 (26 products for S = 8)
// A stage is one (tap, 32-byte K block): the needed digit slices of the 128 gathered source rows (cp.async
// into SWIZZLE_32B K-major atoms) and of the operator rows (TMA, SWIZZLE_32B), then one MMA per product.
// Epilogue (per pass): tcgen05.ld the group accumulators, sum_g acc_g 2^-7g in fp64, times 2^(E+F), add to
// the fp64 check rows (each row belongs to one tile, each column half to one item: no races).
// Warps: 0 TMEM alloc + B TMA producer, 1 MMA issuer, 4-7 epilogue (TMEM lane quarters), 8-11 A producers.
#pragma once

#include "m2l_tc.cuh"

namespace kifmm {
namespace gpu {
namespace oz {

#ifndef KIFMM_OZ_SLICES
#define KIFMM_OZ_SLICES 8
#endif
constexpr int S = KIFMM_OZ_SLICES;  // digit slices per operand
static_assert(S >= 5 && S <= 8, "two passes of <= 4 digit-sum groups");
constexpr int BM = 128;
constexpr int THREADS = 384;
constexpr int EPI_WARP0 = 4, PROD_WARP0 = 8;
constexpr uint32_t TMEM_COLS = 512;
__host__ __device__ constexpr int g_lo(int p) { return p == 0 ? 2 : 6; }
__host__ __device__ constexpr int g_hi(int p) { return p == 0 ? 5 : S + 1; }
__host__ __device__ constexpr int n_slices(int p) { return g_hi(p) - 1; }  // digits 1 .. g_hi - 1 are read
__host__ __device__ constexpr int n_products(int p) {
  int n = 0;
  for (int i = 1; i <= S; ++i)
    for (int j = 1; j <= S; ++j)
      if (i + j >= g_lo(p) && i + j <= g_hi(p)) ++n;
  return n;
}

template <int NP>
struct Cfg {
  static constexpr int NH = NP / 2;   // MMA N: output columns per item
  static constexpr int NKB = NP / 32; // 32-byte K blocks per tap
  static constexpr int A_SL = BM * 32, B_SL = NH * 32;
  static constexpr int STAGE = S * (A_SL + B_SL);
  static constexpr int STAGES = 4 * STAGE + 1280 <= 227 * 1024 ? 4 : 3;  // (tap, K block) stages in flight
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static constexpr uint32_t IDESC = (2u << 4)                 // D: s32
                                    | (1u << 7) | (1u << 10)  // A, B: signed 8-bit
                                    | (uint32_t(NH >> 3) << 17) | (uint32_t(BM >> 4) << 24);
  static_assert(NP % 32 == 0 && NH % 16 == 0 && 4 * NH <= int(TMEM_COLS), "int8 M2L shape");
};

struct Args {
  const int8_t* a8;                 // [(zero_row + 1)][S][NP] digit slices of the multipole rows
  const int* sched;                 // [G + 1] item ranges per CTA, then the item list (item = tile * 2 + h)
  const int* tile_out;              // [n_tiles][BM] output row (-1: padding)
  const int* seg_ptr;               // [n_tiles + 1]
  const int* seg_mat;               // [n_segs] operator (transfer vector) index
  const int* seg_in;                // [n_segs][BM] source row (-1: absent -> zero row)
  const int* tile_level;            // [n_tiles]
  const unsigned long long* lmax;   // [levels] max |M| of a level (fp64 bits)
  double fscale;                    // 2^F
  int zero_row;
  double* dst;                      // check rows (+=), row stride NP
};

__device__ __forceinline__ int level_exp(unsigned long long bits) {
  const double m = __longlong_as_double(static_cast<long long>(bits));
  return m > 0.0 ? ilogb(m) + 2 : 0;  // |x| 2^-E < 1/2
}

// Taps per accumulation unit: every digit-sum group holds <= S products of |d e| <= 64 x 64 over NP K
// values per tap, so int32 cannot overflow within tap_max taps; longer tap lists (only the small upper
// levels of a tree reach 316) are drained into the check rows in several units
template <int NP>
__host__ __device__ constexpr int tap_max() {
  return int(2147483647LL / (int64_t(S) * NP * 64 * 64));
}
template <int NP>
__host__ __device__ constexpr int n_chunks(int ntap) {
  return ntap <= tap_max<NP>() ? 1 : (ntap + tap_max<NP>() - 1) / tap_max<NP>();
}

// SWIZZLE_32B K-major shared-memory descriptor: 8-row atoms of 32-byte rows, 256 B apart
__device__ __forceinline__ uint64_t desc32(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(256 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(6) << 61;
  return d;
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// one stage's MMAs of pass P: every product (i, j) of its digit-sum groups into group slot g - g_lo(P)
template <int NP, int P>
__device__ __forceinline__ void issue_stage(uint32_t tmem, uint32_t a0, uint32_t b0, bool first_stage) {
  using C = Cfg<NP>;
  bool seen[4] = {false, false, false, false};
#pragma unroll
  for (int i = 1; i <= S; ++i)
#pragma unroll
    for (int j = 1; j <= S; ++j) {
      const int g = i + j;
      if (g < g_lo(P) || g > g_hi(P)) continue;
      const int q = g - g_lo(P);
      const uint32_t acc = (!first_stage || seen[q]) ? 1u : 0u;
      seen[q] = true;
      mma_i8(tmem + uint32_t(q * C::NH), desc32(a0 + uint32_t((i - 1) * C::A_SL)),
             desc32(b0 + uint32_t((j - 1) * C::B_SL)), C::IDESC, acc);
    }
}

template <int NP>
__global__ void __launch_bounds__(THREADS, 1) m2l_oz_kernel(const __grid_constant__ CUtensorMap tm_b, Args a) {
  using C = Cfg<NP>;
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int STAGES = C::STAGES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g0 = blockIdx.x;
  const int k_begin = a.sched[g0], k_end = a.sched[g0 + 1];
  const int* list = a.sched + gridDim.x + 1;
  const uint32_t sbase = smem_u32(smem);
  auto a_sl = [&](int s) { return sbase + uint32_t(s * C::STAGE); };                  // + i * A_SL
  auto b_sl = [&](int s) { return sbase + uint32_t(s * C::STAGE + S * C::A_SL); };    // + j * B_SL
  auto full = [&](int s) { return smem_u32(&bars[s]); };
  auto empty = [&](int s) { return smem_u32(&bars[STAGES + s]); };
  const uint32_t tfull = smem_u32(&bars[2 * STAGES]), tempty = smem_u32(&bars[2 * STAGES + 1]);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1 + 128);  // B bytes (expect_tx) + the 128 A producers' cp.async arrivals
      mbar_init(empty(s), 1);       // tcgen05.commit
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);  // one elected lane per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_b) : "memory");
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
    // ---------------- B producer: digit slices of K_t (rows (t S + j) NP + h NH .., K block kb) by TMA
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int kk = k_begin; kk < k_end; ++kk) {
        const int item = list[kk], tile = item >> 1, h = item & 1;
        const int sg0 = a.seg_ptr[tile], sg1 = a.seg_ptr[tile + 1];
        for (int p = 0; p < 2; ++p) {
          const int ns = n_slices(p);
          for (int sg = sg0; sg < sg1; ++sg) {
            const int mat = a.seg_mat[sg];
            for (int kb = 0; kb < C::NKB; ++kb) {
              mbar_wait(empty(s), ph ^ 1u);
              mbar_expect_tx(full(s), uint32_t(ns * C::B_SL));
              for (int j = 0; j < ns; ++j)
                tma_tile<false>(b_sl(s) + uint32_t(j * C::B_SL), &tm_b, full(s), kb * 32, (mat * S + j) * NP + h * C::NH);
              if (++s == STAGES) {
                s = 0;
                ph ^= 1u;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one elected lane; the warp walks the loop)
    int s = 0, units = 0;
    uint32_t ph = 0;
    for (int kk = k_begin; kk < k_end; ++kk) {
      const int item = list[kk], tile = item >> 1;
      const int ntap = a.seg_ptr[tile + 1] - a.seg_ptr[tile];
      for (int u = 0; u < 2 * n_chunks<NP>(ntap); ++u, ++units) {
        const int p = u / n_chunks<NP>(ntap), ch = u % n_chunks<NP>(ntap);
        const int nstage = (min(ntap, (ch + 1) * tap_max<NP>()) - ch * tap_max<NP>()) * C::NKB;
        mbar_wait(tempty, (uint32_t(units) & 1u) ^ 1u);  // the epilogue drained the previous unit
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int i = 0; i < nstage; ++i) {
          mbar_wait(full(s), ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (elect_one()) {
            if (p == 0)
              issue_stage<NP, 0>(tmem_base, a_sl(s), b_sl(s), i == 0);
            else
              issue_stage<NP, 1>(tmem_base, a_sl(s), b_sl(s), i == 0);
            commit<false>(empty(s));
            if (i == nstage - 1) commit<false>(tfull);
          }
          __syncwarp();
          if (++s == STAGES) {
            s = 0;
            ph ^= 1u;
          }
        }
        if (nstage == 0) {  // no taps (never built; keeps the barrier protocol total)
          if (elect_one()) commit<false>(tfull);
          __syncwarp();
        }
      }
    }
  } else if (warp >= PROD_WARP0) {
    // ---------------- A producers: threads 2r', 2r' + 1 copy the two 16-byte halves of the 32-byte K block of
    //                  rows r' and r' + 64, for every needed digit slice, by cp.async into the SWIZZLE_32B
    //                  atoms -- a warp instruction covers 16 rows x 32 B, i.e. whole 32-byte sectors (a
    //                  thread per row issued two half-sector requests per sector: L1TEX 94 % busy)
    const int t = threadIdx.x - 32 * PROD_WARP0;
    const int half = t & 1;
    int rr[2], so[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int r = (t >> 1) + 64 * k;
      rr[k] = r;
      so[k] = (r >> 3) * 256 + (r & 7) * 32 + ((half ^ ((r >> 2) & 1)) << 4);
    }
    int s = 0;
    uint32_t ph = 0;
    for (int kk = k_begin; kk < k_end; ++kk) {
      const int item = list[kk], tile = item >> 1;
      const int sg0 = a.seg_ptr[tile], sg1 = a.seg_ptr[tile + 1];
      for (int p = 0; p < 2; ++p) {
        const int ns = n_slices(p);
        int nxt[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) nxt[k] = sg0 < sg1 ? a.seg_in[size_t(sg0) * BM + rr[k]] : -1;
        for (int sg = sg0; sg < sg1; ++sg) {
          const int8_t* row[2];
          int sz[2];
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const bool ok = nxt[k] >= 0;
            row[k] = a.a8 + size_t(ok ? nxt[k] : a.zero_row) * (S * NP) + half * 16;
            sz[k] = ok ? 16 : 0;
          }
          if (sg + 1 < sg1) {  // one tap ahead
#pragma unroll
            for (int k = 0; k < 2; ++k) nxt[k] = a.seg_in[size_t(sg + 1) * BM + rr[k]];
          }
          for (int kb = 0; kb < C::NKB; ++kb) {
            mbar_wait(empty(s), ph ^ 1u);
            const uint32_t base = a_sl(s);
            for (int i = 0; i < ns; ++i) {
              const uint32_t d = base + uint32_t(i * C::A_SL);
#pragma unroll
              for (int k = 0; k < 2; ++k)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d + uint32_t(so[k])),
                             "l"(row[k] + i * NP + kb * 32), "r"(sz[k])
                             : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full(s)) : "memory");
            if (++s == STAGES) {
              s = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp >= EPI_WARP0 && warp < EPI_WARP0 + 4) {
    // ---------------- epilogue: thread = tile row; groups of the pass -> fp64, scaled, added to dst
    const int q = warp - EPI_WARP0;
    const int r = q * 32 + lane;
    const uint32_t lane_base = tmem_base + (uint32_t(q * 32) << 16);
    int units = 0;
    for (int kk = k_begin; kk < k_end; ++kk) {
      const int item = list[kk], tile = item >> 1, h = item & 1;
      const int o = a.tile_out[size_t(tile) * BM + r];
      const double scale = ldexp(a.fscale, level_exp(a.lmax[a.tile_level[tile]]));
      const int ntap = a.seg_ptr[tile + 1] - a.seg_ptr[tile];
      for (int u = 0; u < 2 * n_chunks<NP>(ntap); ++u, ++units) {
        const int p = u / n_chunks<NP>(ntap);
        mbar_wait_sleep(tfull, uint32_t(units) & 1u);
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int ng = g_hi(p) - g_lo(p) + 1;
        double* drow = o >= 0 ? a.dst + size_t(o) * NP + h * C::NH : nullptr;
        for (int c0 = 0; c0 < C::NH; c0 += 16) {
          double v[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) v[c] = 0.0;
          for (int qg = 0; qg < ng; ++qg) {
            uint32_t x[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];"
                : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]),
                  "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]),
                  "=r"(x[15])
                : "r"(lane_base + uint32_t(qg * C::NH + c0)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const double w = ldexp(1.0, -7 * (g_lo(p) + qg));
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = fma(double(int(x[c])), w, v[c]);
          }
          if (drow) {
#pragma unroll
            for (int c = 0; c < 16; c += 2) {
              double2 d = *reinterpret_cast<const double2*>(drow + c0 + c);
              d.x += v[c] * scale;
              d.y += v[c + 1] * scale;
              *reinterpret_cast<double2*>(drow + c0 + c) = d;
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_local(tempty);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// max |M| per tree level (fp64 bits; positive doubles order like their bit patterns): one warp per row
template <int NP>
__global__ void oz_level_max_kernel(const double* __restrict__ M, int nn, const int* __restrict__ node_level,
                                    unsigned long long* __restrict__ lmax) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= nn) return;
  double m = 0.0;
  for (int k = lane; k < NP; k += 32) m = fmax(m, fabs(M[size_t(row) * NP + k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0 && m > 0.0)
    atomicMax(lmax + node_level[row], static_cast<unsigned long long>(__double_as_longlong(m)));
}

// digit slices: x 2^-E = sum_i d_i 2^-7i, d_i = rint(128 y) of the running remainder y (all steps exact)
template <int NP>
__global__ void oz_slice_kernel(const double* __restrict__ M, int nn, const int* __restrict__ node_level,
                                const unsigned long long* __restrict__ lmax, int8_t* __restrict__ a8) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(nn) * NP) return;
  const int row = int(i / NP), k = int(i % NP);
  double y = ldexp(M[i], -level_exp(lmax[node_level[row]]));
  int8_t* out = a8 + size_t(row) * (S * NP) + k;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    y *= 128.0;
    const double d = rint(y);
    y -= d;
    out[s * NP] = static_cast<int8_t>(static_cast<int>(d));
  }
}

}  // namespace oz

// Host side: 128-row tiles (no tap splitting: a tile's rows are owned by its two items), operator digit
// slices and their TMA map, an LPT schedule of the items over one CTA per SM.
struct M2LOzPlan {
  int np = 0, n_tiles = 0, n_items = 0, grid = 0, levels = 0;
  int zero_row = 0;
  double fscale = 1.0;
  int64_t slots = 0;
  int8_t *d_a8 = nullptr, *d_b8 = nullptr;
  int *d_sched = nullptr, *d_tile_out = nullptr, *d_seg_ptr = nullptr, *d_seg_mat = nullptr, *d_seg_in = nullptr,
      *d_tile_level = nullptr;
  unsigned long long* d_lmax = nullptr;
  CUtensorMap tm_b{};

  ~M2LOzPlan() {
    for (void* p : {(void*)d_a8, (void*)d_b8, (void*)d_sched, (void*)d_tile_out, (void*)d_seg_ptr, (void*)d_seg_mat,
                    (void*)d_seg_in, (void*)d_tile_level, (void*)d_lmax})
      if (p) cudaFree(p);
  }
  template <class V>
  static void up(V** dst, const std::vector<V>& v, size_t* total) {
    KIFMM_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), std::max<size_t>(1, v.size()) * sizeof(V)));
    if (!v.empty()) KIFMM_CUDA(cudaMemcpy(*dst, v.data(), v.size() * sizeof(V), cudaMemcpyHostToDevice));
    *total += v.size() * sizeof(V);
  }
  static bool supported(int np_) { return np_ == 160 || np_ == 224; }

  // groups: target nodes per (level, octant); v lists from the tree view; ops.m2l: n_m2l x n_c x n_e (fp64)
  template <class TreeView, class OpsView, class LevelFn>
  void build(const TreeView& t, const std::vector<std::vector<int64_t>>& groups, int np_, const OpsView& ops,
             int64_t nn, LevelFn node_lvl, int max_level, int sms, size_t* total) {
    np = np_;
    zero_row = int(nn);
    levels = max_level + 1;
    constexpr int BM = oz::BM, S = oz::S;
    // ---- tiles
    std::vector<int> tile_out, seg_ptr{0}, seg_mat, seg_in, tile_level;
    std::vector<int64_t> cost;
    for (const auto& grp : groups) {
      for (size_t s0 = 0; s0 < grp.size(); s0 += BM) {
        std::map<int, std::vector<int>> taps;
        const size_t base = tile_out.size();
        tile_out.resize(base + BM, -1);
        for (int r = 0; r < BM && s0 + r < grp.size(); ++r) {
          const int64_t b = grp[s0 + r];
          tile_out[base + r] = int(b);
          for (int64_t e = t.v_ptr[b]; e < t.v_ptr[b + 1]; ++e) {
            auto& v = taps[t.v_tv[e]];
            if (v.empty()) v.assign(BM, -1);
            v[r] = int(t.v_idx[e]);
          }
        }
        for (auto& kv : taps) {
          seg_mat.push_back(kv.first);
          seg_in.insert(seg_in.end(), kv.second.begin(), kv.second.end());
        }
        seg_ptr.push_back(int(seg_mat.size()));
        tile_level.push_back(node_lvl(grp[s0]));
        cost.push_back(int64_t(taps.size()));
        slots += int64_t(taps.size()) * BM;
      }
    }
    n_tiles = int(tile_level.size());
    n_items = 2 * n_tiles;
    // ---- LPT schedule: items by cost (taps) onto G CTAs
    grid = std::max(1, std::min(sms, n_items));
    std::vector<int> order(n_items);
    for (int i = 0; i < n_items; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return cost[x >> 1] > cost[y >> 1]; });
    std::vector<std::vector<int>> per(grid);
    std::priority_queue<std::pair<int64_t, int>, std::vector<std::pair<int64_t, int>>, std::greater<>> pq;
    for (int g = 0; g < grid; ++g) pq.push({0, g});
    for (int it : order) {
      auto [load, g] = pq.top();
      pq.pop();
      per[g].push_back(it);
      pq.push({load + cost[it >> 1] + 1, g});
    }
    std::vector<int> sched{0};
    std::vector<int> list;
    for (auto& v : per) {
      list.insert(list.end(), v.begin(), v.end());
      sched.push_back(int(list.size()));
    }
    sched.insert(sched.end(), list.begin(), list.end());
    up(&d_sched, sched, total);
    up(&d_tile_out, tile_out, total);
    up(&d_seg_ptr, seg_ptr, total);
    up(&d_seg_mat, seg_mat, total);
    up(&d_seg_in, seg_in, total);
    up(&d_tile_level, tile_level, total);
    KIFMM_CUDA(cudaMalloc(&d_lmax, size_t(levels) * sizeof(unsigned long long)));
    // ---- multipole digit slices (rewritten every evaluate) + the zero row
    const size_t a_bytes = size_t(nn + 1) * S * np;
    KIFMM_CUDA(cudaMalloc(&d_a8, a_bytes));
    KIFMM_CUDA(cudaMemset(d_a8, 0, a_bytes));
    *total += a_bytes;
    // ---- operator digit slices: rows (t S + j) np + n, K-major (np bytes), one exponent F for all
    const int nt = ops.n_m2l, nc = ops.n_c, ne = ops.n_e;
    double kmax = 0.0;
#pragma omp parallel for reduction(max : kmax) schedule(static)
    for (int64_t i = 0; i < int64_t(nt) * nc * ne; ++i) kmax = std::max(kmax, std::fabs(ops.m2l[i]));
    const int F = kmax > 0.0 ? std::ilogb(kmax) + 2 : 0;
    fscale = std::ldexp(1.0, F);
    std::vector<int8_t> b8(size_t(nt) * S * np * np, 0);
#pragma omp parallel for schedule(static)
    for (int tv = 0; tv < nt; ++tv)
      for (int n = 0; n < nc; ++n)
        for (int k = 0; k < ne; ++k) {
          double y = std::ldexp(ops.m2l[(size_t(tv) * nc + n) * ne + k], -F);
          for (int j = 0; j < S; ++j) {
            y *= 128.0;
            const double d = std::nearbyint(y);
            y -= d;
            b8[((size_t(tv) * S + j) * np + n) * np + k] = static_cast<int8_t>(int(d));
          }
        }
    up(&d_b8, b8, total);
    // ---- TMA map of the operator slices: inner dim K (np bytes), box 32 B x NH rows, SWIZZLE_32B
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    KIFMM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn) throw DeviceError(KIFMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {cuuint64_t(np), cuuint64_t(size_t(nt) * S * np)};
    const cuuint64_t strides[1] = {cuuint64_t(np)};
    const cuuint32_t box[2] = {32u, cuuint32_t(np / 2)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = reinterpret_cast<M2LTcPlan::EncodeFn>(fn)(
        &tm_b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d_b8, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw DeviceError(KIFMM_E_CUDA, "cuTensorMapEncodeTiled (int8 operators) failed");
    if (np == 160) set_attr<160>();
    else set_attr<224>();
  }
  template <int NP>
  static void set_attr() {
    KIFMM_CUDA(cudaFuncSetAttribute(oz::m2l_oz_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    oz::Cfg<NP>::SMEM));
  }
  int launches() const { return n_items ? 3 : 0; }

  // check[rows] += M2L(M): level maxima -> digit slices -> int8 tensor-core kernel
  template <int NP>
  void run_np(const double* M, const int* node_level, double* check, cudaStream_t s) const {
    KIFMM_CUDA(cudaMemsetAsync(d_lmax, 0, size_t(levels) * sizeof(unsigned long long), s));
    oz::oz_level_max_kernel<NP><<<(zero_row + 7) / 8, 256, 0, s>>>(M, zero_row, node_level, d_lmax);
    KIFMM_LAUNCH_CHECK();
    const size_t n = size_t(zero_row) * NP;
    oz::oz_slice_kernel<NP><<<unsigned((n + 255) / 256), 256, 0, s>>>(M, zero_row, node_level, d_lmax, d_a8);
    KIFMM_LAUNCH_CHECK();
    oz::Args a{d_a8, d_sched, d_tile_out, d_seg_ptr, d_seg_mat, d_seg_in, d_tile_level, d_lmax, fscale, zero_row,
               check};
    oz::m2l_oz_kernel<NP><<<grid, oz::THREADS, oz::Cfg<NP>::SMEM, s>>>(tm_b, a);
    KIFMM_LAUNCH_CHECK();
  }
  void run(const double* M, const int* node_level, double* check, cudaStream_t s) const {
    if (!n_items) return;
    if (np == 160)
      run_np<160>(M, node_level, check, s);
    else
      run_np<224>(M, node_level, check, s);
  }
};

}  // namespace gpu
}  // namespace kifmm
