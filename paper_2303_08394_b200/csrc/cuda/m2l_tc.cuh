// M2L on the 5th-generation tensor cores (SURVEY 7.3 "M2L batching").
//
// Work: for a tile of same-class target nodes and one transfer vector t,
//   D[rows x NP] += A_t[rows x NP] . K_t^T (NP = n_e padded: 64, 128, 160, 224 for p = 4..7),  A_t rows = multipoles of the
// V-list sources at offset t (a zero row where absent), K_t = reference-level
// kernel matrix (n_c x n_e, K-major).  Two error-compensated operand formats
// (template ES):
//   ES = 2 (default, m2l_backend 2): kind::f16.  fp32 values are scaled by a power of two
//          (per multipole row; 2^8 for K_t) and split x = hi + lo in fp16, and
//          D += A_hi B_hi + A_hi B_lo + A_lo B_hi (the dropped lo.lo term is ~2^-22 relative).
//   ES = 4 (m2l_backend 3, KIFMM_TC_KIND=tf32): kind::tf32 with the same 3-term split in tf32 (3xTF32).
//
// K_t hi/lo arrive by TMA (SWIZZLE_128B, mbarrier transaction counts); the
// gathered A rows (missing sources read an appended zero row) are copied by 128
// threads with cp.async into the same SW128 K-major layout (TMA tile::gather4
// was measured 3x slower for these 128-byte rows).  Stages are (tap, 32-wide K
// block) pairs.
//
// Two variants (template PAIR):
//   PAIR = false: one CTA, M = 128 targets (stage counts below are for NP = 160, 128-byte rows).
//   PAIR = true : a 2-CTA cluster (cta_group::2), M = 256; each CTA gathers its
//                 own 128 A rows and half of K_t (80 check rows), 4 stages of
//                 52 KB; only the leader issues tcgen05.mma, and stage / TMEM
//                 barriers the MMA waits on live in the leader.
//
// Warps: 0 TMEM alloc + B producer, 1 MMA issuer, 2-5 A producers, 6-13
// epilogue, 14 A-arrival forwarder to the leader (pair).  The tensor-core accumulator is not IEEE round-to-
// nearest and its error grows with the accumulation length (measured 1.2e-6 at
// 1 tap, 1.5e-5 at 16, 1.5e-4 at 189 taps), so each transfer vector
// accumulates in a fresh TMEM buffer (two alternate) that the epilogue warps
// drain with tcgen05.ld into fp32 registers ("per-tap promotion").  Partials of
// the tap chunks of a tile are summed by m2l_tc_reduce_kernel in fixed order
// (deterministic; no atomics).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <queue>
#include <set>
#include <array>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace kifmm {
namespace gpu {
namespace tc {

constexpr int BM = 128;  // target rows per CTA
// NP (template parameter of everything below): check / equivalent points per row, padded to a multiple of
// 32 -- 64 (p = 4), 128 (p = 5), 160 (p = 6); see tc_np_supported() / tc_dispatch_np().
// Warpgroups: 0 = {TMA + TMEM alloc, MMA issuer, A-arrival forwarder (pair), idle}, 1 = A producers,
// 2-3 = epilogue.  The kernel launches with 80 registers per thread (__maxnreg__) and rebalances with
// setmaxnreg (warpgroups 0-1 down to 48, epilogue up to 112): a CTA holds 40 K registers, leaving
// room on the SM for three near-field blocks next to it (measured fastest end to end, despite a few
// hundred bytes of epilogue spills; 96/56/136 with two near blocks: +2.5 %).
constexpr int EPI_WARPS = 8;                      // 2 warps per TMEM lane quarter, NP / 2 columns each
constexpr int EPI_WARP0 = 8;                      // epilogue warps 8..15
constexpr int PROD_WARP0 = 4;                     // A producer warps 4..7
constexpr int FWD_WARP = 2;                       // A-arrival forwarder (pair)
constexpr int THREADS = 512;
#ifndef KIFMM_TC_LAUNCH_REGS
#define KIFMM_TC_LAUNCH_REGS 80
#define KIFMM_TC_LOW_REGS 48
#define KIFMM_TC_EPI_REGS 112
#endif
// Row width 224 (p = 7, M2L pair kernel only): an epilogue thread keeps 112 fp32 sums, so that instantiation
// launches with 104 registers per thread and rebalances to 40 / 168 (one near-field side block fits next to it).
template <int NP>
struct Regs {
  static constexpr int LAUNCH = NP > 160 ? 104 : KIFMM_TC_LAUNCH_REGS;
  static constexpr int LOW = NP > 160 ? 40 : KIFMM_TC_LOW_REGS;
  static constexpr int EPI = NP > 160 ? 168 : KIFMM_TC_EPI_REGS;
  static_assert(4 * 32 * LOW * 2 + 8 * 32 * EPI <= THREADS * LAUNCH, "setmaxnreg budget");
};
constexpr uint32_t TMEM_COLS = 512;  // accumulator sets of NP columns at 0, NP, 2 NP (two sets at NP = 224)
constexpr int NACC = 3;              // accumulator buffers: the MMA runs up to two taps ahead of the epilogue
// The tensor-core accumulator rounds toward zero after every MMA (1 ulp per K step, measured), a bias that
// adds up coherently along a chain of GEMMs.  The single-CTA instantiation (the factored solves, M2M and
// L2L chain -- up to ten GEMMs deep) therefore keeps three accumulators per tap: the A_hi B_hi products of
// even and odd K steps in two of them (5 truncations each instead of 30 in one) and the 2^-11-smaller
// A_hi B_lo + A_lo B_hi corrections in the third; the epilogue sums them in fp32 round-to-nearest.  One
// such set fills 480 TMEM columns, so that variant runs one tap at a time (NSET 1).  The M2L pair keeps
// one accumulator per tap and three sets in flight (its taps are summed in fp32 per tap anyway).
template <int NP, bool PAIR>
struct Acc {
  static constexpr int NSET = PAIR ? (NACC * NP <= int(TMEM_COLS) ? NACC : 2) : 1;  // accumulator sets in TMEM
  static constexpr int SET_COLS = PAIR ? NP : 3 * NP;  // columns per set
};

// ROWB: bytes of one operand row per stage (K block of ROWB/4 fp32): 128 (SWIZZLE_128B) or 64 (SWIZZLE_64B,
// twice the stages for the same shared memory => deeper latency hiding).
#ifndef KIFMM_TC_STAGE_KB
#define KIFMM_TC_STAGE_KB 136
#endif
// shared memory for pipeline stages: 136 KB (5 stages for the f16 pair, 3 for the single CTA) leaves
// room on the SM for three near-field blocks next to a tcgen05 CTA (a full 216 KB pipeline, with the
// near field waiting for whole SMs, measured 6-7 % slower end to end; M2L alone is insensitive to 112-216)
constexpr int kStageBudgetKB = KIFMM_TC_STAGE_KB;
#ifndef KIFMM_TC_EG
#define KIFMM_TC_EG 1
#endif

template <int NP, bool PAIR, int ROWB, int ES = 4>
struct Cfg {
  static constexpr int KB = ROWB / ES;           // operand elements per K block (tf32: 4 B, f16: 2 B)
  static constexpr int NKB = NP / KB;            // K blocks per tap
  static constexpr int NB = PAIR ? NP / 2 : NP;  // B rows held per CTA
  static constexpr int A_BYTES = BM * ROWB;
  static constexpr int B_BYTES = NB * ROWB;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = (kStageBudgetKB * 1024) / STAGE_BYTES;
  // stages can be released to the producers in groups of EG (one tcgen05.commit per group; a commit
  // costs ~50 cycles of MMA issue in tools/ubench/mma_pair.cu) -- measured slower in the kernel (the
  // shorter effective lookahead costs more than the commits save), so EG = 1
  static constexpr int EG = (STAGES % KIFMM_TC_EG == 0) ? KIFMM_TC_EG : 1;
  // + barriers, row-max exchange, and (single CTA: direct GEMM epilogue) the 8 x 32 x 20-float transpose buffer
  //   and the column unscale
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 512 + 2048 + (PAIR ? 0 : 8 * 32 * 20 * 4 + NP * 4);
  static constexpr int ATOM = 8 * ROWB;           // bytes of an 8-row swizzle atom (= SBO)
  static constexpr uint64_t LAYOUT = ROWB == 128 ? 2 : 4;  // SWIZZLE_128B / SWIZZLE_64B
  static constexpr int CTAS = PAIR ? 2 : 1;
  static constexpr uint32_t TX = uint32_t(CTAS * 2 * B_BYTES);  // TMA bytes landing on the leader per stage
  static constexpr uint32_t FMT = ES == 4 ? 2u : 0u;  // tf32 / f16
  static constexpr uint32_t IDESC = (1u << 4) | (FMT << 7) | (FMT << 10) | (uint32_t(NP >> 3) << 17) |
                                    (uint32_t((CTAS * BM) >> 4) << 24);
};

#ifdef KIFMM_EXPERIMENTS
#define TC_DBG(bit) (epi.debug & (bit))
#else
#define TC_DBG(bit) 0
#endif

struct Item {
  int tile, seg_begin, seg_end, slot;
};

// Epilogue destination: per-item partial rows (summed later by m2l_tc_reduce_kernel), or -- when
// direct_out is set and every tile is one item -- the output rows themselves:
//   dst[direct_out[tile][r]][c] = (accumulate ? dst[..][c] : 0) + acc[r][c] * col_unscale[c]
// Optionally (split_hi set, direct mode) the epilogue also emits the fp16 hi / lo split of every output
// row with its power-of-two unscale -- the A operand of the next tcgen05 GEMM -- exactly as
// split_f16_rows_kernel would; dst may then be null (the fp32 row is not needed).
struct Epi {
  float* partial;
  const int* direct_out;
  const float* col_unscale;
  float* dst;
  int accumulate;
  int debug;  // experiments only (-DKIFMM_EXPERIMENTS, KIFMM_TC_DBG): bit 0 skips the A gathers, bit 1 the B
              // TMA loads; the product build compiles every TC_DBG test to 0
  __half* split_hi;
  __half* split_lo;
  float* split_un;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_local(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
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
// Wait with a nanosleep back-off, for roles whose barrier completes on a coarse time scale (epilogue,
// producers): their spinning would otherwise take issue slots from blocks of other kernels sharing
// the SM (the near field runs next to these kernels).
#ifndef KIFMM_TC_SLEEP_NS
#define KIFMM_TC_SLEEP_NS 64
#endif
#ifndef KIFMM_TC_PROD_SLEEP
#define KIFMM_TC_PROD_SLEEP 0  // producers poll without back-off (their wait gates the refill)
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
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
    if (KIFMM_TC_SLEEP_NS > 0) __nanosleep(KIFMM_TC_SLEEP_NS);
    if (spin > (1u << 26)) asm volatile("trap;");
  }
}

__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(e));
  return e != 0;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// SM100 UMMA shared-memory descriptor: K-major, swizzled, 8-row atoms SBO bytes apart.
template <int ROWB>
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);          // start address
  d |= uint64_t(1) << 16;                         // LBO (unused for swizzled K-major) = 16 B
  d |= uint64_t((8 * ROWB) >> 4) << 32;           // SBO = one 8-row atom
  d |= uint64_t(1) << 46;                         // version (sm100)
  d |= uint64_t(ROWB == 128 ? 2 : 4) << 61;       // SWIZZLE_128B / SWIZZLE_64B
  return d;
}

// The three MMAs of one K step of the 3-term split: D (+)= A_hi B_hi, += A_hi B_lo, += A_lo B_hi.
#ifndef KIFMM_MMA3_BFIRST
#define KIFMM_MMA3_ORDER(GROUP, KIND)                                            \
  "tcgen05.mma.cta_group::" GROUP ".kind::" KIND " [%0], %1, %4, %5, t;\n"      \
  "tcgen05.mma.cta_group::" GROUP ".kind::" KIND " [%0], %2, %3, %5, t;\n"
#else  // experiment: A_lo B_hi second (B_hi reused by consecutive MMAs)
#define KIFMM_MMA3_ORDER(GROUP, KIND)                                            \
  "tcgen05.mma.cta_group::" GROUP ".kind::" KIND " [%0], %2, %3, %5, t;\n"      \
  "tcgen05.mma.cta_group::" GROUP ".kind::" KIND " [%0], %1, %4, %5, t;\n"
#endif
template <bool PAIR, int ES>
__device__ __forceinline__ void mma3(uint32_t tmem_d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl,
                                     uint32_t idesc, uint32_t accumulate) {
#define KIFMM_MMA3(GROUP, KIND)                                                                  \
  asm volatile(                                                                                  \
      "{\n.reg .pred p, t;\nsetp.ne.b32 p, %6, 0;\nsetp.eq.b32 t, %6, %6;\n"                \
      "tcgen05.mma.cta_group::" GROUP ".kind::" KIND " [%0], %1, %3, %5, p;\n"                 \
      KIFMM_MMA3_ORDER(GROUP, KIND)                                                              \
      "}" ::"r"(tmem_d),                                                                         \
      "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(accumulate))
  if constexpr (PAIR && ES == 4)
    KIFMM_MMA3("2", "tf32");
  else if constexpr (ES == 4)
    KIFMM_MMA3("1", "tf32");
  else if constexpr (PAIR)
    KIFMM_MMA3("2", "f16");
  else
    KIFMM_MMA3("1", "f16");
#undef KIFMM_MMA3
}

// Split accumulation of one K step (single CTA): main (=/+=) A_hi B_hi; corr (=/+=) A_hi B_lo; corr += A_lo B_hi.
template <int ES>
__device__ __forceinline__ void mma3_split(uint32_t d_main, uint32_t d_corr, uint64_t ah, uint64_t al, uint64_t bh,
                                           uint64_t bl, uint32_t idesc, uint32_t acc_main, uint32_t acc_corr) {
#define KIFMM_MMA3S(KIND)                                                                        \
  asm volatile(                                                                                  \
      "{\n.reg .pred p, q, t;\nsetp.ne.b32 p, %7, 0;\nsetp.ne.b32 q, %8, 0;\nsetp.eq.b32 t, %7, %7;\n" \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%0], %2, %4, %6, p;\n"                          \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%1], %2, %5, %6, q;\n"                          \
      "tcgen05.mma.cta_group::1.kind::" KIND " [%1], %3, %4, %6, t;\n"                          \
      "}" ::"r"(d_main), "r"(d_corr), "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(acc_main),   \
      "r"(acc_corr))
  if constexpr (ES == 4)
    KIFMM_MMA3S("tf32");
  else
    KIFMM_MMA3S("f16");
#undef KIFMM_MMA3S
}

// tcgen05.commit: arrive on `bar` (in both CTAs of the pair when PAIR) once prior MMAs complete
template <bool PAIR>
__device__ __forceinline__ void commit(uint32_t bar) {
  if constexpr (PAIR)
    asm volatile(
        "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(
            bar)
        : "memory");
  else
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void tma_tile(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  if constexpr (PAIR)
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, uint32_t bar, int col, int r0,
                                            int r1, int r2, int r3) {
  if constexpr (PAIR)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.cta_group::2 [%0], "
        "[%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
        "l"(map), "r"(bar), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
        "%5, %6, %7}], [%2];" ::"r"(dst),
        "l"(map), "r"(bar), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

template <int NP, bool PAIR, int ROWB, int ES>
__global__ void __maxnreg__(Regs<NP>::LAUNCH)
    m2l_tc_kernel(const __grid_constant__ CUtensorMap tm_khi, const __grid_constant__ CUtensorMap tm_klo,
                  const void* __restrict__ m_hi, const void* __restrict__ m_lo, const Item* __restrict__ items,
                  const int* __restrict__ sched, const int* __restrict__ seg_mat, const int* __restrict__ seg_in, int zero_row,
                  const float* __restrict__ row_unscale, float k_unscale, Epi epi) {
  using C = Cfg<NP, PAIR, ROWB, ES>;
  using AccT = Acc<NP, PAIR>;
  constexpr int KB = C::KB, NKB = C::NKB;
  constexpr int EPI_COLS = NP / 2;
  static_assert(NP % 32 == 0 && AccT::NSET * AccT::SET_COLS <= int(TMEM_COLS), "row width / TMEM budget");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  // bars: [0,S) full, [S,2S) empty, [2S,2S+2) tmem_full[b], [2S+2,2S+4) tmem_empty[b],
  //       [2S+4,3S+4) a_full (this CTA's A rows landed; PAIR only); then the TMEM address
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * C::STAGES + 2 * NACC);
  float* xmax = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES + 512);  // [2][2][128]
  float* tbuf = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES + 2560);  // !PAIR: [8 warps][32][20]
  float* s_colun = tbuf + (PAIR ? 0 : 8 * 32 * 20);                                   // !PAIR: [NP] col_unscale
  if (!PAIR && epi.direct_out && threadIdx.x < NP) s_colun[threadIdx.x] = epi.col_unscale[threadIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
#ifdef KIFMM_TC_PROBE  // experiments: phase timestamps of CTA 0 (globaltimer ns), printed at the end
  __shared__ unsigned long long probe[12];
  if (threadIdx.x < 12) probe[threadIdx.x] = 0;
  if (threadIdx.x == 0) probe[0] = globaltimer();
#define TC_PROBE(i, cond) \
  if ((cond) && blockIdx.x == 0) probe[i] = globaltimer();
#else
#define TC_PROBE(i, cond)
#endif
  // persistent: this CTA (pair) g0 runs the items sched[gs + 1 + k], k in [sched[g0], sched[g0 + 1]) -- a
  // longest-processing-time-first assignment made on the host; every role walks the same item sequence
  // with running stage (gi) and tap (gj) counters, so the pipeline runs on across item boundaries
  const int g0 = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int gs = PAIR ? int(gridDim.x >> 1) : int(gridDim.x);
  const int k_begin = sched[g0], k_end = sched[g0 + 1];
  const int* sched_list = sched + gs + 1;
  const int rows = C::CTAS * BM;  // rows per tile in seg_in / partial
  const uint32_t sbase = smem_u32(smem);
  auto a_hi = [&](int s) { return sbase + s * C::STAGE_BYTES; };
  auto a_lo = [&](int s) { return sbase + s * C::STAGE_BYTES + C::A_BYTES; };
  auto b_hi = [&](int s) { return sbase + s * C::STAGE_BYTES + 2 * C::A_BYTES; };
  auto b_lo = [&](int s) { return sbase + s * C::STAGE_BYTES + 2 * C::A_BYTES + C::B_BYTES; };
  auto full = [&](int s) { return smem_u32(&bars[s]); };
  auto empty = [&](int s) { return smem_u32(&bars[C::STAGES + s / C::EG]); };  // one barrier per stage group
  auto tfull = [&](int b) { return smem_u32(&bars[2 * C::STAGES + b]); };
  auto tempty = [&](int b) { return smem_u32(&bars[2 * C::STAGES + NACC + b]); };
  auto afull = [&](int s) { return smem_u32(&bars[2 * C::STAGES + 2 * NACC + s]); };
  // barriers the MMA waits on live in the leader; their cluster addresses
  auto leader = [&](uint32_t a) { return PAIR ? mapa(a, 0) : a; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      // full: the leader's arrive.expect_tx (B bytes of every CTA) + A arrivals: 128 producer threads
      // (single CTA) or one forwarder per CTA (pair)
      mbar_init(full(s), PAIR ? 1 + 2 : 1 + 128);
      mbar_init(empty(s), 1);  // one tcgen05.commit per stage (multicast to both CTAs when PAIR)
      mbar_init(afull(s), 128);
    }
    for (int b = 0; b < AccT::NSET; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), C::CTAS * EPI_WARPS);  // one elected lane per epilogue warp per CTA
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_khi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_klo) : "memory");
  }
  if (warp == 0) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  // set-up done (barriers, TMEM, tensor-map prefetch): let the next kernel start launching, then wait
  // for the previous one before reading the schedule's operands
  if (threadIdx.x == 0) pdl_trigger();
  pdl_wait();
  TC_PROBE(1, threadIdx.x == 0)
  timeline_begin(PAIR ? 1 : 2);
#ifdef KIFMM_TIMELINE_PROBES
  if (PAIR && blockIdx.x == 0 && threadIdx.x == 0 && g_timeline_on) {  // SM clock probe (experiments)
    g_timeline[8][0] = globaltimer();
    g_timeline[8][1] = clock64();
  }
#endif
  if (warp >= EPI_WARP0) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Regs<NP>::EPI));

    // ---------------- epilogue: per-tap promotion; warp w reads TMEM lanes 32*(w%4).. (its rows)
    //                  and columns [h*80, h*80+80), h = (w-6)/4
    const int q = warp & 3, h = (warp - EPI_WARP0) >> 2;
    const int row = q * 32 + lane;
    int b = 0;
    uint32_t tph = 0;
    for (int kk = k_begin; kk < k_end; ++kk) {
      const Item it = items[sched_list[kk]];
      const int ntap = it.seg_end - it.seg_begin;
      float acc[EPI_COLS];
#pragma unroll
      for (int k = 0; k < EPI_COLS; ++k) acc[k] = 0.f;
      // f16 kind: the per-row (source) and K_t power-of-two unscale of each tap, loaded one tap ahead
      auto unscale_of = [&](int j) {
        if constexpr (ES == 2) {
          const int sr = seg_in[size_t(it.seg_begin + j) * rows + rank * BM + row];
          return sr < 0 ? 0.f : row_unscale[sr] * k_unscale;
        }
        return 1.f;
      };
      float f_next = ntap > 0 ? unscale_of(0) : 1.f;
      for (int j = 0; j < ntap; ++j) {
        const float f = f_next;
        if (j + 1 < ntap) f_next = unscale_of(j + 1);
        mbar_wait_sleep(tfull(b), tph);
        TC_PROBE(4, warp == EPI_WARP0 && lane == 0 && kk == k_begin && j == 0)
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t taddr =
            tmem_base + (uint32_t(q * 32) << 16) + uint32_t(b * AccT::SET_COLS + h * EPI_COLS);
        auto ld16 = [&](uint32_t a, uint32_t (&v)[16]) {
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(a));
        };
        if constexpr (PAIR) {
#pragma unroll
          for (int cb = 0; cb < (TC_DBG(4) ? 0 : EPI_COLS / 16); ++cb) {
            uint32_t v[16];
            ld16(taddr + uint32_t(cb * 16), v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 16; ++k) acc[cb * 16 + k] = fmaf(__uint_as_float(v[k]), f, acc[cb * 16 + k]);
          }
        } else {  // (even + odd) + corrections, fp32 round-to-nearest; 8-column chunks of the three buffers
          auto ld8 = [&](uint32_t a, uint32_t (&v)[8]) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                           "=r"(v[7])
                         : "r"(a));
          };
#pragma unroll
          for (int cb = 0; cb < EPI_COLS / 8; ++cb) {
            uint32_t v0[8], v1[8], v2[8];
            ld8(taddr + uint32_t(cb * 8), v0);
            ld8(taddr + uint32_t(NP + cb * 8), v1);
            ld8(taddr + uint32_t(2 * NP + cb * 8), v2);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 8; ++k)
              acc[cb * 8 + k] = fmaf((__uint_as_float(v0[k]) + __uint_as_float(v1[k])) + __uint_as_float(v2[k]), f,
                                     acc[cb * 8 + k]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (PAIR)
            mbar_arrive_cluster(leader(tempty(b)));
          else
            mbar_arrive_local(tempty(b));
        }
        if (++b == AccT::NSET) {
          b = 0;
          tph ^= 1u;
        }
      }
      TC_PROBE(6, warp == EPI_WARP0 && lane == 0 && kk == k_begin)
      if (!PAIR && epi.direct_out) {
        // Direct GEMM epilogue, coalesced: a thread holds one output ROW, so row-per-thread global
        // loads / stores touch 32 rows (32 lines) per instruction -- 5-12 us per tile in the small
        // GEMMs (globaltimer probes, KIFMM_TC_PROBE).  The warp transposes its 32 x 80 block through
        // shared memory in 16-column chunks; lane (rr, sub) then owns rows rr + 8 i (i < 4) and
        // columns 4 sub .. 4 sub + 3 of every chunk, so one instruction covers 8 rows x 64 bytes.
        // Same operations per element as the row path below (bit-identical results).
        constexpr int TP = 20, NCH = EPI_COLS / 16;
        float* tb = tbuf + (warp - EPI_WARP0) * (32 * TP);
        const int sub = lane & 3, rr = lane >> 2;
        const int my_out = epi.direct_out[size_t(it.tile) * rows + row];
        int outs[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) outs[i] = __shfl_sync(0xffffffffu, my_out, rr + 8 * i);
        float* base = epi.dst ? epi.dst : epi.partial;
        float4 val[NCH][4];
        // transpose and column-unscale (shared memory only: no global load waits behind the __syncwarps)
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<float4*>(tb + lane * TP + 4 * j) =
                make_float4(acc[16 * c + 4 * j], acc[16 * c + 4 * j + 1], acc[16 * c + 4 * j + 2], acc[16 * c + 4 * j + 3]);
          __syncwarp();
          const float4 u = *reinterpret_cast<const float4*>(s_colun + h * EPI_COLS + 16 * c + 4 * sub);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float4 v = *reinterpret_cast<const float4*>(tb + (rr + 8 * i) * TP + 4 * sub);
            v.x *= u.x;
            v.y *= u.y;
            v.z *= u.z;
            v.w *= u.w;
            val[c][i] = v;
          }
        }
        TC_PROBE(10, warp == EPI_WARP0 && lane == 0 && kk == k_begin)
        if (epi.accumulate) {  // independent loads, one latency
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (outs[i] >= 0) {
                const float4 o = *reinterpret_cast<const float4*>(base + size_t(outs[i]) * NP + h * EPI_COLS + 16 * c +
                                                                  4 * sub);
                val[c][i].x += o.x;
                val[c][i].y += o.y;
                val[c][i].z += o.z;
                val[c][i].w += o.w;
              }
        }
        TC_PROBE(11, warp == EPI_WARP0 && lane == 0 && kk == k_begin)
        if (epi.dst) {
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (outs[i] >= 0)
                *reinterpret_cast<float4*>(epi.dst + size_t(outs[i]) * NP + h * EPI_COLS + 16 * c + 4 * sub) = val[c][i];
        }
        TC_PROBE(7, warp == EPI_WARP0 && lane == 0 && kk == k_begin)
        if (epi.split_hi) {
          float mx[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float m = 0.f;
#pragma unroll
            for (int c = 0; c < NCH; ++c)
              m = fmaxf(m, fmaxf(fmaxf(fabsf(val[c][i].x), fabsf(val[c][i].y)), fmaxf(fabsf(val[c][i].z), fabsf(val[c][i].w))));
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
            mx[i] = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
          }
          // row max over both column halves (partner warp: same lane quarter, other half), named barrier
          // 1 + q (64 threads); xmax is double-buffered by item parity
          float* xm = xmax + (kk & 1) * 256;
          if (sub == 0)
#pragma unroll
            for (int i = 0; i < 4; ++i) xm[h * 128 + q * 32 + rr + 8 * i] = mx[i];
          asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
          TC_PROBE(8, warp == EPI_WARP0 && lane == 0 && kk == k_begin)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (outs[i] < 0) continue;
            const float m = fmaxf(mx[i], xm[(1 - h) * 128 + q * 32 + rr + 8 * i]);
            const int e = f16_row_exponent(m);
            const float sc = ldexpf(1.f, e);
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
              const float x[4] = {val[c][i].x * sc, val[c][i].y * sc, val[c][i].z * sc, val[c][i].w * sc};
              uint32_t wh[2], wl[2];
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const __half h0 = __float2half_rn(x[2 * u]), h1 = __float2half_rn(x[2 * u + 1]);
                const __half2 hh = __halves2half2(h0, h1);
                const __half2 ll = __halves2half2(__float2half_rn(x[2 * u] - __half2float(h0)),
                                                  __float2half_rn(x[2 * u + 1] - __half2float(h1)));
                wh[u] = *reinterpret_cast<const uint32_t*>(&hh);
                wl[u] = *reinterpret_cast<const uint32_t*>(&ll);
              }
              const size_t o = size_t(outs[i]) * NP + h * EPI_COLS + 16 * c + 4 * sub;
              *reinterpret_cast<uint2*>(epi.split_hi + o) = make_uint2(wh[0], wh[1]);
              *reinterpret_cast<uint2*>(epi.split_lo + o) = make_uint2(wl[0], wl[1]);
            }
            if (h == 0 && sub == 0) epi.split_un[outs[i]] = ldexpf(1.f, -e);
          }
          TC_PROBE(9, warp == EPI_WARP0 && lane == 0 && kk == k_begin)
        }
      } else if (epi.direct_out) {
        const int out = epi.direct_out[size_t(it.tile) * rows + rank * BM + row];
        if (out >= 0) {
          // loads first (column unscale, then the old output row), stores last: no load waits behind a store
          float4* o4 = reinterpret_cast<float4*>((epi.dst ? epi.dst : epi.partial) + size_t(out) * NP + h * EPI_COLS);
          const float4* u4 = reinterpret_cast<const float4*>(epi.col_unscale + h * EPI_COLS);
#pragma unroll
          for (int k = 0; k < EPI_COLS / 4; ++k) {
            const float4 u = __ldg(u4 + k);
            acc[4 * k] *= u.x;
            acc[4 * k + 1] *= u.y;
            acc[4 * k + 2] *= u.z;
            acc[4 * k + 3] *= u.w;
          }
          if (epi.accumulate) {
#pragma unroll
            for (int k = 0; k < EPI_COLS / 4; ++k) {
              const float4 o = o4[k];
              acc[4 * k] += o.x;
              acc[4 * k + 1] += o.y;
              acc[4 * k + 2] += o.z;
              acc[4 * k + 3] += o.w;
            }
          }
          if (epi.dst) {
#pragma unroll
            for (int k = 0; k < EPI_COLS / 4; ++k)
              o4[k] = make_float4(acc[4 * k], acc[4 * k + 1], acc[4 * k + 2], acc[4 * k + 3]);
          }
        }
        TC_PROBE(7, warp == EPI_WARP0 && lane == 0 && kk == k_begin)
        if (epi.split_hi) {
          // row max over both column halves: the partner warp (same lane quarter, other half) meets
          // this one on named barrier 1 + q (64 threads); xmax is double-buffered by item parity
          float mx = 0.f;
          if (out >= 0) {
#pragma unroll
            for (int k = 0; k < EPI_COLS; ++k) mx = fmaxf(mx, fabsf(acc[k]));
          }
          float* xm = xmax + (kk & 1) * 256;
          xm[h * 128 + row] = mx;
          asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
          TC_PROBE(8, warp == EPI_WARP0 && lane == 0 && kk == k_begin)
          mx = fmaxf(mx, xm[(1 - h) * 128 + row]);
          if (out >= 0) {
            const int e = f16_row_exponent(mx);
            const float sc = ldexpf(1.f, e);
            uint4* ph = reinterpret_cast<uint4*>(epi.split_hi + size_t(out) * NP + h * EPI_COLS);
            uint4* pl = reinterpret_cast<uint4*>(epi.split_lo + size_t(out) * NP + h * EPI_COLS);
#pragma unroll
            for (int k = 0; k < EPI_COLS / 8; ++k) {  // 16-byte stores: 8 halves each
              uint32_t wh[4], wl[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float x0 = acc[8 * k + 2 * u] * sc, x1 = acc[8 * k + 2 * u + 1] * sc;
                const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
                const __half2 hh = __halves2half2(h0, h1);
                const __half2 ll =
                    __halves2half2(__float2half_rn(x0 - __half2float(h0)), __float2half_rn(x1 - __half2float(h1)));
                wh[u] = *reinterpret_cast<const uint32_t*>(&hh);
                wl[u] = *reinterpret_cast<const uint32_t*>(&ll);
              }
              ph[k] = make_uint4(wh[0], wh[1], wh[2], wh[3]);
              pl[k] = make_uint4(wl[0], wl[1], wl[2], wl[3]);
            }
            if (h == 0) epi.split_un[out] = ldexpf(1.f, -e);
          }
          TC_PROBE(9, warp == EPI_WARP0 && lane == 0 && kk == k_begin)
        }
      } else {
        float4* o4 =
            reinterpret_cast<float4*>(epi.partial + (size_t(it.slot) * rows + rank * BM + row) * NP + h * EPI_COLS);
#pragma unroll
        for (int k = 0; k < EPI_COLS / 4; ++k)
          o4[k] = make_float4(acc[4 * k], acc[4 * k + 1], acc[4 * k + 2], acc[4 * k + 3]);
      }
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Regs<NP>::LOW));
    if (warp == 0) {
      // ---------------- B producer: this CTA's rows of K_t hi/lo (TMA tile, swizzled); the whole warp
      //                  walks the loop (uniform values), one elected lane issues
      {
        int s = 0, kb = 0;
        uint32_t ph = 0;
        for (int kk = k_begin; kk < k_end; ++kk) {
          const Item it = items[sched_list[kk]];
          int mat_next = it.seg_end > it.seg_begin ? seg_mat[it.seg_begin] : 0;  // one tap ahead
          for (int seg = it.seg_begin; seg < it.seg_end; ++seg) {
            const int row = mat_next * NP + int(rank) * C::NB;
            if (seg + 1 < it.seg_end) mat_next = seg_mat[seg + 1];
            for (kb = 0; kb < NKB; ++kb) {
              mbar_wait(empty(s), ph ^ 1u);
              if (elect_one()) {
                if (TC_DBG(2)) {
                  if (rank == 0) mbar_expect_tx(full(s), 0);
                } else {
                  if (rank == 0) mbar_expect_tx(full(s), C::TX);
                  const uint32_t fb = leader(full(s));
                  tma_tile<PAIR>(b_hi(s), &tm_khi, fb, kb * KB, row);
                  tma_tile<PAIR>(b_lo(s), &tm_klo, fb, kb * KB, row);
                }
              }
              __syncwarp();
              if (++s == C::STAGES) {
                s = 0;
                ph ^= 1u;
              }
            }
          }
        }
      }
    } else if (warp == 1) {
      // ---------------- MMA issuer (leader only): a fresh accumulator per tap.  Kept short: the
      //                  tensor pipe waits on this one thread, and every instruction it issues competes
      //                  for its SMSP with the epilogue / producer warps (and co-resident blocks), so
      //                  the stage / parity counters run without div/mod, descriptors are a base plus
      //                  an offset, and the three MMAs of a K step are one asm block.
      if (rank == 0) {  // the whole warp walks the loop (warp-uniform values); one elected lane issues
        const bool prof = TC_DBG(8) != 0;
        unsigned long long t_all = clock64(), t_te = 0, t_fu = 0;
        const uint64_t dah0 = make_desc<ROWB>(a_hi(0)), dal0 = make_desc<ROWB>(a_lo(0));
        const uint64_t dbh0 = make_desc<ROWB>(b_hi(0)), dbl0 = make_desc<ROWB>(b_lo(0));
        constexpr uint64_t SD = uint64_t(C::STAGE_BYTES >> 4);  // descriptor start-address step per stage
        constexpr uint32_t IDESC = C::IDESC;
        int s = 0, gj = 0, ntaps = 0, nst = 0, ab = 0;
        uint32_t ph = 0, aph = 0;
        for (int kk = k_begin; kk < k_end; ++kk) {
          const Item it = items[sched_list[kk]];
          const int ntap = it.seg_end - it.seg_begin;
          for (int j = 0; j < ntap; ++j, ++gj) {
            unsigned long long c0 = prof ? clock64() : 0;
            mbar_wait(tempty(ab), aph ^ 1u);
            if (prof) t_te += clock64() - c0;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t d = tmem_base + uint32_t(ab * AccT::SET_COLS);
            for (int kb = 0; kb < NKB; ++kb) {
              c0 = prof ? clock64() : 0;
              mbar_wait(full(s), ph);
              TC_PROBE(2, lane == 0 && nst == 0)
              if (prof) t_fu += clock64() - c0;
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
              const uint64_t so = uint64_t(s) * SD;
              if (elect_one()) {
#pragma unroll
                for (int k = 0; k < ROWB / 32; ++k) {  // 32 bytes of K per MMA (8 tf32 / 16 f16)
                  const uint64_t o = so + uint64_t(2 * k);
                  if constexpr (PAIR) {
                    mma3<PAIR, ES>(d, dah0 + o, dal0 + o, dbh0 + o, dbl0 + o, IDESC, (kb > 0 || k > 0) ? 1u : 0u);
                  } else {  // K step ks: main buffer ks & 1, corrections in the third buffer
                    const int ks = kb * (ROWB / 32) + k;
                    mma3_split<ES>(d + uint32_t((ks & 1) * NP), d + uint32_t(2 * NP), dah0 + o, dal0 + o, dbh0 + o,
                                   dbl0 + o, IDESC, ks >= 2 ? 1u : 0u, ks >= 1 ? 1u : 0u);
                  }
                }
                if (s % C::EG == C::EG - 1) commit<PAIR>(empty(s));
              }
              __syncwarp();
              if (++s == C::STAGES) {
                s = 0;
                ph ^= 1u;
              }
              ++nst;
            }
            if (elect_one()) commit<PAIR>(tfull(ab));
            if (++ab == AccT::NSET) {
              ab = 0;
              aph ^= 1u;
            }
            __syncwarp();
            ++ntaps;
          }
        }
        TC_PROBE(3, lane == 0)
        if (prof && lane == 0)
          printf("cta %d: total %llu wait_tempty %llu wait_full %llu taps %d stages %d\n", int(blockIdx.x),
                 clock64() - t_all, t_te, t_fu, ntaps, nst);
      }
    } else if (warp >= PROD_WARP0 && warp < PROD_WARP0 + 4) {
      // ---------------- A producers: thread -> (16-byte chunk c, rows r0 + 16 j) of this CTA, cp.async
      //                  into the swizzled K-major layout; up to STAGES stages in flight per thread
      constexpr int CH = ROWB / 16;     // 16-byte chunks per row
      constexpr int RPI = 128 / CH;     // rows covered by the 128 producer threads per pass
      constexpr int J = BM / RPI;       // passes (rows per thread)
      const int t = threadIdx.x - 32 * PROD_WARP0;  // 0..127
      const int c = t % CH, r0 = t / CH;
      // per-thread constants: swizzled shared-memory offsets of its rows; per tap: the global byte
      // offsets of its gathered rows (zero-filled when absent); per stage only the K-block advances
      uint32_t soff[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int r = r0 + RPI * j;
        const int sw = ROWB == 128 ? (r & 7) : ((r & 7) >> 1);  // Swizzle<3,4,3> / Swizzle<2,4,3>
        soff[j] = uint32_t((r >> 3) * C::ATOM + (r & 7) * ROWB + ((c ^ sw) << 4));
      }
      const char* mh = static_cast<const char*>(m_hi) + c * 16;
      const char* ml = static_cast<const char*>(m_lo) + c * 16;
      size_t gofs[J];
      int gsz[J];
      int s = 0;
      uint32_t ph = 0;
      for (int kk = k_begin; kk < k_end; ++kk) {
        const Item it = items[sched_list[kk]];
        const int nstage = (it.seg_end - it.seg_begin) * NKB;
        int seg = it.seg_begin, kb = 0;
        // the gather rows of the next tap are loaded one tap ahead (their latency is otherwise exposed
        // at every tap start)
        int nxt[J];
#pragma unroll
        for (int j = 0; j < J; ++j) nxt[j] = seg < it.seg_end ? seg_in[size_t(seg) * rows + rank * BM + r0 + RPI * j] : -1;
        for (int i = 0; i < nstage; ++i) {
          if (kb == 0) {
#pragma unroll
            for (int j = 0; j < J; ++j) {
              const bool ok = nxt[j] >= 0;  // absent source: zero-fill, no global read
              gofs[j] = size_t(ok ? nxt[j] : zero_row) * (NP * ES);
              gsz[j] = ok ? 16 : 0;
            }
            if (seg + 1 < it.seg_end) {
#pragma unroll
              for (int j = 0; j < J; ++j) nxt[j] = seg_in[size_t(seg + 1) * rows + rank * BM + r0 + RPI * j];
            }
          }
#if KIFMM_TC_PROD_SLEEP
          mbar_wait_sleep(empty(s), ph ^ 1u);
#else
          mbar_wait(empty(s), ph ^ 1u);
#endif
          if (!TC_DBG(1)) {
            const uint32_t ahs = a_hi(s), als = a_lo(s);
            const size_t kbo = size_t(kb) * ROWB;
#pragma unroll
            for (int j = 0; j < J; ++j) {
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ahs + soff[j]),
                           "l"(mh + gofs[j] + kbo), "r"(gsz[j])
                           : "memory");
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(als + soff[j]),
                           "l"(ml + gofs[j] + kbo), "r"(gsz[j])
                           : "memory");
            }
          }
          // non-blocking: the barrier receives this thread's arrival when its copies have landed
          // (as CUTLASS's cp.async UMMA mainloops do; the full barrier's count includes these arrivals)
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(PAIR ? afull(s) : full(s))
                       : "memory");
          if (++s == C::STAGES) {
            s = 0;
            ph ^= 1u;
          }
          if (++kb == NKB) {
            kb = 0;
            ++seg;
          }
        }
      }
    } else if (warp == FWD_WARP) {
      // ---------------- forwarder (pair): this CTA's A rows landed -> one arrive on the leader's stage barrier
      if (PAIR) {
        int s = 0;
        uint32_t ph = 0;
        for (int kk = k_begin; kk < k_end; ++kk) {
          const Item it = items[sched_list[kk]];
          const int nstage = (it.seg_end - it.seg_begin) * NKB;
          for (int i = 0; i < nstage; ++i) {
            mbar_wait(afull(s), ph);
            if (elect_one()) mbar_arrive_cluster(leader(full(s)));
            __syncwarp();
            if (++s == C::STAGES) {
              s = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  }
  TC_PROBE(5, warp == EPI_WARP0 && lane == 0)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  timeline_end(PAIR ? 1 : 2);
#ifdef KIFMM_TC_PROBE
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("tcprobe pair=%d grid=%d items=%d setup %.2f first_full %.2f last_mma %.2f first_epi %.2f epi_end %.2f | item0: tmem done %.2f loads+dst %.2f xchg %.2f split %.2f us\n",
           int(PAIR), int(gridDim.x), k_end - k_begin, (probe[1] - probe[0]) * 1e-3, (probe[2] - probe[0]) * 1e-3,
           (probe[3] - probe[0]) * 1e-3, (probe[4] - probe[0]) * 1e-3, (probe[5] - probe[0]) * 1e-3,
           (probe[6] - probe[0]) * 1e-3, (probe[7] - probe[0]) * 1e-3, (probe[8] - probe[0]) * 1e-3,
           (probe[9] - probe[0]) * 1e-3);
  if (blockIdx.x == 0 && threadIdx.x == 0 && probe[10])
    printf("tcprobe   transposed %.2f accumulated %.2f\n", (probe[10] - probe[0]) * 1e-3, (probe[11] - probe[0]) * 1e-3);
#endif
#ifdef KIFMM_TIMELINE_PROBES
  if (PAIR && blockIdx.x == 0 && threadIdx.x == 0 && g_timeline_on) {
    g_timeline[9][0] = globaltimer();
    g_timeline[9][1] = clock64();
  }
#endif
  if (PAIR) cluster_sync();
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}


// x = hi + lo with hi = tf32(x) (round to nearest, ties away), lo exact in fp32.
__global__ void split_tf32_kernel(const float* __restrict__ x, size_t n, float* __restrict__ hi,
                                  float* __restrict__ lo) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = x[i];
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
  const float hv = __uint_as_float(h);
  hi[i] = hv;
  lo[i] = v - hv;
}

// Per operand row r in [r0, r1): scale by 2^e so max|row| lands in [2^9, 2^10) (far inside the fp16
// range), split x*2^e = hi + lo in fp16 (round to nearest), and record 2^-e.  Rows >= nn are zero rows
// (the appended gather target of absent sources).  One warp per row.
template <int NP>
__global__ void split_f16_rows_kernel(const float* __restrict__ M, int r0, int r1, int nn, __half* __restrict__ hi,
                                      __half* __restrict__ lo, float* __restrict__ unscale) {
  const int row = r0 + blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= r1) return;
  float v[NP / 32];
  float mx = 0.f;
#pragma unroll
  for (int k = 0; k < NP / 32; ++k) {
    v[k] = row < nn ? M[size_t(row) * NP + lane + 32 * k] : 0.f;
    mx = fmaxf(mx, fabsf(v[k]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0.f) {
    int ex;
    frexpf(mx, &ex);  // mx in [2^(ex-1), 2^ex)
    e = 10 - ex;
  }
  const float sc = ldexpf(1.f, e);
#pragma unroll
  for (int k = 0; k < NP / 32; ++k) {
    const float x = v[k] * sc;
    const __half h = __float2half_rn(x);
    hi[size_t(row) * NP + lane + 32 * k] = h;
    lo[size_t(row) * NP + lane + 32 * k] = __float2half_rn(x - __half2float(h));
  }
  if (lane == 0) unscale[row] = ldexpf(1.f, -e);
}

// Split the listed rows (warp per row).
template <int NP>
__global__ void split_f16_list_kernel(const float* __restrict__ X, const int* __restrict__ list, int n,
                                      __half* __restrict__ hi, __half* __restrict__ lo, float* __restrict__ un) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n) return;
  const int row = list[i];
  float v[NP / 32];
#pragma unroll
  for (int k = 0; k < NP / 32; ++k) v[k] = X[size_t(row) * NP + lane + 32 * k];
  split_row_warp<NP>(v, lane, size_t(row), hi, lo, un);
}

// check[out(r)] += sum over the tile's items (fixed order) of partial[slot][r], warp per row (grid
// (tiles, rows / 8), 256 threads); with hi set, also the fp16 split of the finished row.
template <int NP>
__global__ void m2l_tc_reduce_split_kernel(const float* __restrict__ partial, const int* __restrict__ tile_out,
                                           const int* __restrict__ tile_slot, int rows, float* __restrict__ check,
                                           __half* __restrict__ hi, __half* __restrict__ lo,
                                           float* __restrict__ un) {
  pdl_trigger();
  pdl_wait();
  const int tile = blockIdx.x;
  const int r = blockIdx.y * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int out = tile_out[size_t(tile) * rows + r];
  if (out < 0) return;
  const int s0 = tile_slot[tile], s1 = tile_slot[tile + 1];
  // check == nullptr: no P2L rows, the check rows would be zeros and only their split is read later --
  // neither read nor written (48 MB less traffic at config 2; 0.f + x keeps the sums bit-identical)
  float v[NP / 32];
#pragma unroll
  for (int k = 0; k < NP / 32; ++k) v[k] = check ? check[size_t(out) * NP + lane + 32 * k] : 0.f;
  for (int sl = s0; sl < s1; ++sl) {
    const float* pr = partial + (size_t(sl) * rows + r) * NP;
#pragma unroll
    for (int k = 0; k < NP / 32; ++k) v[k] += pr[lane + 32 * k];
  }
  if (check)
#pragma unroll
    for (int k = 0; k < NP / 32; ++k) check[size_t(out) * NP + lane + 32 * k] = v[k];
  if (hi) split_row_warp<NP>(v, lane, size_t(out), hi, lo, un);
}

// check[out(r)] += sum over the tile's items (fixed order) of partial[slot][r]
// grid (tiles, rows / 16); thread = (row, float4 column group), 640 threads
template <int NP>
__global__ void m2l_tc_reduce_kernel(const float* __restrict__ partial, const int* __restrict__ tile_out,
                                     const int* __restrict__ tile_slot, int rows, float* __restrict__ check) {
  const int tile = blockIdx.x;
  const int r = blockIdx.y * 16 + threadIdx.x / (NP / 4);
  const int c4 = threadIdx.x % (NP / 4);
  if (r >= rows) return;
  const int out = tile_out[size_t(tile) * rows + r];
  if (out < 0) return;
  const int s0 = tile_slot[tile], s1 = tile_slot[tile + 1];
  float4* dst = reinterpret_cast<float4*>(check + size_t(out) * NP) + c4;
  float4 acc = *dst;
  for (int s = s0; s < s1; ++s) {
    const float4 v = reinterpret_cast<const float4*>(partial + (size_t(s) * rows + r) * NP)[c4];
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  *dst = acc;
}

}  // namespace tc

// Longest-processing-time-first assignment of items (cost = taps + 1) to g persistent CTAs (pairs):
// returns [ptr (g + 1)][item lists], each list in decreasing cost.
inline std::vector<int> lpt_schedule(const std::vector<tc::Item>& items, int g) {
  std::vector<int> order(items.size());
  for (size_t i = 0; i < items.size(); ++i) order[i] = int(i);
  auto cost = [&](int i) { return int64_t(items[i].seg_end - items[i].seg_begin) + 1; };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost(a) > cost(b); });
  std::vector<std::vector<int>> lists(g);
  using E = std::pair<int64_t, int>;  // (load, cta)
  std::priority_queue<E, std::vector<E>, std::greater<E>> pq;
  for (int c = 0; c < g; ++c) pq.push({0, c});
  for (int i : order) {
    E e = pq.top();
    pq.pop();
    lists[e.second].push_back(i);
    pq.push({e.first + cost(i), e.second});
  }
  std::vector<int> out{0};
  for (int c = 0; c < g; ++c) out.push_back(out.back() + int(lists[c].size()));
  for (int c = 0; c < g; ++c) out.insert(out.end(), lists[c].begin(), lists[c].end());
  return out;
}

#ifdef KIFMM_EXPERIMENTS
inline int tc_debug() {  // experiments only: skips operand loads (wrong results), never in the product build
  static const int d = [] {
    const char* e = std::getenv("KIFMM_TC_DBG");
    return e ? std::atoi(e) : 0;
  }();
  return d;
}
#else
inline int tc_debug() { return 0; }
#endif

inline int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// launch attribute for programmatic dependent launch (KIFMM_PDL=0: ordinary stream order)
inline cudaLaunchAttribute pdl_attr() {  // read per launch (a captured graph keeps the choice of its capture)
  const char* env = std::getenv("KIFMM_PDL");
  const int on = env ? std::atoi(env) : 1;
  cudaLaunchAttribute a{};
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = on ? 1 : 0;
  return a;
}
template <class... KArgs, class... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1] = {pdl_attr()};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KIFMM_CUDA(cudaLaunchKernelEx(&cfg, k, args...));
}

inline bool m2l_tc_available() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0;
}

// Row widths (n_e padded to a multiple of 32) the tcgen05 kernels are instantiated for: p = 4, 5, 6 (M2L and
// the GEMM chain), and p = 7 (224) for the M2L 2-CTA pair kernel alone -- three 224-column accumulators of the
// single-CTA GEMM exceed the 512 TMEM columns.
inline bool tc_np_supported(int np) { return np == 64 || np == 128 || np == 160; }
inline bool tc_m2l_np_supported(int np) { return tc_np_supported(np) || np == 224; }
template <class F>
inline void tc_dispatch_m2l_np(int np, F&& f) {
  switch (np) {
    case 64: f(std::integral_constant<int, 64>{}); break;
    case 128: f(std::integral_constant<int, 128>{}); break;
    case 160: f(std::integral_constant<int, 160>{}); break;
    case 224: f(std::integral_constant<int, 224>{}); break;
    default: throw InvalidArgument("tcgen05 M2L: row width (n_e padded to 32) must be 64, 128, 160 or 224 (p = 4..7)");
  }
}
template <class F>
inline void tc_dispatch_np(int np, F&& f) {
  switch (np) {
    case 64: f(std::integral_constant<int, 64>{}); break;
    case 128: f(std::integral_constant<int, 128>{}); break;
    case 160: f(std::integral_constant<int, 160>{}); break;
    default: throw InvalidArgument("tcgen05 path: row width (n_e padded to 32) must be 64, 128 or 160 (p = 4, 5, 6)");
  }
}

// fp32 operand rows split for the kind::f16 GEMMs: rows+1 rows (the last one zero) of hi / lo fp16 and
// the per-row power-of-two unscale.
struct TcSplit {
  __half *hi = nullptr, *lo = nullptr;
  float* un = nullptr;
  int rows = 0, np = 0;
  TcSplit() = default;
  TcSplit(const TcSplit&) = delete;
  TcSplit& operator=(const TcSplit&) = delete;
  ~TcSplit() {
    for (void* p : {(void*)hi, (void*)lo, (void*)un})
      if (p) cudaFree(p);
  }
  void alloc(int r, int width, size_t* total) {
    if (!tc_np_supported(width)) throw InvalidArgument("TcSplit: unsupported row width");
    rows = r;
    np = width;
    const size_t n = size_t(r + 1) * np;
    KIFMM_CUDA(cudaMalloc(&hi, n * sizeof(__half)));
    KIFMM_CUDA(cudaMalloc(&lo, n * sizeof(__half)));
    KIFMM_CUDA(cudaMalloc(&un, size_t(r + 1) * sizeof(float)));
    // all zero: the appended zero row, and rows a plan never writes read as zero rows
    KIFMM_CUDA(cudaMemset(hi, 0, n * sizeof(__half)));
    KIFMM_CUDA(cudaMemset(lo, 0, n * sizeof(__half)));
    KIFMM_CUDA(cudaMemset(un, 0, size_t(r + 1) * sizeof(float)));
    *total += 2 * n * sizeof(__half) + size_t(r + 1) * sizeof(float);
  }
  // split rows [r0, r1) of the fp32 buffer X (row stride NP)
  void split(const float* X, int r0, int r1, cudaStream_t s) const {
    if (r1 <= r0) return;
    tc_dispatch_np(np, [&](auto w) {
      tc::split_f16_rows_kernel<decltype(w)::value><<<unsigned((r1 - r0 + 7) / 8), 256, 0, s>>>(X, r0, r1, rows, hi, lo, un);
    });
    KIFMM_LAUNCH_CHECK();
  }
};

// Host side: tiles/items, split operators, TMA descriptors.
struct M2LTcPlan {
  bool pair = false;  // 2-CTA (cta_group::2) kernel on large trees; KIFMM_TC_PAIR=0/1 forces the choice
  int rows = 256;    // output rows per tile
  int np = 0;        // row width (n_e padded to 32): 64, 128 or 160
  int rowb = 128;    // bytes per operand row per stage (128: SWIZZLE_128B, 64: SWIZZLE_64B)
  bool f16 = true;  // 3-term fp16 split (kind::f16) with power-of-two row scaling; KIFMM_TC_KIND=tf32 for 3xTF32
  float k_scale = 256.f;  // power of two that puts max |K_t| in [2^6, 2^7) before the fp16 split (256 for a unit domain)
  __half *d_khi16 = nullptr, *d_klo16 = nullptr, *d_mhi16 = nullptr, *d_mlo16 = nullptr;
  float* d_unscale = nullptr;
  CUtensorMap tm_khi16{}, tm_klo16{};
  int n_items = 0, n_tiles = 0, n_segs = 0;
  int sched_g = 0;         // persistent CTAs (pairs) of the tcgen05 kernel
  int* d_sched = nullptr;  // lpt_schedule(items, sched_g)
  size_t nn = 0;
  float *d_khi = nullptr, *d_klo = nullptr, *d_mhi = nullptr, *d_mlo = nullptr, *d_partial = nullptr;
  int *d_tile_out = nullptr, *d_tile_slot = nullptr, *d_seg_mat = nullptr, *d_seg_in = nullptr;
  tc::Item* d_items = nullptr;
  CUtensorMap tm_khi{}, tm_klo{};
  int64_t slots = 0;

  ~M2LTcPlan() {
    for (void* p : {(void*)d_khi, (void*)d_klo, (void*)d_mhi, (void*)d_mlo, (void*)d_partial, (void*)d_tile_out,
                    (void*)d_tile_slot, (void*)d_seg_mat, (void*)d_seg_in, (void*)d_items, (void*)d_khi16,
                    (void*)d_klo16, (void*)d_mhi16, (void*)d_mlo16, (void*)d_unscale, (void*)d_sched})
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

  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

  static void encode(EncodeFn fn, CUtensorMap* m, void* base, int np, uint64_t rows_total, uint32_t box_rows, int rowb,
                     int es = 4) {
    const cuuint64_t dims[2] = {cuuint64_t(np), cuuint64_t(rows_total)};
    const cuuint64_t strides[1] = {cuuint64_t(np) * es};
    const cuuint32_t box[2] = {cuuint32_t(rowb / es), box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(m, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base,
                          dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE,
                          rowb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw DeviceError(KIFMM_E_CUDA, "cuTensorMapEncodeTiled failed");
  }

  // Tile-aligned sub-groups of one large (level, octant) group.  Its targets fall into tap-set classes:
  // interior (all transfer vectors of the octant), and boundary classes whose parents touch domain
  // faces, edges, corners -- each a subset of the interior set.  A tile pays for the union of its rows'
  // taps, so a tile straddling two face classes pays for most of the interior set on every row.  Here:
  // whole tiles of interior rows; then each boundary class (largest first) with the unplaced classes
  // that are subsets of it and still fit in its last tile; then the interior tail; then what is left.
  // Config 2, level 5: 6.06 M -> 5.75 M computed pair slots (5.40 M real).
  // Applied only where it pays: at most 64 distinct tap sets (uniform regions; adaptive trees have
  // thousands, and per-class tiles would multiply the padding -- config 5 M2L 18 -> 207 ms), and only
  // when the computed slots (sum over tiles of rows x |union of taps|) drop.
  template <class TreeView>
  void split_by_face(const TreeView& t, const std::vector<int64_t>& grp, std::vector<std::vector<int64_t>>& out) {
    constexpr int NW = (316 + 63) / 64;
    using Sig = std::array<uint64_t, NW>;
    auto sig_of = [&](int64_t b) {
      Sig sg{};
      for (int64_t e = t.v_ptr[b]; e < t.v_ptr[b + 1]; ++e) sg[t.v_tv[e] >> 6] |= uint64_t(1) << (t.v_tv[e] & 63);
      return sg;
    };
    auto pop = [](const Sig& x) {
      int c = 0;
      for (uint64_t w : x) c += __builtin_popcountll(w);
      return c;
    };
    auto slots_of = [&](const std::vector<std::vector<int64_t>>& gs) {
      int64_t tot = 0;
      for (const auto& g : gs)
        for (size_t s0 = 0; s0 < g.size(); s0 += size_t(rows)) {
          Sig u{};
          for (size_t r = s0; r < std::min(g.size(), s0 + size_t(rows)); ++r) {
            const Sig x = sig_of(g[r]);
            for (int w = 0; w < NW; ++w) u[w] |= x[w];
          }
          tot += int64_t(rows) * pop(u);
        }
      return tot;
    };
    std::map<Sig, std::vector<int64_t>> bys;
    for (int64_t b : grp) {
      bys[sig_of(b)].push_back(b);
      if (bys.size() > 64) {
        out.push_back(grp);
        return;
      }
    }
    std::vector<std::vector<int64_t>> cand;
    std::vector<const Sig*> sets;
    for (auto& kv : bys) sets.push_back(&kv.first);
    std::stable_sort(sets.begin(), sets.end(), [&](const Sig* a, const Sig* b) { return pop(*a) > pop(*b); });
    auto subset = [](const Sig& a, const Sig& b) {  // a within b
      for (int w = 0; w < NW; ++w)
        if (a[w] & ~b[w]) return false;
      return true;
    };
    std::set<const Sig*> placed{sets[0]};
    const std::vector<int64_t>& inter = bys[*sets[0]];
    const size_t full = inter.size() / size_t(rows) * size_t(rows);
    if (full) cand.emplace_back(inter.begin(), inter.begin() + full);
    for (size_t i = 1; i < sets.size(); ++i) {
      if (placed.count(sets[i])) continue;
      placed.insert(sets[i]);
      std::vector<int64_t> ch = bys[*sets[i]];
      for (size_t j = 1; j < sets.size(); ++j) {
        if (placed.count(sets[j]) || !subset(*sets[j], *sets[i])) continue;
        const size_t cap = (ch.size() + size_t(rows) - 1) / size_t(rows) * size_t(rows);
        if (ch.size() + bys[*sets[j]].size() > cap) continue;
        placed.insert(sets[j]);
        ch.insert(ch.end(), bys[*sets[j]].begin(), bys[*sets[j]].end());
      }
      cand.push_back(std::move(ch));
    }
    if (full < inter.size()) cand.emplace_back(inter.begin() + full, inter.end());
    std::vector<int64_t> left;
    for (const Sig* sg : sets)
      if (!placed.count(sg)) left.insert(left.end(), bys[*sg].begin(), bys[*sg].end());
    if (!left.empty()) cand.push_back(std::move(left));
    if (slots_of(cand) < slots_of({grp}))
      for (auto& g : cand) out.push_back(std::move(g));
    else
      out.push_back(grp);
  }

  template <class TreeView, class OpsView>
  void build(const TreeView& t, const std::vector<std::vector<int64_t>>& groups, int width, const OpsView& ops,
             size_t* total, bool own_split = true) {
    if (!tc_m2l_np_supported(width))
      throw InvalidArgument("tcgen05 M2L: instantiated for p = 4, 5, 6, 7 (n_e padded to 64, 128, 160, 224)");
    np = width;
    // KIFMM_TC_KIND=tf32: the kind::tf32 variant (reported as m2l_backend 3), instantiated for p = 6 only
    if (const char* e = std::getenv("KIFMM_TC_KIND")) f16 = std::string(e) != "tf32" || np != 160;
    nn = size_t(t.n_nodes);
    pair = nn >= 20000;  // 2-CTA pays off once there are enough 256-row tiles (measured at 1e5 / 1e6 points)
    if (const char* e = std::getenv("KIFMM_TC_PAIR")) pair = std::atoi(e) != 0;
    if (width > 160) pair = true;  // row width 224: only the 2-CTA pair kernel is instantiated
    rows = pair ? 2 * tc::BM : tc::BM;
    // ---- tiles (rows same-class targets) and their tap segments
    std::vector<int> tile_out, seg_mat, seg_in, tile_seg{0};
    // Inside a (level, octant) group, targets with the same transfer-vector set are made contiguous
    // (signature = hash of the sorted tap list; ties keep Z-order), so a tile's taps are present for
    // (nearly) all of its rows: boundary targets no longer pad interior tiles with zero rows.
    bool by_sig = true;
    if (const char* e = std::getenv("KIFMM_TC_SIG")) by_sig = std::atoi(e) != 0;
    bool by_face = true;  // KIFMM_TC_FACE=0: large groups as one sorted run (tiles straddle tap sets)
    if (const char* e = std::getenv("KIFMM_TC_FACE")) by_face = std::atoi(e) != 0;
    std::vector<std::vector<int64_t>> sorted_groups;
    for (const auto& g0 : groups) {
      std::vector<int64_t> grp(g0.begin(), g0.end());
      if (by_sig) {
        std::vector<std::pair<uint64_t, int64_t>> key(grp.size());
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < int64_t(grp.size()); ++i) {
          const int64_t b = grp[i];
          uint64_t bits[(316 + 63) / 64] = {};  // order-free signature: the set of transfer vectors
          for (int64_t e = t.v_ptr[b]; e < t.v_ptr[b + 1]; ++e) bits[t.v_tv[e] >> 6] |= uint64_t(1) << (t.v_tv[e] & 63);
          uint64_t h = 1469598103934665603ull;
          for (uint64_t w : bits) h = (h ^ w) * 1099511628211ull;
          key[i] = {h, b};
        }
        std::stable_sort(key.begin(), key.end(),
                         [](const auto& x, const auto& y) { return x.first < y.first; });
        for (size_t i = 0; i < grp.size(); ++i) grp[i] = key[i].second;
      }
      if (by_face && int64_t(grp.size()) >= 8 * int64_t(rows)) {
        split_by_face(t, grp, sorted_groups);
        continue;
      }
      sorted_groups.push_back(std::move(grp));
    }
    // tiles: (group, first row); built in two parallel passes (tap sets, then the rows)
    std::vector<std::pair<int, size_t>> tiles_def;
    for (int gi = 0; gi < int(sorted_groups.size()); ++gi)
      for (size_t s0 = 0; s0 < sorted_groups[gi].size(); s0 += size_t(rows)) tiles_def.push_back({gi, s0});
    const int nt_tiles = int(tiles_def.size());
    std::vector<std::vector<int>> tile_taps(nt_tiles);
#pragma omp parallel for schedule(dynamic, 16)
    for (int ti = 0; ti < nt_tiles; ++ti) {
      const auto& grp = sorted_groups[tiles_def[ti].first];
      const size_t s0 = tiles_def[ti].second;
      uint64_t bits[(316 + 63) / 64] = {};
      for (int r = 0; r < rows && s0 + r < grp.size(); ++r)
        for (int64_t e = t.v_ptr[grp[s0 + r]]; e < t.v_ptr[grp[s0 + r] + 1]; ++e)
          bits[t.v_tv[e] >> 6] |= uint64_t(1) << (t.v_tv[e] & 63);
      for (int w = 0; w < (316 + 63) / 64; ++w)  // ascending transfer-vector id
        for (uint64_t m = bits[w]; m; m &= m - 1) tile_taps[ti].push_back(64 * w + __builtin_ctzll(m));
    }
    tile_seg.assign(nt_tiles + 1, 0);
    for (int ti = 0; ti < nt_tiles; ++ti) tile_seg[ti + 1] = tile_seg[ti] + int(tile_taps[ti].size());
    tile_out.assign(size_t(nt_tiles) * rows, -1);
    seg_mat.assign(tile_seg[nt_tiles], 0);
    seg_in.assign(size_t(tile_seg[nt_tiles]) * rows, -1);
#pragma omp parallel for schedule(dynamic, 16)
    for (int ti = 0; ti < nt_tiles; ++ti) {
      const auto& grp = sorted_groups[tiles_def[ti].first];
      const size_t s0 = tiles_def[ti].second;
      int slot[316];
      for (size_t k = 0; k < tile_taps[ti].size(); ++k) {
        slot[tile_taps[ti][k]] = tile_seg[ti] + int(k);
        seg_mat[tile_seg[ti] + k] = tile_taps[ti][k];
      }
      for (int r = 0; r < rows && s0 + r < grp.size(); ++r) {
        const int64_t b = grp[s0 + r];
        tile_out[size_t(ti) * rows + r] = int(b);
        for (int64_t e = t.v_ptr[b]; e < t.v_ptr[b + 1]; ++e)
          seg_in[size_t(slot[t.v_tv[e]]) * rows + r] = int(t.v_idx[e]);
      }
    }
    n_tiles = int(tile_seg.size()) - 1;
    n_segs = int(seg_mat.size());
    slots = int64_t(n_segs) * rows;
    // ---- items and their schedule over the persistent CTAs (pairs).  Default: McNaughton's wrap-around
    //      rule -- tiles are laid end to end (taps as the unit of work) and cut into G consecutive bins of
    //      equal length, so every CTA gets the same number of taps (+- 1) and a tile is split only where a
    //      bin boundary falls (few partial slots).  KIFMM_TC_SCHED=lpt: fixed-size chunks (KIFMM_TC_CHUNK)
    //      assigned longest-first (the previous scheme; up to one chunk of imbalance).
    const int G = std::max(1, pair ? sm_count() / 2 : sm_count());
    bool wrap = true;
    if (const char* e = std::getenv("KIFMM_TC_SCHED")) wrap = std::string(e) != "lpt";
    std::vector<tc::Item> items;
    std::vector<int> tile_slot{0};
    std::vector<int> sched;
    if (wrap) {
      const int64_t total_taps = n_segs;
      const int bins = int(std::max<int64_t>(1, std::min<int64_t>(G, total_taps)));
      std::vector<std::vector<int>> lists(bins);
      int bin = 0;
      int64_t fill = 0;
      const int64_t cap = (total_taps + bins - 1) / bins;
      for (int ti = 0; ti < n_tiles; ++ti) {
        int a = tile_seg[ti];
        const int b = tile_seg[ti + 1];
        while (a < b) {
          const int take = int(std::min<int64_t>(b - a, cap - fill));
          lists[bin].push_back(int(items.size()));
          items.push_back({ti, a, a + take, int(items.size())});
          a += take;
          fill += take;
          if (fill == cap && bin + 1 < bins) {
            ++bin;
            fill = 0;
          }
        }
        tile_slot.push_back(int(items.size()));
      }
      sched_g = bins;
      sched.push_back(0);
      for (auto& l : lists) sched.push_back(sched.back() + int(l.size()));
      for (auto& l : lists) sched.insert(sched.end(), l.begin(), l.end());
    } else {
      const int64_t target_items = int64_t(8) * G;
      int chunk = int(std::max<int64_t>(8, (n_segs + target_items - 1) / std::max<int64_t>(1, target_items)));
      if (const char* e = std::getenv("KIFMM_TC_CHUNK")) chunk = std::max(1, std::atoi(e));
      for (int ti = 0; ti < n_tiles; ++ti) {
        const int a = tile_seg[ti], b = tile_seg[ti + 1];
        const int pieces = std::max(1, (b - a + chunk - 1) / chunk);
        for (int pc = 0; pc < pieces; ++pc) {
          const int sa = a + int(int64_t(b - a) * pc / pieces), sb = a + int(int64_t(b - a) * (pc + 1) / pieces);
          items.push_back({ti, sa, sb, int(items.size())});
        }
        tile_slot.push_back(int(items.size()));
      }
      // longest first (slots keep the fixed reduction order)
      std::stable_sort(items.begin(), items.end(), [](const tc::Item& x, const tc::Item& y) {
        return (x.seg_end - x.seg_begin) > (y.seg_end - y.seg_begin);
      });
      sched_g = std::max(1, std::min(int(items.size()), G));
      sched = lpt_schedule(items, sched_g);
    }
    n_items = int(items.size());
    up(&d_tile_out, tile_out, total);
    up(&d_tile_slot, tile_slot, total);
    up(&d_seg_mat, seg_mat, total);
    up(&d_seg_in, seg_in, total);
    up(&d_items, items, total);
    up(&d_sched, sched, total);
    // ---- operators and A-operand buffers of the chosen kind only (the other kind's 2 x 32 MB of K_t and
    //      2 x n_nodes rows are neither built nor allocated)
    const int ne = ops.n_e, nc = ops.n_c, nt = ops.n_m2l;
    KIFMM_CUDA(cudaMalloc(&d_partial, std::max(1, n_items) * size_t(rows) * np * sizeof(float)));
    *total += size_t(n_items) * rows * np * sizeof(float);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    KIFMM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn) throw DeviceError(KIFMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (const char* e = std::getenv("KIFMM_TC_ROWB")) rowb = std::atoi(e) == 64 ? 64 : 128;
    const uint32_t brow = uint32_t(pair ? np / 2 : np);
    const size_t kn = size_t(nt) * np * np;
    if (!f16) {
      // kind::tf32 (m2l_backend 3, p = 6 only): K_t split into tf32 hi / lo, padded to np x np per
      // transfer vector; multipole hi / lo with one appended zero row (gather target of absent sources)
      std::vector<float> khi(kn, 0.f), klo(kn, 0.f);
#pragma omp parallel for schedule(static)
      for (int v = 0; v < nt; ++v)
        for (int c = 0; c < nc; ++c)
          for (int e = 0; e < ne; ++e) {
            const float x = float(ops.m2l[(size_t(v) * nc + c) * ne + e]);
            const float h = tf32_rna(x);
            const size_t idx = (size_t(v) * np + c) * np + e;
            khi[idx] = h;
            klo[idx] = x - h;
          }
      up(&d_khi, khi, total);
      up(&d_klo, klo, total);
      KIFMM_CUDA(cudaMalloc(&d_mhi, (nn + 1) * np * sizeof(float)));
      KIFMM_CUDA(cudaMalloc(&d_mlo, (nn + 1) * np * sizeof(float)));
      KIFMM_CUDA(cudaMemset(d_mhi + nn * np, 0, np * sizeof(float)));
      KIFMM_CUDA(cudaMemset(d_mlo + nn * np, 0, np * sizeof(float)));
      *total += 2 * (nn + 1) * np * sizeof(float);
      // TMA descriptors (SWIZZLE_128B / 64B, 32- / 16-float boxes): K_t tiles of this CTA's rows
      encode(reinterpret_cast<EncodeFn>(fn), &tm_khi, d_khi, np, uint64_t(nt) * np, brow, rowb);
      encode(reinterpret_cast<EncodeFn>(fn), &tm_klo, d_klo, np, uint64_t(nt) * np, brow, rowb);
      set_smem<false, 128>();
      set_smem<true, 128>();
      set_smem<false, 64>();
      set_smem<true, 64>();
    } else {
      // kind::f16: K_t * 2^8 split into fp16 hi / lo (padded to np x np); multipoles are split per row
      // with a power-of-two scale -- by the caller (launch_presplit) or, with own_split, into this
      // plan's own buffers (launch)
      // K_t scales with 1 / (domain side): the power-of-two scale follows its largest entry, so the split keeps
      // its 22 bits for any domain (a fixed 2^8 overflowed fp16 for a domain of side 1e-4 and lost 5 bits at 1e4)
      double kmax = 0.0;
      for (size_t i = 0; i < size_t(nt) * nc * ne; ++i) kmax = std::max(kmax, std::fabs(double(ops.m2l[i])));
      if (kmax > 0.0 && std::isfinite(kmax)) {
        int ex = 0;
        std::frexp(kmax, &ex);  // kmax in [2^(ex-1), 2^ex)
        k_scale = float(std::ldexp(1.0, 7 - ex));
      }
      const float kKScale = k_scale;
      std::vector<__half> h16(kn, __float2half_rn(0.f)), l16(kn, __float2half_rn(0.f));
#pragma omp parallel for schedule(static)
      for (int v = 0; v < nt; ++v)
        for (int c = 0; c < nc; ++c)
          for (int e = 0; e < ne; ++e) {
            const float x = float(ops.m2l[(size_t(v) * nc + c) * ne + e]) * kKScale;
            const __half h = __float2half_rn(x);
            const size_t idx = (size_t(v) * np + c) * np + e;
            h16[idx] = h;
            l16[idx] = __float2half_rn(x - __half2float(h));
          }
      up(&d_khi16, h16, total);
      up(&d_klo16, l16, total);
      if (own_split) {
        KIFMM_CUDA(cudaMalloc(&d_mhi16, (nn + 1) * np * sizeof(__half)));
        KIFMM_CUDA(cudaMalloc(&d_mlo16, (nn + 1) * np * sizeof(__half)));
        KIFMM_CUDA(cudaMalloc(&d_unscale, (nn + 1) * sizeof(float)));
        *total += 2 * (nn + 1) * np * sizeof(__half) + (nn + 1) * sizeof(float);
      }
      encode(reinterpret_cast<EncodeFn>(fn), &tm_khi16, d_khi16, np, uint64_t(nt) * np, brow, 64, 2);
      encode(reinterpret_cast<EncodeFn>(fn), &tm_klo16, d_klo16, np, uint64_t(nt) * np, brow, 64, 2);
      tc_dispatch_m2l_np(np, [&](auto w) {
        constexpr int W = decltype(w)::value;
        if (pair) {
          KIFMM_CUDA(cudaFuncSetAttribute(tc::m2l_tc_kernel<W, true, 64, 2>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          tc::Cfg<W, true, 64, 2>::SMEM_BYTES));
        } else if constexpr (W <= 160) {
          KIFMM_CUDA(cudaFuncSetAttribute(tc::m2l_tc_kernel<W, false, 64, 2>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          tc::Cfg<W, false, 64, 2>::SMEM_BYTES));
        }
      });
    }
  }

  template <bool P, int R>
  static void set_smem() {
    KIFMM_CUDA(cudaFuncSetAttribute(tc::m2l_tc_kernel<160, P, R, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    tc::Cfg<160, P, R, 4>::SMEM_BYTES));
  }
  template <int W, bool P, int R, int ES = 4>
  void run_kernel(cudaStream_t s, const void* ah_ext = nullptr, const void* al_ext = nullptr,
                  const float* un_ext = nullptr) {
    const CUtensorMap& mh = ES == 4 ? tm_khi : tm_khi16;
    const CUtensorMap& ml = ES == 4 ? tm_klo : tm_klo16;
    const void* ah = ah_ext ? ah_ext : ES == 4 ? static_cast<const void*>(d_mhi) : static_cast<const void*>(d_mhi16);
    const void* al = al_ext ? al_ext : ES == 4 ? static_cast<const void*>(d_mlo) : static_cast<const void*>(d_mlo16);
    const float* un = un_ext ? un_ext : ES == 4 ? nullptr : d_unscale;
    const float ku = ES == 4 ? 1.f : 1.f / k_scale;
    if (P) {
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      attr[1] = pdl_attr();
      cfg.gridDim = dim3(2 * sched_g);
      cfg.blockDim = dim3(tc::THREADS);
      cfg.dynamicSmemBytes = tc::Cfg<W, P, R, ES>::SMEM_BYTES;
      cfg.stream = s;
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      KIFMM_CUDA(cudaLaunchKernelEx(&cfg, tc::m2l_tc_kernel<W, P, R, ES>, mh, ml, ah, al, (const tc::Item*)d_items, (const int*)d_sched,
                                    (const int*)d_seg_mat, (const int*)d_seg_in, int(nn), un, ku,
                                    tc::Epi{d_partial, nullptr, nullptr, nullptr, 0, tc_debug(), nullptr, nullptr, nullptr}));
    } else {
      launch_pdl(tc::m2l_tc_kernel<W, P, R, ES>, dim3(sched_g), dim3(tc::THREADS), tc::Cfg<W, P, R, ES>::SMEM_BYTES, s, mh, ml,
                 ah, al, (const tc::Item*)d_items, (const int*)d_sched, (const int*)d_seg_mat, (const int*)d_seg_in,
                 int(nn), un, ku, tc::Epi{d_partial, nullptr, nullptr, nullptr, 0, tc_debug(), nullptr, nullptr, nullptr});
    }
    KIFMM_LAUNCH_CHECK();
  }

  // check += M2L(M) with the multipoles already split into sp (rows = n_nodes, kind::f16 plan); the
  // reduce also writes the fp16 split of the finished check rows into cd (when given)
  void launch_presplit(const TcSplit& sp, float* check, const TcSplit* cd, cudaStream_t s) {
    launch_presplit_main(sp, s);
    launch_presplit_reduce(check, cd, s);
  }
  // the two halves of launch_presplit: the tcgen05 items (partials only: they neither read nor write the check
  // rows, so P2L may fill those concurrently), then the fixed-order reduction into the check rows (+ split)
  void launch_presplit_main(const TcSplit& sp, cudaStream_t s) {
    if (!n_items) return;
    if (!f16 || sp.rows != int(nn)) throw InvalidArgument("M2L presplit: kind::f16 plan over all nodes required");
    if (sp.np != np) throw InvalidArgument("M2L presplit: row width mismatch");
    tc_dispatch_np(np, [&](auto w) {  // presplit operands come from the GEMM chain: widths <= 160
      if (pair)
        run_kernel<decltype(w)::value, true, 64, 2>(s, sp.hi, sp.lo, sp.un);
      else
        run_kernel<decltype(w)::value, false, 64, 2>(s, sp.hi, sp.lo, sp.un);
    });
  }
  void launch_presplit_reduce(float* check, const TcSplit* cd, cudaStream_t s) {
    if (!n_items) return;
    tc_dispatch_np(np, [&](auto w) {
      launch_pdl(tc::m2l_tc_reduce_split_kernel<decltype(w)::value>, dim3(n_tiles, (rows + 7) / 8), dim3(256), 0, s,
                 (const float*)d_partial, (const int*)d_tile_out, (const int*)d_tile_slot, rows, check,
                 cd ? cd->hi : (__half*)nullptr, cd ? cd->lo : (__half*)nullptr, cd ? cd->un : (float*)nullptr);
    });
    KIFMM_LAUNCH_CHECK();
  }

  // check += M2L(M): run the tcgen05 items, reduce partials.
  void launch(const float* M, float* check, int width, cudaStream_t s) {
    if (!n_items) return;
    if (width != np) throw InvalidArgument("M2L launch: row width mismatch");
    if (f16 && !d_mhi16) throw InvalidArgument("M2L launch: plan was built without its own split buffers");
    if (f16) {
      tc_dispatch_m2l_np(np, [&](auto w) {
        constexpr int W = decltype(w)::value;
        tc::split_f16_rows_kernel<W><<<unsigned((nn + 8) / 8), 256, 0, s>>>(M, 0, int(nn) + 1, int(nn), d_mhi16, d_mlo16,
                                                                            d_unscale);
        KIFMM_LAUNCH_CHECK();
        if (pair) run_kernel<W, true, 64, 2>(s);
        if constexpr (W <= 160)
          if (!pair) run_kernel<W, false, 64, 2>(s);
        tc::m2l_tc_reduce_kernel<W><<<dim3(n_tiles, rows / 16), 16 * (W / 4), 0, s>>>(d_partial, d_tile_out, d_tile_slot,
                                                                                    rows, check);
      });
      KIFMM_LAUNCH_CHECK();
      return;
    }
    // kind::tf32 (3xTF32, m2l_backend 3): p = 6 only (checked in build)
    const size_t n = nn * size_t(np);
    tc::split_tf32_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(M, n, d_mhi, d_mlo);
    KIFMM_LAUNCH_CHECK();
    if (pair && rowb == 64) run_kernel<160, true, 64>(s);
    else if (pair) run_kernel<160, true, 128>(s);
    else if (rowb == 64) run_kernel<160, false, 64>(s);
    else run_kernel<160, false, 128>(s);
    tc::m2l_tc_reduce_kernel<160><<<dim3(n_tiles, rows / 16), 16 * (160 / 4), 0, s>>>(d_partial, d_tile_out, d_tile_slot, rows, check);
    KIFMM_LAUNCH_CHECK();
  }
};


// The dense (gathered) fp32 GEMMs of the upward / downward passes -- factored check->equivalent solves,
// M2M and L2L -- on the same tcgen05 kernel as M2L: 128-row tiles, one item per tile
// carrying all of the tile's segments, direct epilogue into the output rows.  B = n_mats matrices
// B[m][j][k] (output column j, reduction index k) in fp64, split into fp16 hi / lo after a power-of-two
// scale per output column common to all matrices (so 1/sigma factors of the pseudo-inverse stay in
// range); the epilogue multiplies the column unscale back.
struct TcGemm {
  int n_tiles = 0, sched_g = 0, np = 0;
  int *d_out = nullptr, *d_seg_mat = nullptr, *d_seg_in = nullptr, *d_sched = nullptr;
  tc::Item* d_items = nullptr;
  __half *d_bhi = nullptr, *d_blo = nullptr;
  float* d_cu = nullptr;
  CUtensorMap tm_hi{}, tm_lo{};
  TcGemm() = default;
  TcGemm(const TcGemm&) = delete;
  TcGemm& operator=(const TcGemm&) = delete;
  ~TcGemm() {
    for (void* p : {(void*)d_out, (void*)d_seg_mat, (void*)d_seg_in, (void*)d_items, (void*)d_bhi, (void*)d_blo,
                    (void*)d_cu, (void*)d_sched})
      if (p) cudaFree(p);
  }

  // tiles: out (128 rows, -1 pad) + segs (matrix, 128 input rows or -1)
  template <class Tile>
  void build(const std::vector<Tile>& tiles, const std::vector<double>& B, int n_mats, int width, size_t* total,
             int max_ctas = 0) {
    if (!tc_np_supported(width)) throw InvalidArgument("TcGemm: unsupported row width");
    np = width;
    const int NP = np;
    if (B.size() != size_t(n_mats) * NP * NP) throw InvalidArgument("TcGemm: B size");
    std::vector<int> out, seg_mat, seg_in;
    std::vector<tc::Item> items;
    for (const auto& t : tiles) {
      if (t.out.size() != size_t(tc::BM)) throw InvalidArgument("TcGemm: tiles must have 128 rows");
      const int sb = int(seg_mat.size());
      out.insert(out.end(), t.out.begin(), t.out.end());
      for (const auto& sg : t.segs) {
        seg_mat.push_back(sg.first);
        seg_in.insert(seg_in.end(), sg.second.begin(), sg.second.end());
      }
      items.push_back({int(items.size()), sb, int(seg_mat.size()), int(items.size())});
    }
    n_tiles = int(items.size());
    M2LTcPlan::up(&d_out, out, total);
    M2LTcPlan::up(&d_seg_mat, seg_mat, total);
    M2LTcPlan::up(&d_seg_in, seg_in, total);
    M2LTcPlan::up(&d_items, items, total);
    sched_g = std::max(1, std::min(n_tiles, max_ctas > 0 ? max_ctas : sm_count()));
    M2LTcPlan::up(&d_sched, lpt_schedule(items, sched_g), total);
    std::vector<float> cu(NP, 1.f);
    std::vector<__half> hi(B.size()), lo(B.size());
    for (int j = 0; j < NP; ++j) {
      double mx = 0;
      for (int m = 0; m < n_mats; ++m)
        for (int k = 0; k < NP; ++k) mx = std::max(mx, std::fabs(B[(size_t(m) * NP + j) * NP + k]));
      int e = 0;
      if (mx > 0) {
        int ex;
        std::frexp(mx, &ex);
        e = 10 - ex;
      }
      cu[j] = float(std::ldexp(1.0, -e));
      for (int m = 0; m < n_mats; ++m)
        for (int k = 0; k < NP; ++k) {
          const size_t i = (size_t(m) * NP + j) * NP + k;
          const double x = std::ldexp(B[i], e);
          const __half h = __float2half_rn(float(x));
          hi[i] = h;
          lo[i] = __float2half_rn(float(x - double(__half2float(h))));
        }
    }
    M2LTcPlan::up(&d_bhi, hi, total);
    M2LTcPlan::up(&d_blo, lo, total);
    M2LTcPlan::up(&d_cu, cu, total);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    KIFMM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn) throw DeviceError(KIFMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    auto enc = reinterpret_cast<M2LTcPlan::EncodeFn>(fn);
    M2LTcPlan::encode(enc, &tm_hi, d_bhi, NP, uint64_t(n_mats) * NP, NP, 64, 2);
    M2LTcPlan::encode(enc, &tm_lo, d_blo, NP, uint64_t(n_mats) * NP, NP, 64, 2);
    tc_dispatch_np(np, [&](auto w) {
      KIFMM_CUDA(cudaFuncSetAttribute(tc::m2l_tc_kernel<decltype(w)::value, false, 64, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      tc::Cfg<decltype(w)::value, false, 64, 2>::SMEM_BYTES));
    });
  }

  // dst[out rows] (=, or += when accumulate) A(split rows) . B^T; with out_split, the fp16 split of the
  // output rows is written too (dst may then be null)
  // fewest persistent CTAs with the same makespan (whole tiles per CTA): frees SMs for a concurrent chain
  static int min_ctas(int tiles) {
    const int per = (tiles + sm_count() - 1) / sm_count();
    return (tiles + per - 1) / per;
  }
  void run(const TcSplit& a, float* dst, bool accumulate, cudaStream_t s, const TcSplit* out_split = nullptr) const {
    if (!n_tiles) return;
    if (a.np != np || (out_split && out_split->np != np)) throw InvalidArgument("TcGemm: row width mismatch");
    tc_dispatch_np(np, [&](auto w) {
      launch_pdl(tc::m2l_tc_kernel<decltype(w)::value, false, 64, 2>, dim3(sched_g), dim3(tc::THREADS),
                 tc::Cfg<decltype(w)::value, false, 64, 2>::SMEM_BYTES, s, tm_hi, tm_lo, (const void*)a.hi, (const void*)a.lo,
                 (const tc::Item*)d_items, (const int*)d_sched, (const int*)d_seg_mat, (const int*)d_seg_in, a.rows,
                 (const float*)a.un, 1.f,
                 tc::Epi{nullptr, d_out, d_cu, dst, accumulate ? 1 : 0, 0, out_split ? out_split->hi : nullptr,
                         out_split ? out_split->lo : nullptr, out_split ? out_split->un : nullptr});
    });
    KIFMM_LAUNCH_CHECK();
  }
};

}  // namespace gpu
}  // namespace kifmm
