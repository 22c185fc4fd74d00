// Gathered, segmented, tiled SIMT GEMM -- the one engine behind every dense
// KIFMM operator application on the FP32/FP64 pipes:
//
//   Y[out(r)][n] (+)= sum_seg sum_k X[in(seg, r)][k] * W[mat(seg)][k][n]
//
//   P2M / P2L solves : factored pinv, two passes (U diag(1/s), then V^T)
//   M2M  per level   : 8 segments (octants), in = child rows
//   M2L  all levels  : one segment per transfer vector of the tile, in = V-list source rows
//   L2L  per level   : 1 segment, tiles grouped by child octant
//
// A tile is BM output rows that share a segment list; rows without a source in
// a segment gather zeros (cp.async zero-fill).  Each CTA computes BM x N with an
// (BM/TM) x (N/TN) thread grid, TM x TN register accumulators, and a
// STAGES-deep cp.async pipeline over (segment, K-chunk) pairs.
#pragma once

#include "common.cuh"

namespace kifmm {
namespace gpu {

template <class T>
struct GemmArgs {
  const int* tile_out;  // n_tiles * BM  (-1 = padding row)
  const int* tile_seg;  // n_tiles + 1
  const int* seg_mat;   // n_segs
  const int* seg_in;    // n_segs * BM   (-1 = zero row)
  const T* X;
  int ldx;
  const T* W;           // [mats][K][ldw]; a CTA of column block blockIdx.y computes columns [y N, y N + N)
  int ldw;              // row stride of W (= N for the widths instantiated directly; 2 N or 4 N for p = 8, 9, 10)
  int K;                // multiple of KC
  T* Y;
  int ldy;
  int accumulate;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <class T, int N>
struct GemmCfg;
// FP32: 128-row tiles, 8x8 per thread, 32-wide K chunks.
template <int N>
struct GemmCfg<float, N> {
  static constexpr int BM = 128, TM = 8, TN = 8, KC = 32, STAGES = 3;
};
// FP64: 64-row tiles, 4x8 per thread, 16-wide K chunks.
template <int N>
struct GemmCfg<double, N> {
  static constexpr int BM = 64, TM = 4, TN = 8, KC = 16, STAGES = 3;
};

template <class T, int N, int BM, int TM, int TN, int KC, int STAGES>
struct GemmShape {
  static constexpr int VEC = 16 / sizeof(T);      // elements per 16-byte chunk
  static constexpr int APAD = VEC;                // row pad of the A tile (bank spread)
  static constexpr int TR = BM / TM;              // thread rows
  static constexpr int TC = N / TN;               // thread cols
  static constexpr int NT = TR * TC;              // threads
  static constexpr int G = TN / VEC;              // column groups per thread
  static constexpr int GSTRIDE = N / G;           // column distance between groups
  static constexpr int A_ELEMS = BM * (KC + APAD);
  static constexpr int W_ELEMS = KC * N;
  static constexpr int STAGE_ELEMS = A_ELEMS + W_ELEMS;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(T);
  static_assert(N % TN == 0 && BM % TM == 0 && TN % VEC == 0 && KC % VEC == 0, "tile shape");
  static_assert(GSTRIDE == TC * VEC, "column interleave");
};

template <class T, int N, int BM, int TM, int TN, int KC, int STAGES>
__global__ void __launch_bounds__(GemmShape<T, N, BM, TM, TN, KC, STAGES>::NT, 1)
    gather_gemm_kernel(GemmArgs<T> a) {
  using S = GemmShape<T, N, BM, TM, TN, KC, STAGES>;
  using vec_t = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);

  const int tile = blockIdx.x;
  const int tid = threadIdx.x;
  const int tr = tid / S::TC, tc = tid % S::TC;
  const int seg0 = a.tile_seg[tile], seg1 = a.tile_seg[tile + 1];
  const int kchunks = a.K / KC;
  const int iters = (seg1 - seg0) * kchunks;

  auto load_stage = [&](int it, int stage) {
    const int seg = seg0 + it / kchunks;
    const int kc = (it % kchunks) * KC;
    T* As = smem + stage * S::STAGE_ELEMS;
    T* Ws = As + S::A_ELEMS;
    constexpr int ACH = BM * (KC / S::VEC);
    for (int c = tid; c < ACH; c += S::NT) {
      const int row = c / (KC / S::VEC), col = c % (KC / S::VEC);
      const int src = a.seg_in[size_t(seg) * BM + row];
      const T* g = a.X + size_t(src < 0 ? 0 : src) * a.ldx + kc + col * S::VEC;
      cp_async16(As + row * (KC + S::APAD) + col * S::VEC, g, src >= 0);
    }
    const T* wm = a.W + (size_t(a.seg_mat[seg]) * a.K + size_t(kc)) * a.ldw + size_t(blockIdx.y) * N;
    constexpr int WCH = KC * N / S::VEC, WROW = N / S::VEC;
    for (int c = tid; c < WCH; c += S::NT) {
      const int k = c / WROW, col = c % WROW;
      cp_async16(Ws + c * S::VEC, wm + size_t(k) * a.ldw + col * S::VEC, true);
    }
  };

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < iters) load_stage(s, s);
    cp_async_commit();
  }

  for (int it = 0; it < iters; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = it + STAGES - 1;
      if (nxt < iters) load_stage(nxt, nxt % STAGES);
      cp_async_commit();
    }
    const T* As = smem + (it % STAGES) * S::STAGE_ELEMS;
    const T* Ws = As + S::A_ELEMS;
#pragma unroll
    for (int k = 0; k < KC; k += S::VEC) {
      T av[TM][S::VEC];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const vec_t v = *reinterpret_cast<const vec_t*>(As + (tr + i * S::TR) * (KC + S::APAD) + k);
        const T* pv = reinterpret_cast<const T*>(&v);
#pragma unroll
        for (int e = 0; e < S::VEC; ++e) av[i][e] = pv[e];
      }
#pragma unroll
      for (int kk = 0; kk < S::VEC; ++kk) {
        T bv[TN];
#pragma unroll
        for (int g = 0; g < S::G; ++g) {
          const vec_t v = *reinterpret_cast<const vec_t*>(Ws + (k + kk) * N + g * S::GSTRIDE + tc * S::VEC);
          const T* pv = reinterpret_cast<const T*>(&v);
#pragma unroll
          for (int e = 0; e < S::VEC; ++e) bv[g * S::VEC + e] = pv[e];
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i][kk], bv[j], acc[i][j]);
      }
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int row = tr + i * S::TR;
    const int out = a.tile_out[size_t(tile) * BM + row];
    if (out < 0) continue;
    T* y = a.Y + size_t(out) * a.ldy + size_t(blockIdx.y) * N;
#pragma unroll
    for (int g = 0; g < S::G; ++g) {
      const int col = g * S::GSTRIDE + tc * S::VEC;
      vec_t v;
      T* pv = reinterpret_cast<T*>(&v);
      if (a.accumulate) v = *reinterpret_cast<const vec_t*>(y + col);
#pragma unroll
      for (int e = 0; e < S::VEC; ++e) pv[e] = (a.accumulate ? pv[e] : T(0)) + acc[i][g * S::VEC + e];
      *reinterpret_cast<vec_t*>(y + col) = v;
    }
  }
}

// FP64 variant on the warp-level FP64 tensor op (DMMA, mma.sync m8n8k4 f64): the same gathered,
// segmented tile (64 rows x N, cp.async pipeline over (segment, 16-wide K chunk)), but each warp owns a
// 32 x N/4 block of 4 x N/32 DMMA accumulators fed by register fragments -- per 4-wide k step a lane
// loads 4 + N/32 doubles from shared memory for 4 N/32 DMMAs (256 FMAs each), where the SIMT kernel's
// shared-memory operand traffic held DFMA at ~50 % of the FP64 peak (config 4, p = 7).
// Fragments (PTX m8n8k4 .f64): A[8x4] lane l -> (row l/4, k l%4); B[4x8] -> (k l%4, col l/4);
// C/D[8x8] -> (row l/4, cols 2 (l%4) + {0, 1}).
// Shared layout (a 64-bit fragment load is served per half-warp, 16 lanes x 8 B = one 128-B wavefront):
// A rows padded to 20 doubles (160 B: the 4 rows of a half-warp start 32 B apart), B rows to N + 4
// doubles (the 4 k rows of a half-warp start 32 B apart).  B rows at N + 8 put k and k + 2 on the
// same banks: 5.6e9 bank conflicts in one config-4 M2L launch (ncu).
template <int N>
struct DmmaShape {
  static constexpr int BM = 64, KC = 16, STAGES = 3, NT = 256;
  static constexpr int AST = KC + 4, BST = N + 4;
  static constexpr int NB = N / 32;  // 8-wide column blocks per warp (warps: 2 along M x 4 along N)
  static constexpr int A_ELEMS = BM * AST, W_ELEMS = KC * BST, STAGE_ELEMS = A_ELEMS + W_ELEMS;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
  static_assert(N % 32 == 0, "DMMA gemm: N multiple of 32");
};

template <int N>
__global__ void __launch_bounds__(256, 1) gather_dmma_kernel(GemmArgs<double> a) {
  using S = DmmaShape<N>;
  constexpr int BM = S::BM, KC = S::KC, STAGES = S::STAGES;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  const int tile = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp & 1, wn = warp >> 1;
  const int seg0 = a.tile_seg[tile], seg1 = a.tile_seg[tile + 1];
  const int kchunks = a.K / KC;
  const int iters = (seg1 - seg0) * kchunks;

  auto load_stage = [&](int it, int stage) {
    const int seg = seg0 + it / kchunks;
    const int kc = (it % kchunks) * KC;
    double* As = smem + stage * S::STAGE_ELEMS;
    double* Ws = As + S::A_ELEMS;
    constexpr int ACH = BM * (KC / 2);  // 16-byte chunks
    for (int c = tid; c < ACH; c += S::NT) {
      const int row = c / (KC / 2), col = c % (KC / 2);
      const int src = a.seg_in[size_t(seg) * BM + row];
      const double* g = a.X + size_t(src < 0 ? 0 : src) * a.ldx + kc + col * 2;
      cp_async16(As + row * S::AST + col * 2, g, src >= 0);
    }
    const double* wm_ = a.W + (size_t(a.seg_mat[seg]) * a.K + size_t(kc)) * a.ldw + size_t(blockIdx.y) * N;
    constexpr int WCH = KC * N / 2;
    for (int c = tid; c < WCH; c += S::NT) {
      const int k = c / (N / 2), col = c % (N / 2);
      cp_async16(Ws + k * S::BST + col * 2, wm_ + size_t(k) * a.ldw + col * 2, true);
    }
  };

  double acc[4][S::NB][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < S::NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < iters) load_stage(s, s);
    cp_async_commit();
  }
  const int ar = wm * 32 + (lane >> 2), ak = lane & 3;         // A fragment coordinates
  const int bk = lane & 3, bn = wn * (N / 4) + (lane >> 2);    // B fragment coordinates
  for (int it = 0; it < iters; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = it + STAGES - 1;
      if (nxt < iters) load_stage(nxt, nxt % STAGES);
      cp_async_commit();
    }
    const double* As = smem + (it % STAGES) * S::STAGE_ELEMS;
    const double* Ws = As + S::A_ELEMS;
#pragma unroll
    for (int ks = 0; ks < KC; ks += 4) {
      double af[4], bf[S::NB];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[(ar + 8 * i) * S::AST + ks + ak];
#pragma unroll
      for (int j = 0; j < S::NB; ++j) bf[j] = Ws[(ks + bk) * S::BST + bn + 8 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < S::NB; ++j)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                       : "d"(af[i]), "d"(bf[j]));
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = wm * 32 + 8 * i + (lane >> 2);
    const int out = a.tile_out[size_t(tile) * BM + row];
    if (out < 0) continue;
    double* y = a.Y + size_t(out) * a.ldy + size_t(blockIdx.y) * N;
#pragma unroll
    for (int j = 0; j < S::NB; ++j) {
      const int col = wn * (N / 4) + 8 * j + 2 * (lane & 3);
      double2 v = make_double2(0.0, 0.0);
      if (a.accumulate) v = *reinterpret_cast<const double2*>(y + col);
      v.x += acc[i][j][0];
      v.y += acc[i][j][1];
      *reinterpret_cast<double2*>(y + col) = v;
    }
  }
}

}  // namespace gpu
}  // namespace kifmm
