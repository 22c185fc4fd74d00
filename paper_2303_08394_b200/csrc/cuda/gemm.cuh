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
  const T* W;           // [mats][K][N]
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
    const T* wm = a.W + size_t(a.seg_mat[seg]) * a.K * N + size_t(kc) * N;
    constexpr int WCH = KC * N / S::VEC;
    for (int c = tid; c < WCH; c += S::NT) cp_async16(Ws + c * S::VEC, wm + c * S::VEC, true);
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
    T* y = a.Y + size_t(out) * a.ldy;
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

}  // namespace gpu
}  // namespace kifmm
