// Near field (self + U list), fp32, one WARP per leaf work, persistent.
//
// Why: the block-per-leaf kernels (leaf_eval_f2_kernel, near_ws_kernel) spend a quarter of their warp
// samples outside the pair loop (ncu, config 2): block prologue (work -> round -> items -> sources),
// waits on the staging barrier, two __syncthreads per round and an 8-slice reduction through shared
// memory.  Here every warp is independent:
//   * a work is <= 64 targets of one leaf: TT = ceil(n / 2) target pairs (FP32x2 lanes) x R = min(8, 32 / TT)
//     source slices fill the warp (config 2: 15-16 pairs x 2 slices);
//   * its sources stream through two per-warp shared-memory buffers of kNwCap float4: while the warp
//     computes round r, the cp.async.bulk copies of round r + 1 -- or of the first round of its NEXT work,
//     taken from the queue one work ahead -- land in the other buffer (one mbarrier per buffer, the round's
//     byte count posted by lane 0);
//   * slice partials are combined with shuffles in fixed order; no block barrier anywhere.
// Rounds are [self section, padded to S][other sources, padded to O] as in the block kernels (S and O
// multiples of 4 R; padding = far-away zero charges written by the lanes), so the r = 0 mask runs only
// on the self section.  Every work is computed by exactly one warp with the same arithmetic, so results do
// not depend on which warp (or which launch) takes it.  Works come from an atomic counter (queue[0]):
//   MODE 0  standalone: the launch takes every work
//   MODE 1  side: stops taking works once queue[1] is raised (by MODE 2)
//   MODE 2  drain: raises queue[1] and takes what is left
#pragma once

#include "m2l_tc.cuh"
#include "p2p.cuh"

namespace kifmm {
namespace gpu {

constexpr int kNwWarps = 8;        // warps per block
constexpr int kNwCap = 128;        // sources per round (per buffer)
constexpr int kNwTargets = 64;     // targets per work: 32 lanes x one FP32x2 pair
__host__ __device__ inline int nw_slices(int nt) {
  const int tt = (nt + 1) >> 1;
  const int r = 32 / (tt > 0 ? tt : 1);
  return r < 1 ? 1 : (r > 8 ? 8 : r);
}

struct NwSmem {
  float4 buf[kNwWarps][2][kNwCap];
  unsigned long long bar[kNwWarps][2];
};

#ifndef KIFMM_NW_MINB
#define KIFMM_NW_MINB 4  // 4 x 8 warps per SM at 64 registers
#endif
template <bool GRAD, int MODE>
__global__ void __launch_bounds__(kNwWarps * 32, KIFMM_NW_MINB) near_warp_kernel(P2PParams<float> p,
                                                                  const LeafWork* __restrict__ works,
                                                                  const int4* __restrict__ rounds,
                                                                  const int4* __restrict__ items,
                                                                  float* __restrict__ pot, float* __restrict__ grad,
                                                                  int n_works, int* __restrict__ queue) {
  __shared__ __align__(16) NwSmem sm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = tc::smem_u32(&sm.bar[warp][0]), bar1 = tc::smem_u32(&sm.bar[warp][1]);
  if (lane == 0) {
    tc::mbar_init(bar0, 1);
    tc::mbar_init(bar1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (MODE == 2 && blockIdx.x == 0 && warp == 0) atomicExch(queue + 1, 1);
  }
  __syncwarp();
  timeline_begin(MODE == 2 ? 4 : 3);
  const float fa = float(kFarAway);
  const float4 far4 = make_float4(fa, fa, fa, 0.f);

  auto take = [&]() {
    int wi = 0;
    if (lane == 0) wi = (MODE == 1 && atomicAdd(queue + 1, 0) != 0) ? n_works : atomicAdd(queue, 1);
    return __shfl_sync(0xffffffffu, wi, 0);
  };
  // stage round rd into buffer b: one cp.async.bulk per contiguous source range (lane k: item k), the
  // padding written by the lanes, lane 0 posting the byte count on the buffer's barrier
  auto issue = [&](int b, const int4 rd) {
    float4* dst = sm.buf[warp][b];
    const uint32_t bar = b ? bar1 : bar0;
    const int S = rd.z & 0xFFFF, ns = rd.z >> 16, O = rd.w & 0xFFFF, no = rd.w >> 16;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior reads of the buffer (generic proxy)
    for (int k = rd.x + lane; k < rd.y; k += 32) {
      const int4 it = items[k];
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              tc::smem_u32(dst + it.w)),
          "l"(p.src + it.y), "r"(16u * uint32_t(it.z)), "r"(bar)
          : "memory");
    }
    for (int i = ns + lane; i < S; i += 32) dst[i] = far4;
    for (int i = S + no + lane; i < S + O; i += 32) dst[i] = far4;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(16u * uint32_t(ns + no))
                   : "memory");
  };

  int wi = take();
  if (wi >= n_works) {
    timeline_end(MODE == 2 ? 4 : 3);
    return;
  }
  LeafWork w = works[wi];
  int r = w.round_begin;
  issue(0, rounds[r]);
  int b = 0;
  uint32_t ph0 = 0, ph1 = 0;
  int nt = 0, TT = 1, R = 1, slice = 0, pi = 0;
  bool act = false;
  f2_t x[1], y[1], z[1], ph[1], gx[1], gy[1], gz[1];
  for (;;) {
    // prefetch: the next round of this work, or the first round of the next work
    int r_next = r + 1, wi_next = wi;
    LeafWork wn = w;
    if (r_next == w.round_end) {
      wi_next = take();
      if (wi_next < n_works) {
        wn = works[wi_next];
        r_next = wn.round_begin;
      } else {
        r_next = -1;
      }
    }
    const int4 rd = rounds[r];
    if (r_next >= 0) issue(b ^ 1, rounds[r_next]);
    if (r == w.round_begin) {  // first round of a work: its geometry and targets
      nt = w.t_count;
      TT = (nt + 1) >> 1;
      R = nw_slices(nt);
      slice = lane / TT;
      pi = lane - slice * TT;
      act = slice < R;
      const int ta = pi, tb = pi + TT;
      const float4 xa = p.src[w.t_begin + (act && ta < nt ? ta : 0)];
      const float4 xb = p.src[w.t_begin + (act && tb < nt ? tb : 0)];
      x[0] = f2_pair(xa.x, xb.x);
      y[0] = f2_pair(xa.y, xb.y);
      z[0] = f2_pair(xa.z, xb.z);
      ph[0] = gx[0] = gy[0] = gz[0] = 0;
    }
    if (b) {
      tc::mbar_wait(bar1, ph1);
      ph1 ^= 1u;
    } else {
      tc::mbar_wait(bar0, ph0);
      ph0 ^= 1u;
    }
    const float4* src = sm.buf[warp][b];
    const int S = rd.z & 0xFFFF, O = rd.w & 0xFFFF;
    if (act) {
      if (S) {
        const int per = S / R;
        p2p_round_fn<GRAD, true, 1>(src, slice * per, slice * per + per, x, y, z, ph, gx, gy, gz);
      }
      if (O) {
        const int per = O / R;
        p2p_round_fn<GRAD, false, 1>(src, S + slice * per, S + slice * per + per, x, y, z, ph, gx, gy, gz);
      }
    }
    if (r == w.round_end - 1) {  // last round: fixed-order slice reduction into slice 0, output
      float v[8];
      f2_unpack(ph[0], v[0], v[4]);
      f2_unpack(gx[0], v[1], v[5]);
      f2_unpack(gy[0], v[2], v[6]);
      f2_unpack(gz[0], v[3], v[7]);
      for (int k = 1; k < R; ++k) {
        const int sl = lane + k * TT;
        const bool tk = slice == 0 && sl < 32;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          const float o = __shfl_sync(0xffffffffu, v[d], tk ? sl : lane);
          if (GRAD || (d & 3) == 0) v[d] += tk ? o : 0.f;
        }
      }
      if (slice == 0) {
        const float c = float(kInv4PiD);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int tl = h ? pi + TT : pi;
          if (tl >= nt) continue;
          const int t = w.t_begin + tl;
          pot[t] = 0.f + c * v[4 * h];
          if (GRAD) {
            float* gp = grad + 3 * size_t(t);
            gp[0] = 0.f - c * v[4 * h + 1];
            gp[1] = 0.f - c * v[4 * h + 2];
            gp[2] = 0.f - c * v[4 * h + 3];
          }
        }
      }
    }
    __syncwarp();  // every lane is done with buffer b before it is refilled
    if (r_next < 0) break;
    w = wn;
    wi = wi_next;
    r = r_next;
    b ^= 1;
  }
  timeline_end(MODE == 2 ? 4 : 3);
}

}  // namespace gpu
}  // namespace kifmm
