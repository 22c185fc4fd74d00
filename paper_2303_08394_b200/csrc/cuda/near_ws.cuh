// Near field (self + U list), fp32, warp-specialised and persistent.
//
// leaf_eval_f2_kernel launches one 128-thread block per leaf work: every block
// starts with a chain of dependent global loads (work -> round -> items ->
// sources) before its first FP32x2 instruction, and at 8 blocks per SM those
// start-up stalls left the FMA pipe idle ~28 % of the time (ncu, config 2).
// Here one producer warp per block walks the same work / round / item lists
// and stages each round's sources into a ring
// of shared-memory stages with one cp.async.bulk per contiguous source range
// (completing on the stage's full mbarrier); four consumer warps compute exactly what
// leaf_eval_f2_kernel computes -- same slice geometry, same p2p_round_fn,
// same fixed-order slice reduction -- so the result is bit-identical to it and
// independent of which block took which work.  Works come from an atomic
// counter (queue[0]), as in queue mode:
//   MODE 0  standalone: the launch takes every work
//   MODE 1  side: stops taking works once queue[1] is raised (by MODE 2)
//   MODE 2  drain: raises queue[1] and takes what is left
#pragma once

#include "m2l_tc.cuh"
#include "p2p.cuh"

namespace kifmm {
namespace gpu {

constexpr int kNearStages = 2;
constexpr int kNearWsThreads = 160;  // warps 0-3 consumers, warp 4 producer

struct NearStage {
  float4 src[kP2PCap];  // [self section, padded to S][other sources, padded to O]; reused for the reduction
  int wi, S, O, flags;      // flags: bit 0 first round of the work, bit 1 last round; wi < 0: stop
  int t_begin, t_count, geom, mul_tt;
  int mul_r, pad0, pad1, pad2;
};

struct NearSmem {
  NearStage st[kNearStages];
  unsigned long long full[kNearStages], empty[kNearStages];
};

__device__ __forceinline__ void near_consumer_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

#ifndef KIFMM_NEAR_WS_MINB
#define KIFMM_NEAR_WS_MINB 6  // blocks per SM the register allocation is sized for (6: 64 registers)
#endif
template <bool GRAD, int MODE>
__global__ void __launch_bounds__(kNearWsThreads, KIFMM_NEAR_WS_MINB) near_ws_kernel(P2PParams<float> p,
                                                                   const LeafWork* __restrict__ works,
                                                                   const int4* __restrict__ rounds,
                                                                   const int4* __restrict__ items,
                                                                   float* __restrict__ pot, float* __restrict__ grad,
                                                                   int n_works, int* __restrict__ queue) {
  __shared__ __align__(16) NearSmem sm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kNearStages; ++s) {
      tc::mbar_init(tc::smem_u32(&sm.full[s]), 32);  // one arrival per producer lane (+ the bulk-copy bytes)
      tc::mbar_init(tc::smem_u32(&sm.empty[s]), 4);  // one per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (MODE == 2 && blockIdx.x == 0) atomicExch(queue + 1, 1);
  }
  __syncthreads();
  timeline_begin(MODE == 2 ? 4 : 3);

  if (warp == 4) {  // ---------------- producer
    int stage = 0;
    uint32_t phase = 0;
    const float fa = float(kFarAway);
    const float4 far4 = make_float4(fa, fa, fa, 0.f);
    for (;;) {
      int wi = 0;
      if (lane == 0) {
        if (MODE == 1) {  // side blocks: stop once draining
#ifdef KIFMM_EXPERIMENTS  // optional pause while M2L runs (queue[3], KIFMM_NEAR_PAUSE)
          for (int pz; (pz = atomicAdd(queue + 3, 0)) != 0 && (pz == 1 || (blockIdx.x & 1)) &&
                       atomicAdd(queue + 1, 0) == 0;)
            __nanosleep(2000);
#endif
          wi = atomicAdd(queue + 1, 0) != 0 ? n_works : atomicAdd(queue, 1);
        } else {
          wi = atomicAdd(queue, 1);
        }
      }
      wi = __shfl_sync(0xffffffffu, wi, 0);
      if (wi >= n_works) {  // tell the consumers to stop
        tc::mbar_wait(tc::smem_u32(&sm.empty[stage]), phase ^ 1);
        if (lane == 0) sm.st[stage].wi = -1;
        tc::mbar_arrive_local(tc::smem_u32(&sm.full[stage]));
        break;
      }
      const LeafWork w = works[wi];
      for (int r = w.round_begin; r < w.round_end; ++r) {
        const int4 rd = rounds[r];
        // item descriptors of this round, one per lane (loaded before the stage wait: latency overlap)
        int4 my_item = make_int4(0, 0, 0, 0);
        if (rd.x + lane < rd.y) my_item = items[rd.x + lane];
        tc::mbar_wait(tc::smem_u32(&sm.empty[stage]), phase ^ 1);
        NearStage& S = sm.st[stage];
        const uint32_t sbase = tc::smem_u32(S.src);
        const int Ssz = rd.z & 0xFFFF, ns = rd.z >> 16, Osz = rd.w & 0xFFFF, no = rd.w >> 16;
        // one cp.async.bulk per contiguous source range (lane k: item k), completing on the full barrier
        // (lane 0 adds the round's byte count to its arrival below)
        for (int kb = rd.x; kb < rd.y; kb += 32) {
          if (kb != rd.x && kb + lane < rd.y) my_item = items[kb + lane];
          if (kb + lane < rd.y) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile(
                "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    sbase + 16u * uint32_t(my_item.w)),
                "l"(p.src + my_item.y), "r"(16u * uint32_t(my_item.z)), "r"(tc::smem_u32(&sm.full[stage]))
                : "memory");
          }
        }
        for (int i = ns + lane; i < Ssz; i += 32) S.src[i] = far4;
        for (int i = Ssz + no + lane; i < Ssz + Osz; i += 32) S.src[i] = far4;
        if (lane == 0) {
          S.wi = wi;
          S.S = Ssz;
          S.O = Osz;
          S.flags = (r == w.round_begin ? 1 : 0) | (r == w.round_end - 1 ? 2 : 0);
          S.t_begin = w.t_begin;
          S.t_count = w.t_count;
          S.geom = w.geom;
          S.mul_tt = w.mul_tt;
          S.mul_r = w.mul_r;
        }
        if (lane == 0)  // release: padding + header stores; the bulk copies' bytes
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(&sm.full[stage])),
                       "r"(16u * uint32_t(ns + no))
                       : "memory");
        else
          tc::mbar_arrive_local(tc::smem_u32(&sm.full[stage]));
        if (++stage == kNearStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    timeline_end(MODE == 2 ? 4 : 3);
    return;
  }

  // ---------------- consumers (warps 0-3): geometry and arithmetic of leaf_eval_f2_kernel
  constexpr int NPR = kNearNPair;  // target pairs per thread: targets t0 + m TT, m < 2 NPR
  int stage = 0;
  uint32_t phase = 0;
  int nt = 0, TT = 1, R = 1, slice = 0, t0 = 0, mul_r = 0;
  bool active = false;
  f2_t x[NPR], y[NPR], z[NPR], ph[NPR], gx[NPR], gy[NPR], gz[NPR];
  for (;;) {
    tc::mbar_wait(tc::smem_u32(&sm.full[stage]), phase);
    NearStage& S = sm.st[stage];
    if (S.wi < 0) break;
    const int flags = S.flags;
    if (flags & 1) {  // first round of a work
      nt = S.t_count;
      TT = S.geom >> 8;
      R = S.geom & 0xFF;
      mul_r = S.mul_r;
      slice = div_mul(tid, S.mul_tt);
      t0 = tid - slice * TT;
      active = slice < R;
      // targets straight from global (L2-resident; staging them too would cost the sixth block per SM)
#pragma unroll
      for (int k = 0; k < NPR; ++k) {
        const int ta = t0 + (2 * k) * TT, tb = t0 + (2 * k + 1) * TT;
        const float4 xa = p.src[S.t_begin + (active && ta < nt ? ta : 0)];
        const float4 xb = p.src[S.t_begin + (active && tb < nt ? tb : 0)];
        x[k] = f2_pair(xa.x, xb.x);
        y[k] = f2_pair(xa.y, xb.y);
        z[k] = f2_pair(xa.z, xb.z);
        ph[k] = gx[k] = gy[k] = gz[k] = 0;
      }
    }
    const int Ssz = S.S, Osz = S.O;
    if (active) {
      if (Ssz) {
        const int per = div_mul(Ssz, mul_r);
        p2p_round_fn<GRAD, true, NPR>(S.src, slice * per, slice * per + per, x, y, z, ph, gx, gy, gz);
      }
      if (Osz) {
        const int per = div_mul(Osz, mul_r);
        p2p_round_fn<GRAD, false, NPR>(S.src, Ssz + slice * per, Ssz + slice * per + per, x, y, z, ph, gx, gy, gz);
      }
    }
    if (flags & 2) {  // last round: fixed-order slice reduction through this stage's source buffer
      const int t_begin = S.t_begin;
      near_consumer_sync();  // every consumer is done reading the sources
      float* red = reinterpret_cast<float*>(S.src);  // [slice][component][n_t]
      constexpr int NC = GRAD ? 4 : 1;
      if (active) {
#pragma unroll
        for (int k = 0; k < NPR; ++k) {
          float a[4], b[4];
          f2_unpack(ph[k], a[0], b[0]);
          f2_unpack(gx[k], a[1], b[1]);
          f2_unpack(gy[k], a[2], b[2]);
          f2_unpack(gz[k], a[3], b[3]);
          const int ta = t0 + (2 * k) * TT, tb = t0 + (2 * k + 1) * TT;
#pragma unroll
          for (int d = 0; d < NC; ++d) {
            if (ta < nt) red[(slice * NC + d) * nt + ta] = a[d];
            if (tb < nt) red[(slice * NC + d) * nt + tb] = b[d];
          }
        }
      }
      near_consumer_sync();
      if (tid < nt) {
        const float c = float(kInv4PiD);
        float a[NC];
#pragma unroll
        for (int d = 0; d < NC; ++d) a[d] = 0;
        for (int sl = 0; sl < R; ++sl)
#pragma unroll
          for (int d = 0; d < NC; ++d) a[d] += red[(sl * NC + d) * nt + tid];
        const int t = t_begin + tid;
        pot[t] = 0.f + c * a[0];  // the expressions of leaf_eval_f2_kernel<.., ACC = false> (signed zeros)
        if (GRAD) {
          float* gp = grad + 3 * size_t(t);
          gp[0] = 0.f - c * a[NC > 1 ? 1 : 0];
          gp[1] = 0.f - c * a[NC > 2 ? 2 : 0];
          gp[2] = 0.f - c * a[NC > 3 ? 3 : 0];
        }
      }
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive_local(tc::smem_u32(&sm.empty[stage]));
    if (++stage == kNearStages) {
      stage = 0;
      phase ^= 1;
    }
  }
  timeline_end(MODE == 2 ? 4 : 3);
}

}  // namespace gpu
}  // namespace kifmm
