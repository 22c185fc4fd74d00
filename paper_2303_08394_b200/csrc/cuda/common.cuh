// Device-side helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "common.hpp"

namespace kifmm {
namespace gpu {

constexpr double kInv4PiD = 0.07957747154594767;  // 1 / (4 pi)

#define KIFMM_CUDA(call)                                                                          \
  do {                                                                                            \
    cudaError_t err_ = (call);                                                                    \
    if (err_ != cudaSuccess)                                                                      \
      throw ::kifmm::DeviceError(err_ == cudaErrorMemoryAllocation ? KIFMM_E_OUT_OF_MEMORY        \
                                                                   : KIFMM_E_CUDA,                \
                                 std::string(#call) + ": " + cudaGetErrorString(err_));          \
  } while (0)

#define KIFMM_LAUNCH_CHECK() KIFMM_CUDA(cudaGetLastError())

// (x, y, z, w) quadruple of the working precision: positions with charge or
// half side in w.  16 B (fp32) / 32 B (fp64) aligned for vector loads.
template <class T>
struct V4;
template <>
struct V4<float> {
  using type = float4;
};
template <>
struct V4<double> {
  using type = double4;
};
template <class T>
using v4_t = typename V4<T>::type;

template <class T>
__device__ __forceinline__ v4_t<T> make4(T x, T y, T z, T w);
template <>
__device__ __forceinline__ float4 make4<float>(float x, float y, float z, float w) {
  return make_float4(x, y, z, w);
}
template <>
__device__ __forceinline__ double4 make4<double>(double x, double y, double z, double w) {
  return make_double4(x, y, z, w);
}

// 1/sqrt(r2): one MUFU.RSQ in fp32 (rsqrt.approx.ftz, no denormal fix-up; r2 is
// either 0 or a squared distance far above FLT_MIN), correctly rounded-ish in fp64.
__device__ __forceinline__ float rinv(float r2) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(r2));
  return r;
}
__device__ __forceinline__ double rinv(double r2) { return rsqrt(r2); }
// ... with the SPEC self-interaction convention (0 at r = 0).
template <class T>
__device__ __forceinline__ T rinv_masked(T r2) {
  return r2 > T(0) ? rinv(r2) : T(0);
}
// Packed FP32 pairs (sm_100a FADD2 / FMUL2 / FFMA2: two fp32 lanes per
// instruction, each rounded exactly like its scalar counterpart).
using f2_t = unsigned long long;
__device__ __forceinline__ f2_t f2_pack(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
// A loop-invariant pair built once by a real FADD2 (a + -0 == a exactly, also for +-0): packed straight from
// two scalars (e.g. the .x of two float4 loads), ptxas keeps the halves apart and rebuilds the 64-bit pair
// with two MOVs at every use inside the loop.
__device__ __forceinline__ f2_t f2_pair(float a, float b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a, b)), "l"(f2_pack(-0.f, -0.f)));
  return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// fp16 operand split of an expansion row for the kind::f16 tensor-core GEMMs: x * 2^e with e chosen so
// max|row| lands in [2^9, 2^10), stored as hi = fp16(x 2^e), lo = fp16(x 2^e - hi), unscale 2^-e.
__device__ __forceinline__ int f16_row_exponent(float mx) {
  int e = 0;
  if (mx > 0.f) {
    int ex;
    frexpf(mx, &ex);  // mx in [2^(ex-1), 2^ex)
    e = 10 - ex;
  }
  return e;
}
// Warp-cooperative split of one W-wide row held as v[k] = row[lane + 32 k].
template <int W>
__device__ __forceinline__ void split_row_warp(const float (&v)[W / 32], int lane, size_t row, __half* hi, __half* lo,
                                               float* un) {
  float mx = 0.f;
#pragma unroll
  for (int k = 0; k < W / 32; ++k) mx = fmaxf(mx, fabsf(v[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int e = f16_row_exponent(mx);
  const float sc = ldexpf(1.f, e);
#pragma unroll
  for (int k = 0; k < W / 32; ++k) {
    const float x = v[k] * sc;
    const __half h = __float2half_rn(x);
    hi[row * W + lane + 32 * k] = h;
    lo[row * W + lane + 32 * k] = __float2half_rn(x - __half2float(h));
  }
  if (lane == 0) un[row] = ldexpf(1.f, -e);
}

// Timeline probes (experiments, KIFMM_TIMELINE): kernel `id` records the earliest block start and the
// latest block end (globaltimer ns) of its launch.
__device__ unsigned long long g_timeline[16][2];
__device__ int g_timeline_on;
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// compiled in only with -DKIFMM_TIMELINE_PROBES (they cost registers in the far kernel)
__device__ __forceinline__ void timeline_begin(int id) {
#ifdef KIFMM_TIMELINE_PROBES
  if (threadIdx.x == 0 && g_timeline_on) atomicMin(&g_timeline[id][0], globaltimer());
#endif
}
__device__ __forceinline__ void timeline_end(int id) {
#ifdef KIFMM_TIMELINE_PROBES
  if (threadIdx.x == 0 && g_timeline_on) atomicMax(&g_timeline[id][1], globaltimer());
#endif
}

// Programmatic dependent launch (kernels launched with cudaLaunchAttributeProgrammaticStreamSerialization):
// pdl_trigger lets the next kernel of the stream start launching (its CTAs take SMs this grid leaves
// free and run their set-up); pdl_wait blocks until every prerequisite grid has completed and its
// memory is visible.  Every kernel launched with the attribute calls pdl_wait before it touches data
// an earlier kernel writes (or reads: WAR); without the attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Far-away zero-charge source used to pad staged source rounds (contributes exactly 0).
constexpr double kFarAway = 1e15;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace gpu
}  // namespace kifmm
