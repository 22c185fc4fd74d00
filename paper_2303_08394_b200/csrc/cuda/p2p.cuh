// P2P-family kernels (SIMT, FP32 or FP64): every KIFMM operator that is a
// kernel sum over explicit points.
//
//  leaf_eval   near field + L2P (467-472) + M2P (474-479) fused:
//              all three are sums of q/(4 pi r) over "sources" that are either
//              particles of U-list leaves or surface points carrying equivalent
//              densities, accumulated into one per-target register set.
//  p2m_check   up-check potentials of a leaf's particles (check step)
//  p2l_check   down-check potentials of X-list particles (check step)
//  direct      verification direct sum at sampled targets
//
// Sources are staged in shared memory and read as warp-broadcast vector loads;
// r^-1 comes from MUFU.RSQ (rsqrtf) with the SPEC's r = 0 -> 0 convention.
// Every target is owned by one thread slot and partial sums of the 4 warps are
// combined in a fixed order, so results are deterministic.
#pragma once

#include "common.cuh"

namespace kifmm {
namespace gpu {

// Source item of leaf_eval: {kind, a, b, 0}
//   kind 0: particles [a, a + b) of the packed source array
//   kind 1: down-equivalent surface of node a (alpha_outer), densities L[a]   (L2P)
//   kind 2: up-equivalent surface of node a (alpha_inner), densities M[a]     (M2P)
//   kind 3: particles [a, a + b) of the target leaf itself (the only sources that can
//           coincide with a target, so the only ones evaluated with the r = 0 mask)
enum : int { kSrcParticles = 0, kSrcL2P = 1, kSrcM2P = 2, kSrcSelf = 3 };

struct LeafWork {
  int leaf;
  int t_begin;  // first target (reordered particle index)
  int t_count;  // <= 128
  int item_begin, item_end;
};

template <class T>
struct P2PParams {
  const v4_t<T>* src;       // N packed (x, y, z, q)
  const v4_t<T>* node_geom; // n_nodes (cx, cy, cz, half_side)
  const T* surface;         // n_e x 3 unit surface grid
  int n_e;
  int ld;                   // row stride of expansion buffers
  T alpha_inner, alpha_outer;
};

constexpr int kP2PThreads = 128;
constexpr int kP2PCap = 512;  // staged sources per round

template <class T>
__device__ __forceinline__ v4_t<T> surface_source(const P2PParams<T>& p, int node, T alpha, const T* dens, int j) {
  const v4_t<T> g = p.node_geom[node];
  const T s = alpha * g.w;
  return make4<T>(g.x + s * p.surface[3 * j], g.y + s * p.surface[3 * j + 1], g.z + s * p.surface[3 * j + 2],
                  dens[size_t(node) * p.ld + j]);
}

// One block per work item (leaf, <=128 targets).  Sources are staged in rounds of
// up to kP2PCap, padded to a multiple of 32 with far-away zero charges; warp w
// takes the contiguous quarter [w*n/4, (w+1)*n/4) of a round and lane l owns
// targets l, l+32, l+64, l+96 of the item.  A round holds either only self-leaf
// particles (masked r = 0 path) or only other sources (no mask).
template <class T, bool GRAD, bool MASK>
__device__ __forceinline__ void p2p_round(const v4_t<T>* sh, int begin, int end, T x, T y, T z, T& ph, T& gx, T& gy,
                                          T& gz) {
  T a_ph = 0, a_gx = 0, a_gy = 0, a_gz = 0;
  for (int j = begin; j < end; j += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const v4_t<T> s = sh[j + u];
      const T dx = x - s.x, dy = y - s.y, dz = z - s.z;
      const T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const T ri = MASK ? rinv_masked(r2) : rinv(r2);
      if (GRAD) {
        const T qr = s.w * ri;
        a_ph += qr;
        const T qr3 = qr * (ri * ri);
        a_gx = fma(qr3, dx, a_gx);
        a_gy = fma(qr3, dy, a_gy);
        a_gz = fma(qr3, dz, a_gz);
      } else {
        a_ph = fma(s.w, ri, a_ph);
      }
    }
  }
  ph += a_ph;
  gx += a_gx;
  gy += a_gy;
  gz += a_gz;
}

template <class T, bool GRAD>
__global__ void __launch_bounds__(kP2PThreads) leaf_eval_kernel(P2PParams<T> p, const LeafWork* __restrict__ works,
                                                                 const int4* __restrict__ items,
                                                                 const T* __restrict__ M, const T* __restrict__ L,
                                                                 T* __restrict__ pot, T* __restrict__ grad) {
  __shared__ v4_t<T> sh[kP2PCap];
  __shared__ T red[4][4][kP2PThreads];  // [warp][component][target]
  const LeafWork w = works[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ngroups = (w.t_count + 31) >> 5;

  T tx[4], ty[4], tz[4], ph[4], gx[4], gy[4], gz[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int t = g * 32 + lane;
    v4_t<T> x = p.src[w.t_begin + (t < w.t_count ? t : 0)];
    tx[g] = x.x;
    ty[g] = x.y;
    tz[g] = x.z;
    ph[g] = gx[g] = gy[g] = gz[g] = T(0);
  }

  int it = w.item_begin, off = 0;
  while (it < w.item_end) {
    int fill = 0;
    const bool masked = items[it].x == kSrcSelf;
    while (it < w.item_end && fill < kP2PCap) {
      const int4 item = items[it];
      if ((item.x == kSrcSelf) != masked) break;
      const bool particles = item.x == kSrcParticles || item.x == kSrcSelf;
      const int len = particles ? item.z : p.n_e;
      const int take = min(len - off, kP2PCap - fill);
      if (particles) {
        for (int i = tid; i < take; i += kP2PThreads) sh[fill + i] = p.src[item.y + off + i];
      } else {
        const bool l2p = item.x == kSrcL2P;
        const T alpha = l2p ? p.alpha_outer : p.alpha_inner;
        const T* dens = l2p ? L : M;
        for (int i = tid; i < take; i += kP2PThreads) sh[fill + i] = surface_source(p, item.y, alpha, dens, off + i);
      }
      fill += take;
      off += take;
      if (off == len) {
        ++it;
        off = 0;
      }
    }
    const int padded = (fill + 31) & ~31;
    for (int i = fill + tid; i < padded; i += kP2PThreads)
      sh[i] = make4<T>(T(kFarAway), T(kFarAway), T(kFarAway), T(0));
    __syncthreads();
    const int q4 = padded >> 2;
    const int jb = warp * q4, je = jb + q4;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (g >= ngroups) break;
      if (masked)
        p2p_round<T, GRAD, true>(sh, jb, je, tx[g], ty[g], tz[g], ph[g], gx[g], gy[g], gz[g]);
      else
        p2p_round<T, GRAD, false>(sh, jb, je, tx[g], ty[g], tz[g], ph[g], gx[g], gy[g], gz[g]);
    }
    __syncthreads();
  }

#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (g >= ngroups) break;
    red[warp][0][g * 32 + lane] = ph[g];
    if (GRAD) {
      red[warp][1][g * 32 + lane] = gx[g];
      red[warp][2][g * 32 + lane] = gy[g];
      red[warp][3][g * 32 + lane] = gz[g];
    }
  }
  __syncthreads();
  for (int t0 = tid; t0 < w.t_count; t0 += kP2PThreads) {
    const T c = T(kInv4PiD);
    const int t = w.t_begin + t0;
    pot[t] = c * (((red[0][0][t0] + red[1][0][t0]) + red[2][0][t0]) + red[3][0][t0]);
    if (GRAD) {
#pragma unroll
      for (int d = 0; d < 3; ++d)
        grad[3 * size_t(t) + d] = -c * (((red[0][d + 1][t0] + red[1][d + 1][t0]) + red[2][d + 1][t0]) + red[3][d + 1][t0]);
    }
  }
}

// Check potentials on a node's surface (alpha) from particle ranges.
// work: {node, out_row, range_begin, range_end} where ranges index `ranges`
// (int2 {first particle, count}).  out[out_row][j] = scale * sum q / (4 pi r),
// scale = 2^(ref_level - level); padding columns get 0.
struct CheckWork {
  int node, out_row, range_begin, range_end;
};

template <class T>
__global__ void __launch_bounds__(kP2PThreads) check_kernel(P2PParams<T> p, const CheckWork* __restrict__ works,
                                                             const int2* __restrict__ ranges,
                                                             const int* __restrict__ node_level, int ref_level,
                                                             T alpha, T* __restrict__ out, int ld_out) {
  __shared__ v4_t<T> sh[kP2PCap];
  const CheckWork w = works[blockIdx.x];
  const int tid = threadIdx.x;
  const v4_t<T> g = p.node_geom[w.node];
  const T s = alpha * g.w;
  T yx[2], yy[2], yz[2], acc[2];
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int j = tid + m * kP2PThreads;
    const int jj = j < p.n_e ? j : 0;
    yx[m] = g.x + s * p.surface[3 * jj];
    yy[m] = g.y + s * p.surface[3 * jj + 1];
    yz[m] = g.z + s * p.surface[3 * jj + 2];
    acc[m] = T(0);
  }
  int r = w.range_begin, off = 0;
  while (r < w.range_end) {
    int fill = 0;
    while (r < w.range_end && fill < kP2PCap) {
      const int2 rg = ranges[r];
      const int take = min(rg.y - off, kP2PCap - fill);
      for (int i = tid; i < take; i += kP2PThreads) sh[fill + i] = p.src[rg.x + off + i];
      fill += take;
      off += take;
      if (off == rg.y) {
        ++r;
        off = 0;
      }
    }
    const int padded = (fill + 7) & ~7;
    for (int i = fill + tid; i < padded; i += kP2PThreads)
      sh[i] = make4<T>(T(kFarAway), T(kFarAway), T(kFarAway), T(0));
    __syncthreads();
    // check surfaces never touch particles (alpha > 1 around the node / X-list separation): no r = 0 mask
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      if (m * kP2PThreads >= p.n_e) break;
      T a = 0;
      for (int i = 0; i < padded; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const v4_t<T> q = sh[i + u];
          const T dx = yx[m] - q.x, dy = yy[m] - q.y, dz = yz[m] - q.z;
          a = fma(q.w, rinv(fma(dz, dz, fma(dy, dy, dx * dx))), a);
        }
      }
      acc[m] += a;
    }
    __syncthreads();
  }
  const int lvl = node_level[w.node];
  const T scale = T(kInv4PiD) * T(ldexp(1.0, ref_level - lvl));
  T* o = out + size_t(w.out_row) * ld_out;
  for (int j = tid; j < ld_out; j += kP2PThreads) {
    const int m = j / kP2PThreads;
    T v = T(0);
    if (j < p.n_e) v = (m == 0 ? acc[0] : acc[1]) * scale;
    o[j] = v;
  }
}

// Direct sum at `m` targets from all `n` sources (verification).
template <class T, bool GRAD>
__global__ void __launch_bounds__(kP2PThreads) direct_kernel(const v4_t<T>* __restrict__ src, int64_t n,
                                                              const int64_t* __restrict__ targets, int64_t m,
                                                              T* __restrict__ pot, T* __restrict__ grad) {
  __shared__ v4_t<T> sh[kP2PThreads];
  const int64_t r = int64_t(blockIdx.x) * kP2PThreads + threadIdx.x;
  v4_t<T> x = src[targets[r < m ? r : 0]];
  T a = 0, ax = 0, ay = 0, az = 0;
  for (int64_t base = 0; base < n; base += kP2PThreads) {
    const int64_t j = base + threadIdx.x;
    sh[threadIdx.x] = j < n ? src[j] : make4<T>(T(0), T(0), T(0), T(0));
    __syncthreads();
    const int cnt = (n - base) < kP2PThreads ? int(n - base) : kP2PThreads;
    for (int i = 0; i < cnt; ++i) {
      const v4_t<T> s = sh[i];
      const T dx = x.x - s.x, dy = x.y - s.y, dz = x.z - s.z;
      const T ri = rinv_masked(dx * dx + dy * dy + dz * dz);
      const T qr = s.w * ri;
      a += qr;
      if (GRAD) {
        const T qr3 = qr * ri * ri;
        ax += qr3 * dx;
        ay += qr3 * dy;
        az += qr3 * dz;
      }
    }
    __syncthreads();
  }
  if (r < m) {
    const T c = T(kInv4PiD);
    pot[r] = c * a;
    if (GRAD) {
      grad[3 * r] = -c * ax;
      grad[3 * r + 1] = -c * ay;
      grad[3 * r + 2] = -c * az;
    }
  }
}

// src[i] = (x_i, y_i, z_i, q_perm(i)); perm = original_index when charges are in input order.
template <class T>
__global__ void pack_sources_kernel(const v4_t<T>* __restrict__ pos, const T* __restrict__ q,
                                    const int* __restrict__ perm, int n, v4_t<T>* __restrict__ src) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  v4_t<T> v = pos[i];
  v.w = q[perm ? perm[i] : i];
  src[i] = v;
}

// out[perm[i]] = in[i] for i in [begin, end) (potential: width 1, gradient: width 3).
template <class T>
__global__ void unpermute_kernel(const T* __restrict__ in, const int* __restrict__ perm, int begin, int end,
                                 int width, T* __restrict__ out) {
  const int i = begin + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= end) return;
  const int o = perm ? perm[i] : i;
  for (int d = 0; d < width; ++d) out[size_t(o) * width + d] = in[size_t(i) * width + d];
}

// FFMA/DFMA throughput probe: 8 independent chains per thread.
template <class T>
__global__ void fma_probe_kernel(T* out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = T(threadIdx.x + i);
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == T(-1.2345)) out[0] = s;
}

}  // namespace gpu
}  // namespace kifmm
