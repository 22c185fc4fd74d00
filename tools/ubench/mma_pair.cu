// Microbenchmark: tcgen05.mma kind::f16 cta_group::2 (M=256 over a CTA pair, K=16) issue rate vs N,
// plain back-to-back issue (mode 0) and with a per-6-MMA commit + mbarrier wait round trip (mode 1,
// the stage structure of the M2L kernel).  Prints clocks per MMA instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t((8 * 64) >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(4) << 61;
  return d;
}
__device__ __forceinline__ uint32_t rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done)
                 : "r"(bar), "r"(par)
                 : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(int n, int iters, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t ring[8];
  unsigned char* s = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  const uint32_t r = rank();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int q = 0; q < 8; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ring[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0 && r == 0) {
    const uint32_t idesc = (1u << 4) | (uint32_t(n >> 3) << 17) | (uint32_t(256 >> 4) << 24);
    const uint32_t a = smem_u32(s), b = smem_u32(s + 128 * 64 * 4);
    unsigned long long t0 = clock64();
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const uint64_t da = desc(a + 32 * (j & 1) + 8192 * (j >> 1)), db = desc(b + 32 * (j & 1));
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(1u));
      }
      if (mode == 4 && (i & 1)) {  // commit every 12 MMAs, multicast
        asm volatile(
            "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(
                smem_u32(&ring[(i >> 1) & 7]))
            : "memory");
      }
      if (mode == 5) {  // commit every 6 MMAs, leader only (no multicast)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&ring[i & 7]))
                     : "memory");
      }
      if (mode == 2 || mode == 3) {
        const int q = i & 7;
        if (mode == 3 && i >= 8) wait(smem_u32(&ring[q]), ((i >> 3) - 1) & 1);
        asm volatile(
            "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(
                smem_u32(&ring[q]))
            : "memory");
      }
      if (mode == 1) {
        asm volatile(
            "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(
                smem_u32(&bar))
            : "memory");
        wait(smem_u32(&bar), ph);
        ph ^= 1;
      }
    }
    asm volatile(
        "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(
            smem_u32(&bar))
        : "memory");
    wait(smem_u32(&bar), ph);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  } else if (threadIdx.x == 0) {
    // peer: wait for the multicast commits
    uint32_t ph = 0;
    const int waits = (mode == 1 ? iters : 0) + 1;
    for (int i = 0; i < waits; ++i) {
      wait(smem_u32(&bar), ph);
      ph ^= 1;
    }
    out[blockIdx.x] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 3000;
  for (int mode : {0, 2, 4, 5})
    for (int n : {64, 128, 160, 256}) {
      k<<<148, 128, 200 * 1024>>>(n, 10, mode, d);
      k<<<148, 128, 200 * 1024>>>(n, iters, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; i += 2) avg += double(h[i]);
      avg /= 74;
      const double per = avg / (iters * 6.0);
      printf("mode %d N %3d: %.1f clk/MMA  -> %.0f flop/clk/SM (%s)\n", mode, n, per, 2.0 * 128 * n * 16 / per,
             cudaGetErrorString(e));
    }
  return 0;
}
