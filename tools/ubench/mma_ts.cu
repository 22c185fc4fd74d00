// Microbenchmark: cta_group::1 kind::f16 M=128 K=16 N=160, three MMAs per K step (the fp16 3-term
// split pattern), commit every 6 MMAs (one stage), A from shared memory (mode 0) or from tensor
// memory (mode 1).  Clocks per MMA instruction.
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

__global__ void __launch_bounds__(128, 1) k(int n, int iters, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t ring[8];
  unsigned char* s = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < 8; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ring[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t ah = smem_u32(s), al = smem_u32(s + 8192), bh = smem_u32(s + 16384), bl = smem_u32(s + 16384 + 10240);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint64_t dbh = desc(bh + 32 * kk), dbl = (mode == 4 || mode == 5 || mode == 6) ? dbh : desc(bl + 32 * kk);
        if (mode == 0 || mode == 2 || mode == 4 || mode >= 6) {
          const uint64_t dah = desc(ah + 32 * kk), dal = mode == 6 ? dah : desc(al + 32 * kk);
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem), "l"(dah), "l"(dbh), "r"(idesc), "r"(1u));
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem), "l"(dah), "l"(dbl), "r"(idesc), "r"(1u));
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem), "l"(dal), "l"(dbh), "r"(idesc), "r"(1u));
        } else {
          const uint32_t tah = tmem + 256 + 8 * kk, tal = tmem + 256 + 16 + 8 * kk;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem), "r"(tah), "l"(dbh), "r"(idesc), "r"(1u));
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem), "r"(tah), "l"(dbl), "r"(idesc), "r"(1u));
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem), "r"(tal), "l"(dbh), "r"(idesc), "r"(1u));
        }
      }
      if (mode != 2 && mode != 3 && mode != 6 && mode != 8)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&ring[i & 7])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&ring[iters & 7])) : "memory");
    uint32_t done = 0;
    const uint32_t par = (iters >> 3) & 1;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(smem_u32(&ring[iters & 7])), "r"(par) : "memory");
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 4000;
  for (int mode : {2, 6, 7, 8})
    for (int n : {160}) {
      k<<<148, 128, 200 * 1024>>>(n, 16, mode, d);
      k<<<148, 128, 200 * 1024>>>(n, iters, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += double(h[i]);
      avg /= 148;
      const double per = avg / (iters * 6.0);
      printf("mode %d (A %s) N %3d: %.1f clk/MMA  -> %.0f flop/clk/SM (%s)\n", mode, mode ? "tmem" : "smem", n, per,
             2.0 * 128 * n * 16 / per, cudaGetErrorString(e));
    }
  return 0;
}
