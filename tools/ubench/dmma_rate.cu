// Microbenchmark: FP64 throughput on the SM -- warp-level DMMA (mma.sync m8n8k4 f64, register operands,
// independent accumulators) vs DFMA (8 independent chains per thread).  Prints TFLOP/s for a full grid.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dmma_k(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[0] = s;
}

__global__ void __launch_bounds__(256) dfma_k(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999, 1e-3);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == -1.2345) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int blocks_per_sm : {2, 4, 8}) {
    const int blocks = sms * blocks_per_sm, iters = 4096;
    dmma_k<<<blocks, 256>>>(out, 64);
    cudaEventRecord(a);
    dmma_k<<<blocks, 256>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fl = double(blocks) * (256 / 32) * iters * 8 * (8 * 8 * 4 * 2);
    dfma_k<<<blocks, 256>>>(out, 64);
    cudaEventRecord(a);
    dfma_k<<<blocks, 256>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms2;
    cudaEventElapsedTime(&ms2, a, b);
    const double fl2 = double(blocks) * 256 * iters * 8 * 2;
    std::printf("blocks/SM %d: DMMA m8n8k4 %.1f TFLOP/s   DFMA %.1f TFLOP/s  (%s)\n", blocks_per_sm,
                fl / (ms * 1e-3) / 1e12, fl2 / (ms2 * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
