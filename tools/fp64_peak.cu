// fp64 FMA peak probe (a measured fp64 peak for the sparse factorization's roofline).
// Each thread runs NACC independent DFMA chains; the grid fills every SM with many warps. Reports TFLOP/s
// (2 flops per FMA) from CUDA events, best of several runs, with the SM clock left alone.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bps : {4, 8}) {
    const int blocks = sms * bps;
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    const double fl = 2.0 * 8.0 * iters * (double)threads * blocks;
    printf("fp64 FMA: %d SMs, %d CTAs x %d threads, 8 chains/thread: %.3f ms -> %.2f TFLOP/s "
           "(nominal at the %.0f MHz max clock: %.2f TFLOP/s = 64 FMA/clk/SM)\n",
           sms, blocks, threads, best, fl / (best * 1e-3) / 1e12, clk / 1e3, 2.0 * 64 * sms * clk * 1e3 / 1e12);
  }
  return 0;
}
