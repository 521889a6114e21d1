// Latency probe: cycles per dependent fp64 operation (DFMA, DMUL, DADD, reciprocal, division, sqrt) and per
// shared-memory round trip / __syncthreads on one SM, from clock64() around unrolled dependent chains.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double x0, int n) {
  __shared__ double sh[64];
  double x = x0 + threadIdx.x * 1e-9, y = 0.9999999;
  if (threadIdx.x < 64) sh[threadIdx.x] = x;
  __syncthreads();
  long long t0, t1;
#define CHAIN(idx, body)                        \
  t0 = clock64();                               \
  for (int i = 0; i < n; ++i) {                 \
    _Pragma("unroll") for (int u = 0; u < 16; ++u) { body; } \
  }                                             \
  t1 = clock64();                               \
  if (threadIdx.x == 0) cyc[idx] = t1 - t0;
  CHAIN(0, x = fma(x, y, 1e-12))
  CHAIN(1, x = x * y)
  CHAIN(2, x = x + 1e-12)
  CHAIN(3, x = 1.0 / (x + 1.5))
  CHAIN(4, x = sqrt(x + 1.0))
  CHAIN(5, x = sh[((int)x) & 63] + x * 1e-3)
  CHAIN(6, { sh[threadIdx.x & 63] = x; __syncthreads(); x = sh[(threadIdx.x + 1) & 63] * y; })
  CHAIN(7, { __syncthreads(); })
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 64 * sizeof(long long));
  const char* names[] = {"DFMA", "DMUL", "DADD", "1/x (div)", "sqrt", "LDS+DFMA", "STS+bar+LDS+DMUL", "bar only"};
  for (int threads : {32, 256}) {
    const int n = 64;
    lat<<<1, threads>>>(out, cyc, 1.0, n);
    cudaDeviceSynchronize();
    lat<<<1, threads>>>(out, cyc, 1.0, n);
    cudaDeviceSynchronize();
    for (int i = 0; i < 8; ++i) printf("%d threads: %-20s %.1f cycles per op\n", threads, names[i], cyc[i] / (16.0 * n));
  }
  return 0;
}
