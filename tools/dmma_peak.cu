// fp64 tensor-core (DMMA, mma.sync .f64) peak probe: whether the sparse factorization's rank-k updates gain from
// the fp64 MMA path over plain DFMA (tools/fp64_peak.cu). Each warp runs NCH independent accumulator chains of
// one MMA shape; flops = 2·m·n·k per MMA per warp. Best of several runs, CUDA events, clocks untouched.
#include <cstdio>
#include <cuda_runtime.h>

template <int NCH>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1e-3 * threadIdx.x, b = 0.999;
  double c[NCH][2];
#pragma unroll
  for (int i = 0; i < NCH; ++i) c[i][0] = c[i][1] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NCH>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int e = 0; e < 8; ++e) a[e] = 1e-3 * threadIdx.x + e;
#pragma unroll
  for (int e = 0; e < 4; ++e) b[e] = 0.999 - 1e-4 * e;
  double c[NCH][4];
#pragma unroll
  for (int i = 0; i < NCH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
            "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
static void run(const char* name, K kern, double flops_per_mma_warp, int nch, int sms) {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  for (int wps : {4, 8, 16}) {
    const int threads = 128, blocks = sms * wps / 4;
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    const cudaError_t err = cudaGetLastError();
    const double fl = flops_per_mma_warp * nch * (double)iters * (blocks * threads / 32);
    printf("%s: %d warps/SM, %d chains/warp: %.3f ms -> %.2f TFLOP/s %s\n", name, wps, nch, best,
           fl / (best * 1e-3) / 1e12, err ? cudaGetErrorString(err) : "");
  }
  cudaFree(out);
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  run("mma m8n8k4 f64", dmma_m8n8k4<8>, 2.0 * 8 * 8 * 4, 8, sms);
  run("mma m16n8k16 f64", dmma_m16n8k16<4>, 2.0 * 16 * 8 * 16, 4, sms);
  return 0;
}
