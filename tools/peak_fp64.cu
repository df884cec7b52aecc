// Measures the B200 fp64 FMA throughput (DFMA/s) -- the second roofline
// denominator of the surrogate kernels ("not measured; measure
// first").  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// /tmp/peak_fp64 tools/peak_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = threadIdx.x * 1e-9 + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += x[q];
  if (s == 1234.5) out[0] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000, threads = 512, blocks = sms * 4;
  dfma_loop<<<blocks, threads>>>(out, 100, 0.999, 1e-3);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double dfma = (double)blocks * threads * iters * 8;
  printf("{\"sms\": %d, \"dfma_per_s\": %.4e, \"fp64_tflops\": %.3f, \"dfma_per_clk_per_sm_at_1965MHz\": %.2f}\n",
         sms, dfma / (best * 1e-3), 2 * dfma / (best * 1e-3) / 1e12, dfma / (best * 1e-3) / sms / 1.965e9);
  return 0;
}
