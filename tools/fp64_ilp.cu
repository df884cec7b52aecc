// DFMA throughput vs. independent chains per thread and warps per SM (dev tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_ilp tools/fp64_ilp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chains(double* out, int iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int q = 0; q < C; ++q) x[q] = threadIdx.x * 1e-9 + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < C; ++q) x[q] = fma(x[q], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < C; ++q) s += x[q];
  if (s == 1234.5) out[0] = s;
}

template <int C>
void run(int sms, int warps_per_sm, double* out) {
  const int threads = 256;
  const int blocks = sms * warps_per_sm * 32 / threads;
  const int iters = 4096 / C;
  chains<C><<<blocks, threads>>>(out, 10, 0.999, 1e-3);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    chains<C><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double dfma = (double)blocks * threads * iters * 8 * C;
  printf("chains %2d warps/SM %2d : %.2f DFMA/clk/SM (at 1.965 GHz)\n", C, warps_per_sm,
         dfma / (best * 1e-3) / sms / 1.965e9);
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  for (int w : {8, 16, 32, 64}) {
    run<1>(sms, w, out);
    run<2>(sms, w, out);
    run<4>(sms, w, out);
    run<8>(sms, w, out);
  }
  return 0;
}
