// Lexicographic volume Gauss-Seidel (the paper's own hybrid smoother,
// PAPER.md:1317-1330): the volume nodes of a macro are
// visited west to east (i), south to north (j), bottom to top (k), each from
// the newest values.
//
// GPU form: node (i,j,k) lies on the hyperplane w = i + 2j + 3k.  Its seven
// lexicographic predecessors among the 14 neighbours (bc, be, bn, bnw, ms,
// mse, mw) have w - 3 .. w - 1 and its seven successors w + 1 .. w + 3, and no
// two neighbours share a hyperplane -- so sweeping the hyperplanes in order,
// all nodes of one hyperplane at once, IS the lexicographic order, exactly.
// One CTA per macro; a thread owns i-lines (j, k) and, at hyperplane w,
// updates the node i = w - 2j - 3k of each of its lines that is inside the
// macro; a CTA barrier separates the hyperplanes.  Weights are evaluated in
// full per node from the macro's coefficients in shared memory (s_w =
// A_w(i,j) + k (B_w(i,j) + k C_w)), neighbours read from global memory (the
// few hyperplanes in flight stay in L1/L2).
#pragma once
#include "march.cuh"

namespace hhg {

constexpr int kLexThreads = 512;

template <int OP>
__global__ void __launch_bounds__(kLexThreads, 2)
    k_gs_lex(int N, int64_t S, const double* __restrict__ coef10, const double* __restrict__ cons,
             double* __restrict__ u, const double* __restrict__ f, int T0) {
  extern __shared__ __align__(16) double lsm[];
  double* cf = lsm;                       // [150] coefficients (surrogate) / [15] constant stencil
  int* po = (int*)(cf + 152);             // [N+2] plane offsets
  uint32_t* lines = (uint32_t*)(po + 260);  // [(N-2)(N-3)/2] (j | k << 16)
  const int64_t T = T0 + blockIdx.x;
  for (int x = threadIdx.x; x < 150; x += blockDim.x)
    cf[x] = OP == HHG_OP_SURROGATE ? coef10[T * 150 + x] : (x < 15 ? cons[T * 15 + x] : 0.0);
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) po[p] = (int)plane_off(N, p);
  // i-lines (j, k), j, k >= 1, j + k <= N - 2, in order of their first hyperplane
  const int nlines = (N - 2) * (N - 3) / 2;
  for (int x = threadIdx.x; x < nlines; x += blockDim.x) {
    int m = (int)((sqrt(8.0 * (double)x + 1.0) - 1.0) * 0.5);  // m = j + k - 2
    while ((m + 1) * (m + 2) / 2 <= x) ++m;
    while (m * (m + 1) / 2 > x) --m;
    const int k = x - m * (m + 1) / 2 + 1, j = m + 2 - k;
    lines[x] = (uint32_t)j | ((uint32_t)k << 16);
  }
  __syncthreads();
  double* ub = u + T * S;
  const double* fb = f + T * S;
  for (int w = 6; w <= 3 * N - 6; ++w) {
    for (int x = threadIdx.x; x < nlines; x += blockDim.x) {
      const int j = (int)(lines[x] & 0xffff), k = (int)(lines[x] >> 16);
      const int i = w - 2 * j - 3 * k;
      if (i < 1 || i + j + k > N - 1) continue;
      const double di = (double)i, dj = (double)j, dk = (double)k;
      double r = 0.0, smc = 0.0;
#pragma unroll
      for (int q = 0; q < 15; ++q) {
        double s;
        if (OP == HHG_OP_SURROGATE) {
          const double* a = cf + q * 10;  // (000)(100)(010)(001)(200)(110)(101)(020)(011)(002)
          const double A = a[0] + di * (a[1] + di * a[4] + dj * a[5]) + dj * (a[2] + dj * a[7]);
          const double B = a[3] + di * a[6] + dj * a[8];
          s = fma(fma(a[9], dk, B), dk, A);
        } else {
          s = cf[q];
        }
        if (q == kMC) {
          smc = s;
        } else {
          const int a = i + kDir[q][0], b = j + kDir[q][1], c = k + kDir[q][2];
          r = fma(s, ub[po[c] + col_idx(a, b)], r);
        }
      }
      const int64_t p = po[k] + col_idx(i, j);
      ub[p] = (fb[p] - r) * rcp_nr(smc);
    }
    __syncthreads();  // hyperplane w written before w + 1 reads it
  }
}

__host__ __device__ inline size_t lex_smem_bytes(int N) {
  return 152 * 8 + 260 * 4 + (size_t)(N - 2) * (N - 3) / 2 * 4;
}

}  // namespace hhg
