// Volume-primitive kernels, baseline version (one thread per lattice node).
#pragma once
#include "fem_device.cuh"
#include "hhg_internal.h"

namespace hhg {

enum { kModeApply = 0, kModeResid = 1, kModeGS = 2 };

// 15 stencil weights of interior node (i,j,k) for operator `op`:
//  SURROGATE: P s_w(i,j,k) = sum_c coef[w][c] i^l j^m k^n (index units,
//             degree-major exponent order, PAPER.md eq. quadraticPolynomial);
//  FEM_ELEMENTWISE here: node-wise exact FEM (24 fine tets);
//  CONST_AFFINE: the macro's constant affine stencil.
__device__ inline void node_weights(int op, int N, int i, int j, int k, const double* geo,
                                    const double* coef, int mq, const double* cons, bool blended,
                                    double s[15]) {
  if (op == HHG_OP_SURROGATE) {
    double pi[5], pj[5], pk[5];
    pi[0] = pj[0] = pk[0] = 1.0;
    for (int e = 1; e < 5; ++e) {
      pi[e] = pi[e - 1] * i;
      pj[e] = pj[e - 1] * j;
      pk[e] = pk[e - 1] * k;
    }
    int q = 0;
    while ((q + 3) * (q + 2) * (q + 1) / 6 < mq) ++q;
    for (int w = 0; w < 15; ++w) {
      const double* a = coef + w * mq;
      double acc = 0.0;
      int c = 0;
      for (int d = 0; d <= q; ++d)
        for (int l = d; l >= 0; --l)
          for (int m = d - l; m >= 0; --m) acc += a[c++] * pi[l] * pj[m] * pk[d - l - m];
      s[w] = acc;
    }
  } else if (op == HHG_OP_CONST_AFFINE) {
    for (int w = 0; w < 15; ++w) s[w] = cons[w];
  } else {
    fem_partial(geo, N, i, j, k, blended, s);
  }
}

static __global__ void k_vol_v1(int N, int64_t S, int64_t P, const double* __restrict__ geo,
                         const double* __restrict__ coef, int mq, const double* __restrict__ cons,
                         int op, bool blended, int mode, int colour, const double* u,
                         const double* __restrict__ f, double* out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t T = blockIdx.y;
  if (p >= P) return;
  int i, j, k;
  decode_pos(N, p, i, j, k);
  if (i < 1 || j < 1 || k < 1 || i + j + k > N - 1) return;
  if (mode == kModeGS && ((i + 2 * j + 3 * k) & 3) != colour) return;
  double s[15];
  node_weights(op, N, i, j, k, geo + T * 16, coef ? coef + T * 15 * mq : nullptr, mq, cons + T * 15,
               blended, s);
  const double* ub = u + T * S;
  double acc = 0.0;
  for (int w = 0; w < 15; ++w) {
    if (mode == kModeGS && w == kMC) continue;
    int64_t q = lattice_pos(N, i + kDir[w][0], j + kDir[w][1], k + kDir[w][2]);
    acc += s[w] * ub[q];
  }
  const int64_t o = T * S + p;
  if (mode == kModeApply) out[o] = acc;
  else if (mode == kModeResid) out[o] = f[o] - acc;
  else out[o] = (f[o] - acc) / s[kMC];
}

}  // namespace hhg
