// On-the-fly FEM apply / residual (the paper's comparison operator,
// PAPER.md:385-394, 1102-1122): every interior node's 15 stencil weights are
// assembled from the local stiffness matrices of its 24 incident fine tets,
// with the fine-tet vertices at their blended positions, on every call
// (nothing stored).  Column-march structure of march.cuh: thread = lattice
// column, planes of u through a TMA ring.  What the v1 node-wise kernel
// recomputed per tet is shared here: every blended node position is computed
// once per call (plane by plane into a 4-plane shared-memory ring, by the
// threads of the band) and the 24 incident tets of an interior node come from
// a fixed direction table.  Per tet the row entry needs only
// sum_a K_T[m][a] u_a = |T| grad(l_m).grad(u_h): 3 cross products, the
// determinant, grad(u_h) from 3 differences, one dot product and one division
// (~55 fp64 instructions, ~1.3 k per node).  Same quantity as the oracle's
// definition (blended vertices, K_T = |T| grad(l_a).grad(l_b)); the order of
// the arithmetic differs.
#pragma once
#include "fem_device.cuh"
#include "march.cuh"

namespace hhg {

constexpr int kFRing = 8;  // u plane slots
constexpr int kFPosPerThread = 3;  // ring columns per thread whose positions it computes

// The 24 fine tets incident to an interior lattice node, as the directions
// (HHG_DIRS_INIT order; 7 = the node) of their 4 vertices -- fem_partial's
// enumeration (6 Kuhn paths x the node's position m = t % 4 on the path).
__device__ constexpr int kFemTet[24][4] = {{7, 8, 10, 14}, {6, 7, 9, 13},  {4, 5, 7, 12},  {0, 1, 2, 7},   {7, 8, 11, 14},
                                {6, 7, 12, 13}, {3, 2, 7, 9},   {0, 1, 5, 7},   {7, 9, 10, 14}, {5, 7, 8, 11},
                                {4, 6, 7, 12},  {0, 3, 2, 7},   {7, 9, 13, 14}, {5, 7, 12, 11}, {1, 2, 7, 8},
                                {0, 3, 6, 7},   {7, 12, 11, 14}, {2, 7, 8, 10},  {3, 6, 7, 9},   {0, 4, 5, 7},
                                {7, 12, 13, 14}, {2, 7, 9, 10},  {1, 5, 7, 8},   {0, 4, 6, 7}};

struct FemSmem {
  double* ring;   // [kFRing][slot_len] u planes
  double* pos;    // [4][3][slot_len] node positions (x, y, z planes) of lattice planes k mod 4
  uint64_t* bars; // [kFRing]
  int* po;        // [N+2]
  __device__ FemSmem(double* smem, int slot_len, int N) {
    ring = smem;
    pos = ring + (size_t)kFRing * slot_len;
    bars = (uint64_t*)(pos + (size_t)12 * slot_len);
    po = (int*)(bars + kFRing);
  }
};

__host__ __device__ inline size_t fem_smem_bytes(int slot_len, int N) {
  return (size_t)kFRing * slot_len * 8 + (size_t)12 * slot_len * 8 + kFRing * 8 + (size_t)(N + 2) * 4;
}

template <int MODE>
__global__ void __launch_bounds__(kMarchThreads, 2)
    k_vol_fem(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
              const double* __restrict__ geo_all, bool blended, const double* __restrict__ u,
              const double* __restrict__ f, double* __restrict__ out) {
  extern __shared__ __align__(16) double smem[];
  FemSmem sm(smem, slot_len, N);
  const int64_t T = blockIdx.x / n_bands;
  const Band b = bands[blockIdx.x - T * n_bands];
  const double* ub = u + T * S;
  const double* geo = geo_all + T * 16;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFRing; ++s) mbar_init(&sm.bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) sm.po[p] = (int)plane_off(N, p);
  __syncthreads();

  const int last_plane = b.kmax + 1;
  int next_issue = min(kFRing - 1, last_plane + 1);
  issue_planes<kFRing>(ub, sm.po, 0, next_issue - 1, b, sm.ring, slot_len, sm.bars);
  const Column q = make_column(b, N);
  const int clo = b.c_lo;
  // lattice columns of the ring range this thread computes positions for
  // (ring range <= 3 x 256 columns: N = 256 single-diagonal bands span 3 diagonals)
  int pc_i[kFPosPerThread], pc_j[kFPosPerThread];
  for (int r = 0; r < kFPosPerThread; ++r) {
    const int c = clo + (int)threadIdx.x + r * kMarchThreads;
    int d = (int)((sqrt(8.0 * (double)c + 1.0) - 1.0) * 0.5);
    while ((d + 1) * (d + 2) / 2 <= c) ++d;
    while (d * (d + 1) / 2 > c) --d;
    pc_j[r] = c - d * (d + 1) / 2;
    pc_i[r] = d - pc_j[r];
  }
  auto positions = [&](int k) {  // plane k -> pos slot k & 3
    double* P = sm.pos + (size_t)(k & 3) * 3 * slot_len;
    for (int r = 0; r < kFPosPerThread; ++r) {
      const int o = (int)threadIdx.x + r * kMarchThreads;
      if (o >= b.ncols + 1) continue;
      const int i = pc_i[r], j = pc_j[r];
      if (i < 0 || j < 0 || i + j + k > N) continue;
      double x[3];
      node_xyz(geo, N, i, j, k, blended, x);
      P[o] = x[0];
      P[slot_len + o] = x[1];
      P[2 * slot_len + o] = x[2];
    }
  };
  positions(0);
  positions(1);
  auto sptr = [&](int p) -> const double* {
    return sm.ring + (p % kFRing) * slot_len + ((sm.po[p] + clo) & 1);
  };
  double* const optr = out + T * S + q.c;
  const double* const fptr = f + T * S + q.c;
  for (int k = 1; k <= b.kmax; ++k) {
    positions(k + 1);
    __syncthreads();  // positions of k+1 visible; every thread is done with step k-1 (u plane k-2 free)
    if (k + 6 <= last_plane && k + 6 >= next_issue) {
      issue_planes<kFRing>(ub, sm.po, k + 6, k + 6, b, sm.ring, slot_len, sm.bars);
      next_issue = k + 7;
    }
    mbar_wait(&sm.bars[(k + 1) % kFRing], ((k + 1) / kFRing) & 1);
    if (k == 1) mbar_wait(&sm.bars[0], 0), mbar_wait(&sm.bars[1], 0);
    if (!(q.active && k <= q.len)) continue;
    double fv = 0.0;
    if (MODE == kModeResid) fv = __ldg(fptr + sm.po[k]);
    const double* Pl0 = sm.pos + (size_t)((k - 1) & 3) * 3 * slot_len;
    const double* Pl1 = sm.pos + (size_t)(k & 3) * 3 * slot_len;
    const double* Pl2 = sm.pos + (size_t)((k + 1) & 3) * 3 * slot_len;
    const double* Ul0 = sptr(k - 1);
    const double* Ul1 = sptr(k);
    const double* Ul2 = sptr(k + 1);
    // y_I = sum over the 24 incident tets T of sum_a |T| grad(l_I).grad(l_a) u_a
    double acc = 0.0;
    // ring offsets of the 15 directions (7 distinct columns)
    const int ocol[15] = {q.o_c, q.o_e, q.o_n, q.o_nw, q.o_s, q.o_se, q.o_w, q.o_c,
                          q.o_e, q.o_nw, q.o_n, q.o_se, q.o_s, q.o_w, q.o_c};
#pragma unroll
    for (int t = 0; t < 24; ++t) {
      double P[4][3], uv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int w = kFemTet[t][a];  // compile-time after unrolling
        const int o = ocol[w];
        const double* pp = w <= 3 ? Pl0 : (w <= 10 ? Pl1 : Pl2);
        const double* up = w <= 3 ? Ul0 : (w <= 10 ? Ul1 : Ul2);
        P[a][0] = pp[o];
        P[a][1] = pp[slot_len + o];
        P[a][2] = pp[2 * slot_len + o];
        uv[a] = up[o];
      }
      double e1[3], e2[3], e3[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        e1[d] = P[1][d] - P[0][d];
        e2[d] = P[2][d] - P[0][d];
        e3[d] = P[3][d] - P[0][d];
      }
      const double c23[3] = {e2[1] * e3[2] - e2[2] * e3[1], e2[2] * e3[0] - e2[0] * e3[2],
                             e2[0] * e3[1] - e2[1] * e3[0]};
      const double c31[3] = {e3[1] * e1[2] - e3[2] * e1[1], e3[2] * e1[0] - e3[0] * e1[2],
                             e3[0] * e1[1] - e3[1] * e1[0]};
      const double c12[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                             e1[0] * e2[1] - e1[1] * e2[0]};
      const double det = e1[0] * c23[0] + e1[1] * c23[1] + e1[2] * c23[2];
      // sum_a |T| grad(l_m).grad(l_a) u_a = |T| grad(l_m).grad(u_h), and with
      // c_a = det grad(l_a) (a = 1..3, c_0 = -(c_1 + c_2 + c_3)) and
      // det grad(u_h) = sum_{a>=1} c_a (u_a - u_0) =: G this is (c_m . G) / (6 |det|)
      const double du1 = uv[1] - uv[0], du2 = uv[2] - uv[0], du3 = uv[3] - uv[0];
      double G[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) G[d] = fma(c23[d], du1, fma(c31[d], du2, c12[d] * du3));
      const int m = t & 3;
      double cm[3];
#pragma unroll
      for (int d = 0; d < 3; ++d)
        cm[d] = m == 1 ? c23[d] : m == 2 ? c31[d] : m == 3 ? c12[d] : -(c23[d] + c31[d] + c12[d]);
      const double dot = fma(cm[0], G[0], fma(cm[1], G[1], cm[2] * G[2]));
      acc = fma(dot, 1.0 / (6.0 * fabs(det)), acc);
      asm volatile("" ::: "memory");  // keep one tet's loads live at a time (register pressure)
    }
    optr[sm.po[k]] = (MODE == kModeResid) ? fv - acc : acc;
  }
}

}  // namespace hhg
