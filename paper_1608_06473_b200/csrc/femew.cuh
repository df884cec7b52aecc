// Element-wise on-the-fly FEM apply / residual (the paper's
// comparison operator): y = sum_T K_T u_T over
// the N^3 fine tets of every macro, K_T = |T| grad(l_a).grad(l_b) from the
// BLENDED vertex positions, recomputed on every call (nothing stored).
//
// Structure (column march of march.cuh): CTA = (macro, band of diagonals
// [d0, d1)), marching the slabs k0 -> k0+1.  The fine tets are the 6 Kuhn
// simplices of the lattice "cubes" anchored at (i0, j0, k0): with
// X = i+j+k, Y = j+k, Z = k the macro is {0 <= Z <= Y <= X <= N} and the fine
// mesh is the Kuhn triangulation of the unit cubes in XYZ (a cube with
// i0 = 0 keeps the 3 tets stepping X before Y, j0 = 0 the 3 stepping Y before
// Z).  Cube corner (a,b,c) (XYZ offsets) is lattice node
// (i0 + a - b, j0 + b - c, k0 + c), so a cube anchored on diagonal D touches
// diagonals D-1..D+1 -- all inside the band's plane range [d0-1, d1] when the
// band computes the cubes anchored on its OWN diagonals.  Every cube is
// therefore computed exactly once per call:
//   * per slab, each thread computes the cubes of its anchor columns (blended
//     positions and u of the 8 corners from shared memory) and leaves the 8
//     corner sums sum_b K_ab u_b in shared memory (bottom corners for this
//     slab, top corners double-buffered for the next one);
//   * each interior node of the band then adds its 8 corner sums (4 cubes of
//     slab k, 4 of slab k-1);
//   * nodes of the two neighbouring diagonals d0-1 and d1 receive the sums of
//     this band's cubes through scratch vectors, added to their owner band's
//     output by k_fem_ew_fixup (fixed order: deterministic).
// Per tet, sum_b K_ab u_b = (c_a . G) / (6 |det|) with c_a = det grad(l_a) and
// G = det grad(u_h) = sum_{b>=1} c_b (u_b - u_0): 3 cross products, one
// reciprocal, 4 dot products.  Same quantity as the oracle's element-wise
// definition (fem.assemble); the order of the sums differs.
#pragma once
#include "fem_device.cuh"
#include "march.cuh"

namespace hhg {

constexpr int kFPosPerThread = 3;  // ring columns per thread whose positions it computes
constexpr int kEwRing = 6;  // u plane slots (slab k0 reads planes k0, k0+1)

// corner index a | b<<1 | c<<2; the 6 Kuhn tets (step orders XYZ, XZY, YXZ,
// YZX, ZXY, ZYX) as corner sequences from (000) to (111)
__device__ constexpr int kKuhn[6][4] = {{0, 1, 3, 7}, {0, 1, 5, 7}, {0, 2, 3, 7},
                                        {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 4, 6, 7}};

struct EwSmem {
  double* ring;  // [kEwRing][slot] u planes
  double* pos;   // [2][3][slot] blended positions of planes k mod 2
  double* bot;   // [4][slot] sums at corners 0..3 (plane k0) of the cubes of slab k0
  double* top;   // [2][4][slot] sums at corners 4..7 (plane k0+1), slab parity
  uint64_t* bars;
  int* po;
  __device__ EwSmem(double* smem, int slot) {
    ring = smem;
    pos = ring + (size_t)kEwRing * slot;
    bot = pos + (size_t)6 * slot;
    top = bot + (size_t)4 * slot;
    bars = (uint64_t*)(top + (size_t)8 * slot);
    po = (int*)(bars + kEwRing);
  }
};

__host__ __device__ inline size_t ew_smem_bytes(int slot, int N) {
  return (size_t)(kEwRing + 6 + 4 + 8) * slot * 8 + kEwRing * 8 + (size_t)(N + 2) * 4;
}

__device__ __forceinline__ void col_ij(int c, int& i, int& j) {
  int d = (int)((sqrt(8.0 * (double)c + 1.0) - 1.0) * 0.5);
  while ((d + 1) * (d + 2) / 2 <= c) ++d;
  while (d * (d + 1) / 2 > c) --d;
  j = c - d * (d + 1) / 2;
  i = d - j;
}

// ring offset of lattice column (i, j), clamped into the slot (values at
// clamped offsets belong to corners of tets that are never used)
__device__ __forceinline__ int ring_off(int i, int j, int clo, int slot) {
  const int o = (int)col_idx(i, j) - clo;
  return min(max(o, 0), slot - 1);
}

template <int MODE>
__global__ void __launch_bounds__(kMarchThreads, 2)
    k_vol_fem_ew(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
                 const double* __restrict__ geo_all, bool blended, const double* __restrict__ u,
                 const double* __restrict__ f, double* __restrict__ out, double* __restrict__ s_lo,
                 double* __restrict__ s_hi) {
  extern __shared__ __align__(16) double smem[];
  EwSmem sm(smem, slot_len);
  const int64_t T = blockIdx.x / n_bands;
  const int bi = (int)(blockIdx.x - T * n_bands);
  Band b = bands[bi];
  // the first band also owns the cubes anchored on diagonal 1 (their corners
  // reach diagonal 0): its plane range starts at column 0
  const int a_lo = b.d0 == 2 ? 1 : b.d0;
  if (b.d0 == 2) {
    b.ncols += b.c_lo;
    b.c_lo = 0;
  }
  const int clo = b.c_lo;
  const double* ub = u + T * S;
  const double* geo = geo_all + T * 16;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kEwRing; ++s) mbar_init(&sm.bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) sm.po[p] = (int)plane_off(N, p);
  for (int x = threadIdx.x; x < 12 * slot_len; x += blockDim.x) sm.bot[x] = 0.0;  // bot and top
  __syncthreads();

  const int last_plane = b.kmax + 1;
  int next_issue = min(kEwRing - 1, last_plane + 1);
  issue_planes<kEwRing>(ub, sm.po, 0, next_issue - 1, b, sm.ring, slot_len, sm.bars);

  // ---- position pass columns (the whole plane range)
  int pc_i[kFPosPerThread], pc_j[kFPosPerThread];
  for (int r = 0; r < kFPosPerThread; ++r) col_ij(clo + (int)threadIdx.x + r * kMarchThreads, pc_i[r], pc_j[r]);
  auto positions = [&](int k) {
    double* P = sm.pos + (size_t)(k & 1) * 3 * slot_len;
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

  // ---- anchor column of this thread: every column (faces included) of the
  // band's diagonals [a_lo, d1) -- at most kMarchThreads (fem bands, setup.cu)
  const int an_lo = (int)col_idx(a_lo, 0) - clo;
  const int an_n = (int)col_idx(0, b.d1 - 1) + 1 - clo - an_lo;
  int an_lim = -1, an_o[8];
  uint8_t an_tm = 0;
  auto anchor_setup = [&](int col, int& lim, uint8_t& tm, int (&o)[8]) {
    int i0, j0;
    col_ij(col, i0, j0);
    lim = N - 1 - (i0 + j0);
    tm = 0x3f;
    if (i0 == 0) tm &= (1 << 0) | (1 << 1) | (1 << 4);  // X before Y
    if (j0 == 0) tm &= (1 << 0) | (1 << 2) | (1 << 3);  // Y before Z
    if (i0 + j0 == N - 1) tm &= (1 << 3) | (1 << 4) | (1 << 5);  // corners 1, 3 lie on diagonal N
    const int di[8] = {0, 1, -1, 0, 0, 1, -1, 0};
    const int dj[8] = {0, 0, 1, 1, -1, -1, 0, 0};
#pragma unroll
    for (int c = 0; c < 8; ++c) o[c] = ring_off(i0 + di[c], j0 + dj[c], clo, slot_len);
  };
  if ((int)threadIdx.x < an_n) anchor_setup(clo + an_lo + (int)threadIdx.x, an_lim, an_tm, an_o);
  // ---- output nodes: the band's interior columns, and the halo diagonals' nodes
  const Column q = make_column(b.d0 == 2 ? bands[bi] : b, N);  // offsets relative to the band's own c_lo
  const int qshift = bands[bi].c_lo - clo;                       // -> relative to this kernel's clo
  double* const optr = out + T * S + q.c;
  const double* const fptr = f + T * S + q.c;
  // halo nodes: interior columns of diagonal d0-1 (sums of this band's anchors on
  // d0, top corners) and of diagonal d1 (anchors on d1-1, bottom corners)
  const int nh_lo = (b.d0 - 1 >= 2 && bi > 0) ? b.d0 - 2 : 0;        // (i,j) i,j >= 1 on diagonal d0-1
  const int nh_hi = (b.d1 <= N - 2 && bi < n_bands - 1) ? b.d1 - 1 : 0;  // on diagonal d1
  // corner sums sum_b K_ab u_b of the valid Kuhn tets of one cube, corners from
  // shared memory (P0/U0: plane k0, P1/U1: plane k0+1)
  auto cube = [&](const int (&o)[8], uint8_t tm, const double* P0, const double* P1, const double* U0,
                  const double* U1, double (&yc)[8]) {
    double P[8][3], U[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double* pp = c < 4 ? P0 : P1;
      P[c][0] = pp[o[c]];
      P[c][1] = pp[slot_len + o[c]];
      P[c][2] = pp[2 * slot_len + o[c]];
      U[c] = (c < 4 ? U0 : U1)[o[c]];
    }
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      if (!((tm >> t) & 1)) continue;
      const int v0 = kKuhn[t][0], v1 = kKuhn[t][1], v2 = kKuhn[t][2], v3 = kKuhn[t][3];
      double e1[3], e2[3], e3[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        e1[d] = P[v1][d] - P[v0][d];
        e2[d] = P[v2][d] - P[v0][d];
        e3[d] = P[v3][d] - P[v0][d];
      }
      const double c1[3] = {e2[1] * e3[2] - e2[2] * e3[1], e2[2] * e3[0] - e2[0] * e3[2],
                            e2[0] * e3[1] - e2[1] * e3[0]};
      const double c2[3] = {e3[1] * e1[2] - e3[2] * e1[1], e3[2] * e1[0] - e3[0] * e1[2],
                            e3[0] * e1[1] - e3[1] * e1[0]};
      const double c3[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                            e1[0] * e2[1] - e1[1] * e2[0]};
      const double det = e1[0] * c1[0] + e1[1] * c1[1] + e1[2] * c1[2];
      const double du1 = U[v1] - U[v0], du2 = U[v2] - U[v0], du3 = U[v3] - U[v0];
      double G[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) G[d] = fma(c1[d], du1, fma(c2[d], du2, c3[d] * du3));
      const double s = rcp_nr(6.0 * fabs(det));  // ~1 ulp (R16)
      const double y1 = fma(c1[0], G[0], fma(c1[1], G[1], c1[2] * G[2])) * s;
      const double y2 = fma(c2[0], G[0], fma(c2[1], G[1], c2[2] * G[2])) * s;
      const double y3 = fma(c3[0], G[0], fma(c3[1], G[1], c3[2] * G[2])) * s;
      yc[v1] += y1;
      yc[v2] += y2;
      yc[v3] += y3;
      yc[v0] -= (y1 + y2) + y3;  // rows of K_T sum to zero
    }
  };
  auto slab_sums = [&](int k0) {
    double* const topb = sm.top + (size_t)(k0 & 1) * 4 * slot_len;
    const double* P0 = sm.pos + (size_t)(k0 & 1) * 3 * slot_len;
    const double* P1 = sm.pos + (size_t)((k0 + 1) & 1) * 3 * slot_len;
    const double* U0 = sm.ring + (k0 % kEwRing) * slot_len + ((sm.po[k0] + clo) & 1);
    const double* U1 = sm.ring + ((k0 + 1) % kEwRing) * slot_len + ((sm.po[k0 + 1] + clo) & 1);
    if ((int)threadIdx.x < an_n) {
      const int oa = an_lo + (int)threadIdx.x;
      double yc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) yc[c] = 0.0;
      if (k0 <= an_lim) cube(an_o, an_tm, P0, P1, U0, U1, yc);
#pragma unroll
      for (int c = 0; c < 4; ++c) sm.bot[c * slot_len + oa] = yc[c];
#pragma unroll
      for (int c = 0; c < 4; ++c) topb[c * slot_len + oa] = yc[4 + c];
    }
    // the last band also owns the cubes anchored on diagonal N-1 (slab 0 only):
    // of their tets only YZX, ZXY, ZYX reach interior nodes (corners 4, 6 on
    // diagonal N-2, plane 1); corners 1, 3 would lie on diagonal N
    if (k0 == 0 && bi == n_bands - 1) {
      for (int x = threadIdx.x; x < N; x += blockDim.x) {
        int lim, o[8];
        uint8_t tm;
        const int col = (int)col_idx(x, N - 1 - x);
        anchor_setup(col, lim, tm, o);
        double yc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) yc[c] = 0.0;
        cube(o, tm, P0, P1, U0, U1, yc);
        topb[col - clo] = yc[4];
        topb[2 * slot_len + col - clo] = yc[6];
      }
    }
  };

  positions(0);
  for (int k0 = 0; k0 <= b.kmax + 1; ++k0) {
    if (k0 + 1 <= N) positions(k0 + 1);
    if (k0 + 1 <= last_plane) mbar_wait(&sm.bars[(k0 + 1) % kEwRing], ((k0 + 1) / kEwRing) & 1);
    if (k0 == 0) mbar_wait(&sm.bars[0], 0);
    __syncthreads();  // positions k0+1 visible; every thread is done with slab k0-1 and its sums
    // plane k0-1's slot is free: refill
    if (next_issue <= last_plane && next_issue <= k0 + kEwRing - 1) {
      issue_planes<kEwRing>(ub, sm.po, next_issue, min(k0 + kEwRing - 1, last_plane), b, sm.ring, slot_len,
                            sm.bars);
      next_issue = min(k0 + kEwRing - 1, last_plane) + 1;
    }
    if (k0 <= b.kmax) slab_sums(k0);
    __syncthreads();  // slab k0 sums visible
    const int k = k0;
    if (k < 1) continue;
    const double* tp = sm.top + (size_t)((k - 1) & 1) * 4 * slot_len;
    if (q.active && k <= q.len) {
      const int oc = q.o_c + qshift, ow = q.o_w + qshift, ose = q.o_se + qshift, os = q.o_s + qshift;
      const int on = q.o_n + qshift, onw = q.o_nw + qshift, oe = q.o_e + qshift;
      const double yb = (sm.bot[oc] + sm.bot[slot_len + ow]) + (sm.bot[2 * slot_len + ose] + sm.bot[3 * slot_len + os]);
      const double yt = (tp[on] + tp[slot_len + onw]) + (tp[2 * slot_len + oe] + tp[3 * slot_len + oc]);
      const double y = yb + yt;
      optr[sm.po[k]] = (MODE == kModeResid) ? __ldg(fptr + sm.po[k]) - y : y;
    }
    // halo nodes (their owners add these in k_fem_ew_fixup)
    for (int x = threadIdx.x; x < nh_lo + nh_hi; x += blockDim.x) {
      const bool lo = x < nh_lo;
      const int d = lo ? b.d0 - 1 : b.d1;
      const int j = lo ? x + 1 : x - nh_lo + 1;
      const int i = d - j;
      if (k > N - 1 - d) continue;
      const int64_t slot = T * S + sm.po[k] + col_idx(i, j);
      if (lo) {  // top corners 4 (anchor (i, j+1)) and 6 (anchor (i+1, j)) of slab k-1
        s_hi[slot] = tp[(int)col_idx(i, j + 1) - clo] + tp[2 * slot_len + (int)col_idx(i + 1, j) - clo];
      } else {   // bottom corners 1 (anchor (i-1, j)) and 3 (anchor (i, j-1)) of slab k
        s_lo[slot] = sm.bot[slot_len + (int)col_idx(i - 1, j) - clo] + sm.bot[3 * slot_len + (int)col_idx(i, j - 1) - clo];
      }
    }
  }
}

// out += (apply) / -= (residual) the halo sums of the neighbouring bands:
// nodes on a band's first diagonal receive s_lo (written by the band below),
// nodes on its last diagonal s_hi (written by the band above).
template <int MODE>
__global__ void k_fem_ew_fixup(int N, int64_t S, const Band* __restrict__ bands, int n_bands,
                               const double* __restrict__ s_lo, const double* __restrict__ s_hi,
                               double* __restrict__ out) {
  const int64_t T = blockIdx.y;
  const int bi = blockIdx.z;
  const Band b = bands[bi];
  const bool has_lo = bi > 0, has_hi = bi < n_bands - 1;
  // (column on diagonal d0 or d1-1, plane) pairs, flattened
  const int nlo = has_lo ? b.d0 - 1 : 0;
  const int nhi = (has_hi && b.d1 - 1 != b.d0) ? b.d1 - 2 : 0;
  const int ncol = nlo + nhi;
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= (int64_t)ncol * (N - 1)) return;
  const int cidx = (int)(x % ncol);
  const int k = 1 + (int)(x / ncol);
  const int d = cidx < nlo ? b.d0 : b.d1 - 1;
  const int j = 1 + (cidx < nlo ? cidx : cidx - nlo);
  const int i = d - j;
  if (k > N - 1 - d) return;
  const int64_t slot = T * S + plane_off(N, k) + col_idx(i, j);
  double s = 0.0;
  if (has_lo && d == b.d0) s += s_lo[slot];
  if (has_hi && d == b.d1 - 1) s += s_hi[slot];
  out[slot] = (MODE == kModeResid) ? out[slot] - s : out[slot] + s;
}

}  // namespace hhg
