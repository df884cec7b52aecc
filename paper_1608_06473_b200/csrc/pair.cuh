// Plane-PAIR pipelined persistent march: the production volume kernel for the
// surrogate / constant-stencil apply and residual (y = L~u, r = f - L~u on
// volume nodes).
//
// Same geometry and static item schedule as pmarch.cuh (item = (macro, band of
// diagonals), thread = lattice column (i,j) marching in k), but the pipeline
// unit is a PAIR of planes (2p, 2p+1): one ring slot, one full and one empty
// mbarrier, two 1-D TMA bulk copies completing on the same barrier.  A thread
// computes the two nodes k, k+1 (k odd) of its column per step, so per node
// the pipeline costs half a wait, half a release and 1/16 of an issue.  The
// inner step is branch-free (inactive lanes and finished columns compute on
// in-range shared memory and only their stores are predicated off), addresses
// are carried incrementally, and the 2-step register rotation of the u window
// needs no moves.  Per node: 45 DFMA (15 weights by Horner in k, 2 DFMA each,
// + 15 for the stencil; PAPER.md:1135 counts the same work as "29+15q"), 7
// shared loads of u, 7.5 broadcast loads of the per-macro k^2 coefficients.
#pragma once
#include "pmarch.cuh"

namespace hhg {

constexpr int kQThreads = 256;
constexpr int kQWarps = kQThreads / 32;
constexpr int kQIQ = 4;  // coefficient slots
constexpr int kQQ = 16;  // item queue entries
constexpr int kQFill = 8;  // items fetched ahead of warp 0

template <int R>  // R = ring slots (pairs)
struct QSmem {
  double* ring;     // [R][2][slot_len]
  double* coef;     // [kQIQ][160]
  uint64_t* full;   // [R]
  uint64_t* empty;  // [R]
  uint64_t* ifull;  // [kQIQ]
  uint64_t* iempty; // [kQIQ]
  int* po;          // [N+2]
  int* bk;          // [n_bands] pairs per item
  int64_t total;    // items of this launch
  __device__ QSmem(double* smem, int slot_len, int N, int n_bands) {
    ring = smem;
    coef = ring + (size_t)R * 2 * slot_len;
    full = (uint64_t*)(coef + kQIQ * 160);
    empty = full + R;
    ifull = empty + R;
    iempty = ifull + kQIQ;
    po = (int*)(iempty + kQIQ);
    bk = po + (N + 2);
  }
};

__host__ __device__ inline size_t pair_smem_bytes(int R, int slot_len, int N, int n_bands) {
  return (size_t)R * 2 * slot_len * 8 + kQIQ * 160 * 8 + (2 * R + 2 * kQIQ) * 8 + (size_t)(N + 2) * 4 +
         (size_t)n_bands * 4 + (kQQ + 1) * 4;
}

// Dynamic item queue: items are handed out in (macro, band) order by a global
// atomic counter, so the bands of a macro run concurrently on different CTAs
// and share their halo diagonals in L2.  Warp 0 (lane 0) keeps kQFill items
// fetched ahead of its own position; every warp reads item n from the queue.
// Returns the item id, -1 past the end, -2 if not fetched yet.
// Static boustrophedon schedule: item n of CTA c is n*G + c for even n and
// n*G + G-1-c for odd n (G = grid).  At any time the CTAs work on a window of
// G consecutive (macro, band) items, so the bands of a macro run concurrently
// and share their halo diagonals in L2; alternating the direction balances the
// band lengths (max/mean work 1.06 on the 480-macro L7 shell).  The item id
// depends only on blockIdx and the loop counter, so the macro index T is
// uniform and the per-macro k^2 coefficients come from constant memory.
template <int R>
__device__ __forceinline__ int queue_item(const QSmem<R>& sm, int n) {
  const int G = (int)gridDim.x, cta = (int)blockIdx.x;
  const int64_t it = (int64_t)n * G + ((n & 1) ? G - 1 - cta : cta);
  return it < sm.total ? (int)it : -1;
}

// Issue cursor of one warp (lane 0): the next pair this warp owns (g = warp mod 8).
// c.n = item index in this CTA's sequence; c.np = 0 while item c.n is unknown.
template <int R>
__device__ __forceinline__ bool qcursor_load(PCursor& c, const PArgs& a, const QSmem<R>& sm) {
  const int it = queue_item(sm, c.n);
  if (it == -2) return false;
  if (it < 0) {
    c.np = 1 << 30;
    c.T = -1;
    return true;
  }
  c.T = it / a.n_bands;
  c.b = it - c.T * a.n_bands;
  c.np = sm.bk[c.b];
  return true;
}

// Move the cursor forward to pair g + pending (stops early if an item is not known yet).
template <int R>
__device__ __forceinline__ void qcursor_settle(PCursor& c, const PArgs& a, const QSmem<R>& sm) {
  for (;;) {
    if (c.np == 0 && !qcursor_load(c, a, sm)) return;
    if (c.T < 0 || c.p < c.np) return;
    c.p -= c.np;
    ++c.n;
    c.np = 0;
  }
}

template <int OP, int R>
__device__ __forceinline__ void qtry_issue(PCursor& c, const PArgs& a, QSmem<R>& sm, int limit) {
  for (;;) {
    qcursor_settle(c, a, sm);
    if (c.np == 0 || c.T < 0 || c.g >= limit) return;
    const int slot = c.g & (R - 1);
    if (c.g >= R && !mbar_test(&sm.empty[slot], ((c.g / R) - 1) & 1)) return;
    if (c.p == 0) {  // first pair of item n: also its coefficients
      const int e = c.n & (kQIQ - 1);
      if (c.n >= kQIQ && !mbar_test(&sm.iempty[e], ((c.n / kQIQ) - 1) & 1)) return;
      if (OP == HHG_OP_SURROGATE) {
        mbar_expect_tx(&sm.ifull[e], 150 * 8);
        tma_load_1d(sm.coef + e * 160, a.coef10 + (int64_t)c.T * 150, 150 * 8, &sm.ifull[e]);
      } else {
        mbar_arrive(&sm.ifull[e]);
      }
    }
    const Band& b = a.bands[c.b];
    const int p0 = 2 * c.p;
    const int g0 = sm.po[p0] + b.c_lo, g1 = sm.po[p0 + 1] + b.c_lo;
    const int a0 = g0 & ~1, a1 = g1 & ~1;
    const uint32_t n0 = (uint32_t)((((g0 + b.ncols + 1) & ~1) - a0) * 8);
    const uint32_t n1 = (uint32_t)((((g1 + b.ncols + 1) & ~1) - a1) * 8);
    double* dst = sm.ring + (size_t)slot * 2 * a.slot_len;
    const double* src = a.u + (int64_t)c.T * a.S;
    mbar_expect_tx(&sm.full[slot], n0 + n1);
    tma_load_1d(dst, src + a0, n0, &sm.full[slot]);
    tma_load_1d(dst + a.slot_len, src + a1, n1, &sm.full[slot]);
    c.g += kQWarps;
    c.p += kQWarps;
  }
}

template <int OP, int R>
__device__ __forceinline__ void qwait(uint64_t* bar, uint32_t parity, PCursor& c, const PArgs& a, QSmem<R>& sm,
                                      int limit) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    if (lane == 0 && c.g < limit) qtry_issue<OP, R>(c, a, sm, limit);
    __syncwarp();
    if (__all_sync(0xffffffffu, mbar_try(bar, parity))) break;
  }
}

// Column of this thread in band b; inactive lanes get a valid column of the
// band (their stores are predicated off) so the inner loop is branch-free.
struct QCol {
  bool active;
  int i, j, len, c;
  int o_c, o_e, o_n, o_nw, o_w, o_s, o_se;
};

__device__ __forceinline__ QCol qcolumn(const Band& b, int N) {
  QCol q;
  int t = threadIdx.x, d = b.d0;
  q.active = t < b.ncolumns;
  if (!q.active) t = 0;
  while (t >= d - 1) { t -= d - 1; ++d; }
  const int j = t + 1, i = d - j;
  q.i = i;
  q.j = j;
  q.len = q.active ? N - 1 - d : 0;
  q.c = (int)col_idx(i, j);
  const int lo = b.c_lo;
  q.o_c = q.c - lo;
  q.o_e = (int)col_idx(i + 1, j) - lo;
  q.o_n = (int)col_idx(i, j + 1) - lo;
  q.o_nw = (int)col_idx(i - 1, j + 1) - lo;
  q.o_w = (int)col_idx(i - 1, j) - lo;
  q.o_s = (int)col_idx(i, j - 1) - lo;
  q.o_se = (int)col_idx(i + 1, j - 1) - lo;
  return q;
}

template <int OP, int MODE, int R>
__global__ void __launch_bounds__(kQThreads, 2)
    k_vol_pair(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
               const double* __restrict__ coef10, const double* __restrict__ cons, const double* __restrict__ u,
               const double* __restrict__ f, double* __restrict__ out, int64_t ntl, int T0) {
  extern __shared__ __align__(16) double smem[];
  constexpr int kAhead = R - 3;  // pairs a warp issues ahead of its own position
  QSmem<R> sm(smem, slot_len, N, n_bands);
  sm.total = ntl * n_bands;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const PArgs a{N, S, bands, n_bands, slot_len, coef10 + (int64_t)T0 * 150, u + (int64_t)T0 * S, nullptr, 0};
  if (threadIdx.x == 0) {
    for (int s = 0; s < R; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kQWarps);
    }
    for (int s = 0; s < kQIQ; ++s) {
      mbar_init(&sm.ifull[s], 1);
      mbar_init(&sm.iempty[s], kQWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) sm.po[p] = (int)plane_off(N, p);
  for (int b = threadIdx.x; b < n_bands; b += blockDim.x) sm.bk[b] = (bands[b].kmax + 3) / 2;
  __syncthreads();

  PCursor cur;
  cur.g = warp;  // this warp issues pairs g = warp, warp + 8, ...
  cur.n = 0;
  cur.p = warp;
  cur.np = 0;
  cur.T = 0;
  cur.b = 0;
  if (lane == 0) qtry_issue<OP, R>(cur, a, sm, kAhead);

  int gp = 0;  // global pair number of pair 0 of the current item
  for (int n = 0;; ++n) {
    const int it = queue_item(sm, n);
    if (it < 0) break;
    const int Tl = it / n_bands;  // macro within this launch chunk (uniform)
    const int T = T0 + Tl;
    const Band b = bands[it - T * n_bands];
    const int e = n & (kQIQ - 1);
    qwait<OP, R>(&sm.ifull[e], (n / kQIQ) & 1, cur, a, sm, gp + kAhead);
    const QCol q = qcolumn(b, N);
    const double* cf = sm.coef + e * 160;
    double A[15], B[15];
    pcolumn_coeffs<OP>(cf, cons, T, q.i, q.j, A, B);
    const int clo = b.c_lo;
    const int kmax = b.kmax;
    const int npairs = (kmax + 3) / 2;

    // shared-memory base of plane p (within its pair slot), incl. the 16-byte alignment shift
    auto pbase = [&](int p, int po_p) -> const double* {
      const int g = gp + (p >> 1);
      return sm.ring + ((size_t)(g & (R - 1)) * 2 + (p & 1)) * slot_len + ((po_p + clo) & 1);
    };
    auto wait_pair = [&](int pp) {
      const int g = gp + pp;
      qwait<OP, R>(&sm.full[g & (R - 1)], (g / R) & 1, cur, a, sm, g + kAhead);
    };
    auto release_pair = [&](int pp) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[(gp + pp) & (R - 1)]);
    };

    wait_pair(0);
    int po_km1 = sm.po[0], po_k = sm.po[1];
    double bc, be, bn, bnw, mc, mw, ms, mse;
    {
      const double* P0 = pbase(0, po_km1);
      const double* P1 = pbase(1, po_k);
      bc = P0[q.o_c]; be = P0[q.o_e]; bn = P0[q.o_n]; bnw = P0[q.o_nw];
      mc = P1[q.o_c]; mw = P1[q.o_w]; ms = P1[q.o_s]; mse = P1[q.o_se];
    }
    double* optr = out + (int64_t)T * S + q.c;
    const double* fptr = f + (int64_t)T * S + q.c;
    for (int k = 1; k <= kmax; k += 2) {
      wait_pair((k + 1) >> 1);  // planes k+1, k+2
      const int po_k1 = sm.po[k + 1], po_k2 = sm.po[k + 2];
      double fa = 0.0, fb = 0.0;
      if (MODE == kModeResid) {
        if (k <= q.len) fa = __ldg(fptr + po_k);
        if (k + 1 <= q.len) fb = __ldg(fptr + po_k1);
      }
      const double* Pk = pbase(k, po_k);
      const double* Pk1 = pbase(k + 1, po_k1);
      const double* Pk2 = pbase(k + 2, po_k2);
      const double me = Pk[q.o_e], mn = Pk[q.o_n], mnw = Pk[q.o_nw];
      const double tc = Pk1[q.o_c], tw = Pk1[q.o_w], ts = Pk1[q.o_s], tse = Pk1[q.o_se];
      const double me2 = Pk1[q.o_e], mn2 = Pk1[q.o_n], mnw2 = Pk1[q.o_nw];
      const double tc2 = Pk2[q.o_c], tw2 = Pk2[q.o_w], ts2 = Pk2[q.o_s], tse2 = Pk2[q.o_se];
      const double ua[15] = {bc, be, bn, bnw, ms, mse, mw, mc, me, mnw, mn, tse, ts, tw, tc};
      const double ub[15] = {mc, me, mn, mnw, ts, tse, tw, tc, me2, mnw2, mn2, tse2, ts2, tw2, tc2};
      double ra, rb;
      pnode2<OP>(A, B, g_cC + Tl * 15, (double)k, ua, ub, ra, rb);
      if (k <= q.len) optr[po_k] = (MODE == kModeResid) ? fa - ra : ra;
      if (k + 1 <= q.len) optr[po_k1] = (MODE == kModeResid) ? fb - rb : rb;
      bc = tc; be = me2; bn = mn2; bnw = mnw2;
      mc = tc2; mw = tw2; ms = ts2; mse = tse2;
      po_k = po_k2;
      release_pair((k - 1) >> 1);  // planes k-1, k
    }
    release_pair(npairs - 1);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.iempty[e]);
    gp += npairs;
  }
}

}  // namespace hhg
