// Persistent column-march kernel for the surrogate apply / residual (y = L~u,
// r = f - L~u on volume nodes) -- the "v3" volume
// path.
//
// Geometry is the one of march.cuh: a work item is (macro T, band b of
// diagonals), one thread = one interior lattice column (i,j) marching in k,
// planes of the band brought into shared memory by 1-D TMA bulk copies.
// What changes is the execution model:
//   * persistent CTAs (grid = #SM x occupancy), each with a STATIC list of
//     items (host-side greedy balance in macro-major order, so neighbouring
//     bands of a macro run at the same time and share their halo diagonals in
//     L2).  The CTA's plane stream is the concatenation of its items' planes,
//     numbered g = 0, 1, 2, ...; the TMA ring runs continuously ACROSS items
//     (the next item's first planes and coefficients land while the current
//     item drains);
//   * ring slots are recycled through per-slot "empty" mbarriers (one arrive
//     per warp) instead of CTA-wide __syncthreads: warps drift freely;
//   * the producer role is distributed: plane g is issued by warp g mod 8
//     (lane 0), non-blockingly, when that warp passes within R - 5 planes of
//     it -- every warp computes, none is a serial bottleneck;
//   * NPS nodes per thread step (2: the per-macro k^2 coefficient is read once
//     for both nodes and two independent FMA chains interleave).
// Per node: 15 weights by Horner in k, s_w(k) = A_w + k (B_w + k C_w) with
// A_w, B_w per column (registers) and C_w = c_002 per macro (shared memory),
// 2 DFMA per weight + 15 DFMA for the stencil = 45 DFMA (Table flops "29+15q",
// PAPER.md:1135, counts the same work).
#pragma once
#include <algorithm>
#include <vector>

#include "hhg_internal.h"
#include "march.cuh"

namespace hhg {

constexpr int kPThreads = 256;
constexpr int kPWarps = kPThreads / 32;
constexpr int kPIQ = 4;              // coefficient slots (items in flight)
// R = ring slots (template parameter); a warp issues its planes up to R - 5
// planes ahead of itself.

template <int R>
struct PSmem {
  double* ring;     // [R][slot_len]
  double* coef;     // [kPIQ][160]
  uint64_t* full;   // [R]
  uint64_t* empty;  // [R]
  uint64_t* ifull;  // [kPIQ]
  uint64_t* iempty; // [kPIQ]
  int* po;          // [N+2]
  int* bk;          // [n_bands] kmax + 2 (planes per item)
  __device__ PSmem(double* smem, int slot_len, int N) {
    ring = smem;
    coef = ring + (size_t)R * slot_len;
    full = (uint64_t*)(coef + kPIQ * 160);
    empty = full + R;
    ifull = empty + R;
    iempty = ifull + kPIQ;
    po = (int*)(iempty + kPIQ);
    bk = po + (N + 2);
  }
};

__host__ __device__ inline size_t pmarch_smem_bytes(int R, int slot_len, int N, int n_bands) {
  return (size_t)R * slot_len * 8 + kPIQ * 160 * 8 + (2 * R + 2 * kPIQ) * 8 + (size_t)(N + 2) * 4 +
         (size_t)n_bands * 4;
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}


// Issue cursor of one warp (lane 0's registers): the next plane this warp owns.
struct PCursor {
  int g;      // global plane number (g mod kPWarps == warp)
  int n;      // item index in this CTA's list
  int p;      // plane within item n
  int np;     // planes of item n
  int T, b;   // macro, band of item n
};

struct PArgs {
  int N;
  int64_t S;
  const Band* bands;
  int n_bands;
  int slot_len;
  const double* coef10;
  const double* u;
  const int* items;  // this CTA's item list
  int n_items;
};

template <int R>
__device__ __forceinline__ void cursor_load_item(PCursor& c, const PArgs& a, const PSmem<R>& sm) {
  if (c.n < a.n_items) {
    const int it = __ldg(a.items + c.n);
    c.T = it / a.n_bands;
    c.b = it - c.T * a.n_bands;
    c.np = sm.bk[c.b];
  } else {
    c.np = 1 << 30;
  }
}

// Advance the cursor by `by` planes.
template <int R>
__device__ __forceinline__ void cursor_advance(PCursor& c, const PArgs& a, const PSmem<R>& sm, int by) {
  c.g += by;
  c.p += by;
  while (c.n < a.n_items && c.p >= c.np) {
    c.p -= c.np;
    ++c.n;
    cursor_load_item(c, a, sm);
  }
}

// Issue this warp's planes with g < limit as far as ring slots are free (lane 0).
template <int OP, int R>
__device__ __forceinline__ void try_issue(PCursor& c, const PArgs& a, PSmem<R>& sm, int limit) {
  while (c.g < limit && c.n < a.n_items) {
    const int slot = c.g % R;
    if (c.g >= R && !mbar_test(&sm.empty[slot], ((c.g / R) - 1) & 1)) return;
    if (c.p == 0) {  // first plane of item n: also bring its coefficients
      const int e = c.n % kPIQ;
      if (c.n >= kPIQ && !mbar_test(&sm.iempty[e], ((c.n / kPIQ) - 1) & 1)) return;
      if (OP == HHG_OP_SURROGATE) {
        mbar_expect_tx(&sm.ifull[e], 150 * 8);
        tma_load_1d(sm.coef + e * 160, a.coef10 + (int64_t)c.T * 150, 150 * 8, &sm.ifull[e]);
      } else {
        mbar_arrive(&sm.ifull[e]);
      }
    }
    const Band& b = a.bands[c.b];
    const int g0 = sm.po[c.p] + b.c_lo;
    const int a0 = g0 & ~1;
    const int a1 = (g0 + b.ncols + 1) & ~1;
    const uint32_t bytes = (uint32_t)((a1 - a0) * 8);
    mbar_expect_tx(&sm.full[slot], bytes);
    tma_load_1d(sm.ring + (size_t)slot * a.slot_len, a.u + (int64_t)c.T * a.S + a0, bytes, &sm.full[slot]);
    cursor_advance(c, a, sm, kPWarps);
  }
}

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Wait for phase `parity` of `bar`, issuing this warp's due planes (g < limit)
// first and again whenever the (hardware-suspended) try_wait times out, so a
// warp never sleeps on a plane while it still owes the ring a plane.
template <int OP, int R>
__device__ __forceinline__ void pwait(uint64_t* bar, uint32_t parity, PCursor& c, const PArgs& a, PSmem<R>& sm,
                                      int limit) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    if (lane == 0 && c.g < limit) try_issue<OP, R>(c, a, sm, limit);
    __syncwarp();
    if (__all_sync(0xffffffffu, mbar_try(bar, parity))) break;
  }
}

template <int OP>
__device__ __forceinline__ void pcolumn_coeffs(const double* cf, const double* __restrict__ cons, int T, int i, int j,
                                               double (&A)[15], double (&B)[15]) {
  if (OP == HHG_OP_SURROGATE) {
    const double di = (double)i, dj = (double)j;
#pragma unroll
    for (int w = 0; w < 15; ++w) {
      const double* q = cf + w * 10;  // (000)(100)(010)(001)(200)(110)(101)(020)(011)(002)
      A[w] = q[0] + di * (q[1] + di * q[4] + dj * q[5]) + dj * (q[2] + dj * q[7]);
      B[w] = q[3] + di * q[6] + dj * q[8];
    }
  } else {
#pragma unroll
    for (int w = 0; w < 15; ++w) {
      A[w] = __ldg(cons + (int64_t)T * 15 + w);
      B[w] = 0.0;
    }
  }
}

// y_I = sum_w s_w(k) u_w for one node (uu in direction order, HHG_DIRS_INIT);
// C_w read from shared memory (broadcast).
template <int OP>
__device__ __forceinline__ double pnode(const double (&A)[15], const double (&B)[15], const double* cf, double kd,
                                        const double (&uu)[15]) {
  double acc[3] = {0.0, 0.0, 0.0};
  if (OP == HHG_OP_SURROGATE) {
#pragma unroll
    for (int w = 0; w < 15; ++w) {
      const double s = fma(fma(cf[w * 10 + 9], kd, B[w]), kd, A[w]);
      acc[w % 3] = fma(s, uu[w], acc[w % 3]);
    }
  } else {
#pragma unroll
    for (int w = 0; w < 15; ++w) acc[w % 3] = fma(A[w], uu[w], acc[w % 3]);
  }
  return (acc[0] + acc[1]) + acc[2];
}

// Two nodes k, k+1 of one column (cf = the 15 per-macro k^2 coefficients C_w).
// The weight polynomial is expanded instead
// of evaluated by Horner per weight:
//   sum_w s_w(k) u_w = sum_w A_w u_w + k sum_w B_w u_w + k^2 sum_w C_w u_w,
// six independent accumulation chains (three per node) instead of fifteen
// dependent 3-deep Horner chains, so the fp64 pipe is fed without extra
// registers; each C_w (per macro, shared memory broadcast) is read once for
// both nodes.  Same 45 DFMA per node (+2 to combine).
template <int OP>
__device__ __forceinline__ void pnode2(const double (&A)[15], const double (&B)[15], const double* cf, double kd,
                                       const double (&ua)[15], const double (&ub)[15], double& ra, double& rb) {
  if (OP == HHG_OP_SURROGATE) {
    double xa = 0.0, ya = 0.0, za = 0.0, xb = 0.0, yb = 0.0, zb = 0.0;
#pragma unroll
    for (int w = 0; w < 15; ++w) {
      const double c = cf[w];
      xa = fma(A[w], ua[w], xa);
      xb = fma(A[w], ub[w], xb);
      ya = fma(B[w], ua[w], ya);
      yb = fma(B[w], ub[w], yb);
      za = fma(c, ua[w], za);
      zb = fma(c, ub[w], zb);
    }
    const double kd1 = kd + 1.0;
    ra = fma(fma(za, kd, ya), kd, xa);
    rb = fma(fma(zb, kd1, yb), kd1, xb);
  } else {
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int w = 0; w < 15; ++w) {
      if (w & 1) {
        a1 = fma(A[w], ua[w], a1);
        b1 = fma(A[w], ub[w], b1);
      } else {
        a0 = fma(A[w], ua[w], a0);
        b0 = fma(A[w], ub[w], b0);
      }
    }
    ra = a0 + a1;
    rb = b0 + b1;
  }
}

// NPS = nodes per thread per step (1 or 2).  items/item_off: static schedule.
template <int OP, int MODE, int NPS, int R>
__global__ void __launch_bounds__(kPThreads, 2)
    k_vol_pmarch(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
                 const double* __restrict__ coef10, const double* __restrict__ cons, const double* __restrict__ u,
                 const double* __restrict__ f, double* __restrict__ out, const int* __restrict__ items,
                 const int* __restrict__ item_off) {
  extern __shared__ __align__(16) double smem[];
  constexpr int kAhead = R - 5;
  PSmem<R> sm(smem, slot_len, N);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int i0 = item_off[blockIdx.x];
  const PArgs a{N, S, bands, n_bands, slot_len, coef10, u, items + i0, item_off[blockIdx.x + 1] - i0};
  if (threadIdx.x == 0) {
    for (int s = 0; s < R; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kPWarps);
    }
    for (int s = 0; s < kPIQ; ++s) {
      mbar_init(&sm.ifull[s], 1);
      mbar_init(&sm.iempty[s], kPWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) sm.po[p] = (int)plane_off(N, p);
  for (int b = threadIdx.x; b < n_bands; b += blockDim.x) sm.bk[b] = bands[b].kmax + 2;
  __syncthreads();

  // this warp's issue cursor starts at plane g = warp
  PCursor cur;
  cur.g = 0;
  cur.n = 0;
  cur.p = 0;
  cur.np = 0;
  cur.T = 0;
  cur.b = 0;
  if (lane == 0) {
    cursor_load_item(cur, a, sm);
    cursor_advance(cur, a, sm, warp);
    try_issue<OP, R>(cur, a, sm, kAhead);
  }

  int gp = 0;  // global plane number of plane 0 of the current item
  for (int n = 0; n < a.n_items; ++n) {
    const int it = __ldg(a.items + n);
    const int T = it / n_bands;
    const Band b = bands[it - T * n_bands];
    const int e = n % kPIQ;
    pwait<OP, R>(&sm.ifull[e], (n / kPIQ) & 1, cur, a, sm, gp + kAhead);
    const Column q = make_column(b, N);
    const double* cf = sm.coef + e * 160;
    double A[15], B[15];
    pcolumn_coeffs<OP>(cf, cons, T, q.i, q.j, A, B);

    const int clo = b.c_lo;
    auto sptr = [&](int p) -> const double* {
      const int g = gp + p;
      return sm.ring + (size_t)(g % R) * slot_len + ((sm.po[p] + clo) & 1);
    };
    auto wait_plane = [&](int p) {
      const int g = gp + p;
      pwait<OP, R>(&sm.full[g % R], (g / R) & 1, cur, a, sm, g + kAhead);
    };
    auto release = [&](int p) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[(gp + p) % R]);
    };

    wait_plane(0);
    wait_plane(1);
    double bc, be, bn, bnw, mc, mw, ms, mse;
    {
      const double* P0 = sptr(0);
      const double* P1 = sptr(1);
      bc = P0[q.o_c]; be = P0[q.o_e]; bn = P0[q.o_n]; bnw = P0[q.o_nw];
      mc = P1[q.o_c]; mw = P1[q.o_w]; ms = P1[q.o_s]; mse = P1[q.o_se];
    }
    const int64_t base = (int64_t)T * S + q.c;
    double* const optr = out + base;
    const double* const fptr = f + base;
    const int kmax = b.kmax;
    if (NPS == 1) {
      double fn = 0.0;
      if (MODE == kModeResid && q.active && 1 <= q.len) fn = __ldg(fptr + sm.po[1]);
      for (int k = 1; k <= kmax; ++k) {
        wait_plane(k + 1);
        const double fv = fn;
        if (MODE == kModeResid && q.active && k + 1 <= q.len) fn = __ldg(fptr + sm.po[k + 1]);
        if (q.active && k <= q.len) {
          const double* Pk = sptr(k);
          const double* Pk1 = sptr(k + 1);
          const double me = Pk[q.o_e], mn = Pk[q.o_n], mnw = Pk[q.o_nw];
          const double tc = Pk1[q.o_c], tw = Pk1[q.o_w], ts = Pk1[q.o_s], tse = Pk1[q.o_se];
          const double uu[15] = {bc, be, bn, bnw, ms, mse, mw, mc, me, mnw, mn, tse, ts, tw, tc};
          const double r = pnode<OP>(A, B, cf, (double)k, uu);
          optr[sm.po[k]] = (MODE == kModeResid) ? fv - r : r;
          bc = mc; mc = tc; be = me; bn = mn; bnw = mnw; mw = tw; ms = ts; mse = tse;
        }
        release(k - 1);
      }
    } else {
      double f0 = 0.0, f1 = 0.0;
      if (MODE == kModeResid && q.active) {
        if (1 <= q.len) f0 = __ldg(fptr + sm.po[1]);
        if (2 <= q.len) f1 = __ldg(fptr + sm.po[2]);
      }
      for (int k = 1; k <= kmax; k += 2) {
        // nodes k and k+1 read planes k-1 .. k+2
        const bool two = k + 1 <= kmax;  // uniform: plane k+2 exists
        wait_plane(k + 1);
        if (two) wait_plane(k + 2);
        const double fa = f0, fb = f1;
        if (MODE == kModeResid && q.active) {
          f0 = (k + 2 <= q.len) ? __ldg(fptr + sm.po[k + 2]) : 0.0;
          f1 = (k + 3 <= q.len) ? __ldg(fptr + sm.po[k + 3]) : 0.0;
        }
        if (q.active && k <= q.len) {
          const double* Pk = sptr(k);
          const double* Pk1 = sptr(k + 1);
          const double me = Pk[q.o_e], mn = Pk[q.o_n], mnw = Pk[q.o_nw];
          const double tc = Pk1[q.o_c], tw = Pk1[q.o_w], ts = Pk1[q.o_s], tse = Pk1[q.o_se];
          const double ua[15] = {bc, be, bn, bnw, ms, mse, mw, mc, me, mnw, mn, tse, ts, tw, tc};
          if (k + 1 <= q.len) {  // implies two
            const double me2 = Pk1[q.o_e], mn2 = Pk1[q.o_n], mnw2 = Pk1[q.o_nw];
            const double* Pk2 = sptr(k + 2);
            const double tc2 = Pk2[q.o_c], tw2 = Pk2[q.o_w], ts2 = Pk2[q.o_s], tse2 = Pk2[q.o_se];
            const double ub[15] = {mc, me, mn, mnw, ts, tse, tw, tc, me2, mnw2, mn2, tse2, ts2, tw2, tc2};
            double ra, rb, cw[15];
#pragma unroll
            for (int w = 0; w < 15; ++w) cw[w] = cf[w * 10 + 9];
            pnode2<OP>(A, B, cw, (double)k, ua, ub, ra, rb);
            optr[sm.po[k]] = (MODE == kModeResid) ? fa - ra : ra;
            optr[sm.po[k + 1]] = (MODE == kModeResid) ? fb - rb : rb;
            bc = tc; be = me2; bn = mn2; bnw = mnw2;
            mc = tc2; mw = tw2; ms = ts2; mse = tse2;
          } else {
            const double r = pnode<OP>(A, B, cf, (double)k, ua);
            optr[sm.po[k]] = (MODE == kModeResid) ? fa - r : r;
          }
        }
        release(k - 1);
        if (two) release(k);
      }
    }
    // planes kmax and kmax+1 are still held (both NPS and both parities of kmax)
    release(kmax);
    release(kmax + 1);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.iempty[e]);
    gp += kmax + 2;
  }
}

// Host: static item lists for `grid` persistent CTAs.  Items (macro-major,
// band order) are dealt greedily to the CTA with the least accumulated work
// (nodes + a fixed per-item cost), so at any time the CTAs work on a window
// of consecutive macros.
inline void build_pmarch_schedule(const std::vector<Band>& bands, int64_t ntl, int grid, std::vector<int>& items,
                                  std::vector<int>& off) {
  const int nb = (int)bands.size();
  std::vector<std::vector<int>> per(grid);
  std::vector<std::pair<double, int>> heap;  // (work, cta) min-heap
  for (int c = 0; c < grid; ++c) heap.push_back({0.0, c});
  auto cmp = [](const std::pair<double, int>& x, const std::pair<double, int>& y) {
    return x.first > y.first || (x.first == y.first && x.second > y.second);
  };
  std::make_heap(heap.begin(), heap.end(), cmp);
  for (int64_t it = 0; it < ntl * nb; ++it) {
    const Band& b = bands[it % nb];
    const double w = (double)b.ncolumns * (b.kmax + 1) * 0.5 + 64.0 * (b.kmax + 2) + 4000.0;
    std::pop_heap(heap.begin(), heap.end(), cmp);
    auto& top = heap.back();
    per[top.second].push_back((int)it);
    top.first += w;
    std::push_heap(heap.begin(), heap.end(), cmp);
  }
  items.clear();
  off.assign(grid + 1, 0);
  for (int c = 0; c < grid; ++c) {
    off[c] = (int)items.size();
    items.insert(items.end(), per[c].begin(), per[c].end());
  }
  off[grid] = (int)items.size();
}

}  // namespace hhg
