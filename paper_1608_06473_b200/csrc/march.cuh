// Column-march volume kernels (apply / residual / GS colour pass) -- the
// surrogate hot path.
//
// Layout (include/hhg.h): pos(i,j,k) = planeoff(k) + col(i,j), col(i,j) =
// d(d+1)/2 + j with d = i+j, so a lattice column (i,j) has the SAME column
// index in every plane and plane k is the prefix col < (N-k+1)(N-k+2)/2.
//
// One CTA = (macro, band of diagonals [d0,d1)), one thread = one interior
// column (i,j), marching in k.  The CTA needs, per plane, the diagonals
// [d0-1, d1] only: a CONTIGUOUS range of every plane, brought into a 16-slot
// shared-memory ring by one 1-D TMA bulk copy (cp.async.bulk + mbarrier
// complete_tx) issued >= 8 planes ahead of use.  In plane k-1 / k / k+1 all 15
// stencil neighbours of (i,j,k) sit at only 7 column offsets
// (i,j) (i+1,j) (i,j+1) (i-1,j+1) (i-1,j) (i,j-1) (i+1,j-1).
//
// Stencil weights (fix two indices, evaluate a 1-D
// polynomial incrementally): for q <= 2 the surrogate polynomial restricted to
// column (i,j) is s_w(k) = A_w + B_w k + C_w k^2; A_w, B_w are computed once
// per column (registers) from the macro's coefficients and C_w = c_002 is per
// macro (shared memory, broadcast), so each weight costs 2 DFMA per node
// (Horner in k) and the stencil 15 more: 45 DFMA per unknown (Table flops
// "29+15q" counts the same work).  f and the output are
// read/written straight from/to HBM: consecutive threads own consecutive
// columns => coalesced (apply) or 1 double per sector per colour (GS).
#pragma once
#include "hhg_internal.h"

namespace hhg {


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// mbarrier wait on a precomputed shared-window address
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Delays of the protocol stress tests (HHG_GS_STRESS): a 32-bit hash.
__device__ __forceinline__ uint32_t stress_hash(uint32_t seed, uint32_t a, uint32_t b) {
  uint32_t h = seed * 0x9e3779b9u ^ (a + 0x7f4a7c15u) * 0x85ebca6bu ^ (b + 0x165667b1u) * 0xc2b2ae35u;
  h ^= h >> 15;
  h *= 0x2c1b3c6du;
  h ^= h >> 12;
  return h;
}

// Upper bound of a cross-CTA wait (polls of >= 32 ns: > 1 s) before it traps.
constexpr long long kSpinLimit = 1ll << 25;

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Issue the bulk copy of plane p's band range into ring slot p % RING
// (po = plane offset table in shared memory).
template <int RING = kRing>
__device__ __forceinline__ void issue_plane(const double* ub, const int* po, int p, const Band& b, double* ring,
                                            int slot_len, uint64_t* bars) {
  const int g0 = po[p] + b.c_lo;
  const int a0 = g0 & ~1;
  const int a1 = (g0 + b.ncols + 1) & ~1;
  const uint32_t bytes = (uint32_t)((a1 - a0) * 8);
  const int s = p % RING;
  mbar_expect_tx(&bars[s], bytes);
  tma_load_1d(ring + s * slot_len, ub + a0, bytes, &bars[s]);
}

// Warp 0 issues planes [from, to] in parallel, one lane per plane (to - from < 32).
template <int RING = kRing>
__device__ __forceinline__ void issue_planes(const double* ub, const int* po, int from, int to, const Band& b,
                                             double* ring, int slot_len, uint64_t* bars) {
  if (threadIdx.x < 32) {
    const int p = from + (int)threadIdx.x;
    if (p <= to) issue_plane<RING>(ub, po, p, b, ring, slot_len, bars);
  }
}

// 1/x to ~1 ulp: hardware approximation + two Newton steps (R16:
// the GS division differs from IEEE division by at most a few ulp).
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// GS node value u_I = (f_I - sum_{w != mc} s_w u_w) / s_mc (eq. iteration-scheme,
// PAPER.md:1306-1315) with s_w(k) = A_w + B_w k + C_w k^2, expanded as
// x + k (y + k z) over three accumulation chains; shared by every GS kernel
// (colour passes and the wavefront, gsfront.cuh), so their sweeps are bit-identical.
// uu[15]: neighbour values in direction order (entry kMC unused).
template <int OP, class CW>
__device__ __forceinline__ double gs_node_value_acc(const double (&A)[15], const double (&B)[15], CW Cw, int k,
                                                    const double (&uu)[15], double fv) {
  const double kd = (double)k;
  const double smc = (OP == HHG_OP_SURROGATE) ? fma(fma(Cw(kMC), kd, B[kMC]), kd, A[kMC]) : A[kMC];
  const double rinv = rcp_nr(smc);
  double r;
  if (OP == HHG_OP_SURROGATE) {
    double x = 0.0, y = 0.0, z = 0.0;
#pragma unroll
    for (int w = 0; w < 15; ++w) {
      if (w == kMC) continue;
      x = fma(A[w], uu[w], x);
      y = fma(B[w], uu[w], y);
      z = fma(Cw(w), uu[w], z);
    }
    r = fma(fma(z, kd, y), kd, x);
  } else {
    double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int w = 0; w < 15; ++w) {
      if (w == kMC) continue;
      acc[w % 3] = fma(A[w], uu[w], acc[w % 3]);
    }
    r = (acc[0] + acc[1]) + acc[2];
  }
  return (fv - r) * rinv;
}

template <int OP>
__device__ __forceinline__ double gs_node_value(const double (&A)[15], const double (&B)[15],
                                                const double* __restrict__ Cw, int k, const double (&uu)[15],
                                                double fv) {
  return gs_node_value_acc<OP>(A, B, [&](int w) { return Cw[w]; }, k, uu, fv);
}

// Shared-memory carve-up common to the march kernels (RING plane slots).
template <int RING = kRing>
struct MarchSmem {
  double* ring;     // [RING][slot_len]
  uint64_t* bars;   // [RING]
  double* Cw;       // [16] k^2 coefficients of the 15 weights (per macro)
  int* po;          // [N+2] plane offsets
  int* roff;        // [N+2] ring offset of plane p for the current band (GS passes; set by band_setup)
  __device__ MarchSmem(double* smem, int slot_len, int N = 0) {
    ring = smem;
    bars = (uint64_t*)(smem + RING * slot_len);
    Cw = (double*)(bars + RING);
    po = (int*)(Cw + 16);
    roff = po + (N + 2);
  }
};

__host__ __device__ inline size_t march_smem_bytes(int slot_len, int N, int ring = kRing) {
  return (size_t)ring * slot_len * 8 + ring * 8 + 16 * 8 + (size_t)2 * (N + 2) * 4;
}

struct Column {
  bool active;
  int i, j, d, len, c;
  int o_c, o_e, o_n, o_nw, o_w, o_s, o_se;  // ring offsets of (i,j)(i+1,j)(i,j+1)(i-1,j+1)(i-1,j)(i,j-1)(i+1,j-1)
};

__device__ __forceinline__ Column make_column(const Band& b, int N) {
  Column q;
  int t = threadIdx.x, d = b.d0, j = 0;
  q.active = t < b.ncolumns;
  if (q.active) {
    while (t >= d - 1) { t -= d - 1; ++d; }
    j = t + 1;
  }
  q.d = d;
  q.j = j;
  q.i = d - j;
  q.len = N - 1 - d;
  q.c = (int)col_idx(q.i, j);
  const int lo = b.c_lo;
  q.o_c = q.c - lo;
  q.o_e = (int)col_idx(q.i + 1, j) - lo;
  q.o_n = (int)col_idx(q.i, j + 1) - lo;
  q.o_nw = (int)col_idx(q.i - 1, j + 1) - lo;
  q.o_w = (int)col_idx(q.i - 1, j) - lo;
  q.o_s = (int)col_idx(q.i, j - 1) - lo;
  q.o_se = (int)col_idx(q.i + 1, j - 1) - lo;
  return q;
}

// A_w, B_w of the column's 1-D polynomial s_w(k) = A_w + B_w k + C_w k^2.
template <int OP>
__device__ __forceinline__ void column_coeffs(const double* coef10, const double* cons, int64_t T, int i, int j,
                                              double A[15], double B[15]) {
  if (OP == HHG_OP_SURROGATE) {
    const double* a = coef10 + T * 150;
    const double di = (double)i, dj = (double)j;
#pragma unroll
    for (int w = 0; w < 15; ++w) {
      const double* q = a + w * 10;  // (000)(100)(010)(001)(200)(110)(101)(020)(011)(002)
      A[w] = q[0] + di * (q[1] + di * q[4] + dj * q[5]) + dj * (q[2] + dj * q[7]);
      B[w] = q[3] + di * q[6] + dj * q[8];
    }
  } else {
#pragma unroll
    for (int w = 0; w < 15; ++w) {
      A[w] = cons[T * 15 + w];
      B[w] = 0.0;
    }
  }
}

__device__ __forceinline__ void march_prologue(MarchSmem<>& sm, const Band& b, int N, const double* coef10,
                                               int64_t T, int op) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) mbar_init(&sm.bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 15) sm.Cw[threadIdx.x] = (op == HHG_OP_SURROGATE) ? coef10[T * 150 + threadIdx.x * 10 + 9] : 0.0;
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) sm.po[p] = (int)plane_off(N, p);
  __syncthreads();
}

// ---------------------------------------------------------------------------
// apply / residual: march k = 1..len, one node per step, 7 new shared loads
// ---------------------------------------------------------------------------
// k^2 coefficients C_w (= c_002 of weight w) of up to kCMax macros [T - T0][15],
// uploaded per launch chunk.  T is uniform in the non-persistent march kernel
// (blockIdx), so the compiler keeps the 15 C_w of the CTA's macro in uniform
// registers and feeds them to DFMA directly (no per-node shared loads).
constexpr int kCMax = 512;
// k-loop unroll factors (measured on the B200, tools/kbench.py): the residual's
// f-prefetch rotation and plane-register rotation vanish with 2 (1.66 -> 1.45
// ms); the apply gains nothing (1.10 either way); the GS pass 3 = its refill
// period (2.95 -> 2.89 ms).
#ifndef HHG_RESID_UNROLL
#define HHG_RESID_UNROLL 2
#endif
constexpr int kResidUnroll = HHG_RESID_UNROLL;
#ifndef HHG_APPLY_UNROLL
#define HHG_APPLY_UNROLL 1
#endif
constexpr int kApplyUnroll = HHG_APPLY_UNROLL;
__constant__ double g_cC[kCMax * 15];

template <int OP, int MODE>
__global__ void __launch_bounds__(kMarchThreads, 2)
    k_vol_march(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
                const double* __restrict__ coef10, const double* __restrict__ cons,
                const double* __restrict__ u, const double* __restrict__ f, double* __restrict__ out, int T0) {
  extern __shared__ __align__(16) double smem[];
  MarchSmem<> sm(smem, slot_len);
  const int Tl = blockIdx.y;  // macro within the launch chunk (uniform: S2UR)
  const int64_t T = T0 + Tl;
  const Band b = bands[blockIdx.x];
  const double* ub = u + T * S;
  // barriers + plane offsets, then the first kRing planes are put in flight
  // BEFORE the column coefficients are computed (their HBM latency overlaps it)
  march_prologue(sm, b, N, coef10, T, OP);
  const int last_plane = b.kmax + 1;
  int next_issue = min(kRing, last_plane + 1);  // uniform across the CTA
  issue_planes(ub, sm.po, 0, next_issue - 1, b, sm.ring, slot_len, sm.bars);
  const Column q = make_column(b, N);
  double A[15], B[15];
  column_coeffs<OP>(coef10, cons, T, q.i, q.j, A, B);

  const int clo = b.c_lo;
  auto sptr = [&](int p, int pof) -> const double* {
    return sm.ring + (p & (kRing - 1)) * slot_len + ((pof + clo) & 1);
  };
  int po1 = sm.po[1];
  mbar_wait(&sm.bars[0], 0);
  mbar_wait(&sm.bars[1], 0);
  double bc, be, bn, bnw, mc, mw, ms, mse;
  {
    const double* P0 = sptr(0, 0);
    const double* P1 = sptr(1, po1);
    bc = P0[q.o_c]; be = P0[q.o_e]; bn = P0[q.o_n]; bnw = P0[q.o_nw];
    mc = P1[q.o_c]; mw = P1[q.o_w]; ms = P1[q.o_s]; mse = P1[q.o_se];
  }
  double* const optr = out + T * S + q.c;
  const double* const fptr = f + T * S + q.c;
  // residual: f is loaded FPD steps ahead (its HBM latency hides behind them)
  constexpr int FPD = 5;  // (3: 1.451 ms, 5: 1.440, 8: spills, 1.586)
  double fq[FPD];
#pragma unroll
  for (int x = 0; x < FPD; ++x)
    fq[x] = (MODE == kModeResid && q.active && 1 + x <= q.len) ? __ldg(fptr + sm.po[1 + x]) : 0.0;
#pragma unroll(MODE == kModeResid ? kResidUnroll : kApplyUnroll)
  for (int k = 1; k <= b.kmax; ++k) {
    const int po2 = sm.po[k + 1];
    const double fv = fq[0];
#pragma unroll
    for (int x = 0; x + 1 < FPD; ++x) fq[x] = fq[x + 1];
    if (MODE == kModeResid) fq[FPD - 1] = (q.active && k + FPD <= q.len) ? __ldg(fptr + sm.po[k + FPD]) : 0.0;
    mbar_wait(&sm.bars[(k + 1) & (kRing - 1)], ((k + 1) / kRing) & 1);
    if (q.active && k <= q.len) {
      const double* Pk = sptr(k, po1);
      const double* Pk1 = sptr(k + 1, po2);
      const double me = Pk[q.o_e], mn = Pk[q.o_n], mnw = Pk[q.o_nw];
      const double tc = Pk1[q.o_c], tw = Pk1[q.o_w], ts = Pk1[q.o_s], tse = Pk1[q.o_se];
      const double uu[15] = {bc, be, bn, bnw, ms, mse, mw, mc, me, mnw, mn, tse, ts, tw, tc};
      double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      if (OP == HHG_OP_SURROGATE) {
        const double kd = (double)k;
#pragma unroll
        for (int w = 0; w < 15; ++w) {
          const double s = fma(fma(g_cC[Tl * 15 + w], kd, B[w]), kd, A[w]);
          acc[w % 5] = fma(s, uu[w], acc[w % 5]);
        }
      } else {
#pragma unroll
        for (int w = 0; w < 15; ++w) acc[w % 5] = fma(A[w], uu[w], acc[w % 5]);
      }
      const double r = (acc[0] + acc[1]) + (acc[2] + acc[3]) + acc[4];
      optr[po1] = (MODE == kModeResid) ? fv - r : r;
      bc = mc; mc = tc; be = me; bn = mn; bnw = mnw; mw = tw; ms = ts; mse = tse;
    }
    po1 = po2;
    // every 8 steps: all warps are done with planes <= k; refill their slots.
    // Warps drift freely between these barriers (ring of 16 keeps >= 8 planes ahead).
    if ((k & 7) == 0) {
      __syncthreads();
      const int to = min(k + kRing, last_plane);
      issue_planes(ub, sm.po, next_issue, to, b, sm.ring, slot_len, sm.bars);
      next_issue = max(next_issue, to + 1);
    }
  }
}

// ---------------------------------------------------------------------------
// GS colour pass over one band: every node of colour c = (i+2j+3k) mod 4 of the
// band, in place (eq. iteration-scheme).  Nodes of one
// colour are never neighbours (R14), so the pass is order-free; each
// thread visits its colour-c nodes k = delta + 4s (one per step of 4 planes).
// The column coefficients (A, B) are computed by the caller once per band.
// ---------------------------------------------------------------------------

template <int OP, int RING = kRing>
__device__ __forceinline__ void gs_colour_pass(MarchSmem<RING>& sm, int slot_len, int N, const Band& b, const Column& q,
                                               const double (&A)[15], const double (&B)[15], int colour,
                                               double* __restrict__ ub, const double* __restrict__ fb,
                                               double* __restrict__ wb) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) mbar_init(&sm.bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // colour(i,j,k) = (d + j + 3k) mod 4 == colour  <=>  k == 3 (colour - d - j) mod 4
  const int delta = (3 * ((((colour - q.d - q.j) % 4) + 4) % 4)) % 4;
  const int last_plane = b.kmax + 1;
  int next_issue = min(RING, last_plane + 1);
  issue_planes<RING>(ub, sm.po, 0, next_issue - 1, b, sm.ring, slot_len, sm.bars);
  const int clo = b.c_lo;
  auto sptr = [&](int p) -> const double* { return sm.ring + sm.roff[p]; };
  auto wait_plane = [&](int p) {
    if (p <= last_plane) mbar_wait(&sm.bars[p % RING], (p / RING) & 1);
  };
  const int nsteps = (b.kmax + 4) / 4;
  double f_next = 0.0;
  if (q.active && delta >= 1 && delta <= q.len) f_next = __ldg(fb + sm.po[delta]);
  {
    wait_plane(0);
    wait_plane(1);
  }
  for (int s = 0; s < nsteps; ++s) {
    // planes 4s+1 .. 4s+4 become needed at step s (4s-1, 4s were waited before)
    wait_plane(4 * s + 1);
    wait_plane(4 * s + 2);
    wait_plane(4 * s + 3);
    wait_plane(4 * s + 4);
    const int k = 4 * s + delta;
    const double fv = f_next;
    if (q.active && k + 4 >= 1 && k + 4 <= q.len) f_next = __ldg(fb + sm.po[k + 4]);
    if (q.active && k >= 1 && k <= q.len) {
      const double* Pb = sptr(k - 1);
      const double* Pm = sptr(k);
      const double* Pt = sptr(k + 1);
      const double uu[15] = {Pb[q.o_c],  Pb[q.o_e],  Pb[q.o_n],  Pb[q.o_nw], Pm[q.o_s],
                             Pm[q.o_se], Pm[q.o_w],  0.0,        Pm[q.o_e],  Pm[q.o_nw],
                             Pm[q.o_n],  Pt[q.o_se], Pt[q.o_s],  Pt[q.o_w],  Pt[q.o_c]};
      wb[sm.po[k]] = gs_node_value<OP>(A, B, sm.Cw, k, uu, fv);
    }
    // every 3 steps: all warps done with planes <= 4s+2 (next step reads >= 4s+3);
    // refill up to plane 4s+2+RING (the following 3 steps need <= 4s+16; with
    // RING = 24 the planes of the step after the next refill are already in flight).
    if (s % 3 == 2 || s == nsteps - 1) {
      __syncthreads();
      const int to = min(4 * s + 2 + RING, last_plane);
      issue_planes<RING>(ub, sm.po, next_issue, to, b, sm.ring, slot_len, sm.bars);
      next_issue = max(next_issue, to + 1);
    }
  }
}

// GS colour pass of the persistent sweep (k_gs_items) with QUAD mbarriers: the
// ring of RING planes is RING/4 slots of 4 planes whose bulk copies complete
// on one barrier (arrival count 4: one arrive.expect_tx per plane, plain
// arrives past the last plane), so a thread waits once per step of 4 planes;
// the slot / phase of the next quad advance by one per step.  The 7 neighbour
// columns of column c on diagonal d are c, c +- 1, c - d, c - d - 1,
// c + d + 1, c + d + 2 (col(i,j) = d(d+1)/2 + j), so a plane needs three base
// addresses and immediate offsets.  Refill every R = RING/4 - 3 steps behind a
// CTA barrier; f is loaded FPD steps ahead.  The arithmetic per node is
// gs_node_value_acc's, shared with every GS kernel (bit-identical sweeps).
// The caller initialises the quad barriers (gs_quad_bars_init) before the
// pass-start CTA barrier.
template <int OP, int RING, class CW>
__device__ __forceinline__ void gs_colour_pass_t(MarchSmem<RING>& sm, int slot_len, const Band& b, const Column& q,
                                                 const double (&A)[15], const double (&B)[15], int colour,
                                                 double* __restrict__ ub, const double* __restrict__ fb,
                                                 double* __restrict__ wb, CW Cw, bool pre_issued = false) {
  constexpr int NQ = RING / 4;
  constexpr int R = NQ - 3;  // refill period (steps)
  constexpr int FPD = 2;  // f loaded 2 steps ahead
  const int delta = (3 * ((((colour - q.d - q.j) % 4) + 4) % 4)) % 4;
  const int last_plane = b.kmax + 1;
  const int last_quad = last_plane / 4;
  auto issue_quads = [&](int q0, int q1) {
    if (threadIdx.x < 32 && q1 >= q0) {
      for (int p = 4 * q0 + (int)threadIdx.x; p <= 4 * q1 + 3; p += 32) {
        uint64_t* bar = &sm.bars[(p >> 2) % NQ];
        if (p <= last_plane) {
          const int g0 = sm.po[p] + b.c_lo;
          const int a0 = g0 & ~1;
          const int a1 = (g0 + b.ncols + 1) & ~1;
          const uint32_t bytes = (uint32_t)((a1 - a0) * 8);
          mbar_expect_tx(bar, bytes);
          tma_load_1d(sm.ring + (p % RING) * slot_len, ub + a0, bytes, bar);
        } else {
          mbar_arrive(bar);
        }
      }
    }
  };
  int next_quad = min(NQ, last_quad + 1);
  if (!pre_issued) issue_quads(0, next_quad - 1);  // else gs_issue_first did
  const uint32_t bar0 = smem_u32(sm.bars);
  int wslot = 0;
  uint32_t wph = 0;
  auto wait_next = [&]() {
    mbar_wait_a(bar0 + 8u * (uint32_t)wslot, wph);
    if (++wslot == NQ) {
      wslot = 0;
      wph ^= 1u;
    }
  };
  const double* const rc = sm.ring + q.o_c;
  const int d1 = q.d + 1;
  const unsigned lenu = q.active ? (unsigned)q.len : 0u;  // node k exists iff (unsigned)(k - 1) < lenu
  const int nsteps = (b.kmax + 4) / 4;
  double fq[FPD];  // (issued before the first quad wait: the latencies overlap)
#pragma unroll
  for (int x = 0; x < FPD; ++x) {
    const int kk = 4 * x + delta;
    fq[x] = ((unsigned)(kk - 1) < lenu) ? __ldg(fb + (unsigned)sm.po[kk]) : 0.0;
  }
  wait_next();  // quad 0
  int cd = R;  // steps to the next refill
#pragma unroll(R)
  for (int s = 0; s < nsteps; ++s) {
    if (s + 1 <= last_quad) wait_next();  // quad s+1: planes 4s-1 .. 4s+4 are in
    const int k = 4 * s + delta;
    const double fv = fq[0];
#pragma unroll
    for (int x = 0; x + 1 < FPD; ++x) fq[x] = fq[x + 1];
    {
      const int kf = k + 4 * FPD;
      fq[FPD - 1] = ((unsigned)(kf - 1) < lenu) ? __ldg(fb + (unsigned)sm.po[kf]) : 0.0;
    }
    if ((unsigned)(k - 1) < lenu) {
      const double* Pb = rc + sm.roff[k - 1];
      const double* Pm = rc + sm.roff[k];
      const double* Pt = rc + sm.roff[k + 1];
      const double* Pbh = Pb + d1;  // (i+1, j) (i, j+1)
      const double* Pmh = Pm + d1;
      const double* Pml = Pm - d1;  // (i, j-1) (i-1, j)
      const double* Ptl = Pt - d1;
      const double uu[15] = {Pb[0],  Pbh[0], Pbh[1], Pb[1],  Pml[0], Pm[-1], Pml[1], 0.0,
                             Pmh[0], Pm[1],  Pmh[1], Pt[-1], Ptl[0], Ptl[1], Pt[0]};
      wb[(unsigned)sm.po[k]] = gs_node_value_acc<OP>(A, B, Cw, k, uu, fv);
    }
    // every R steps: all warps done with quads <= s-1 (the next step reads planes >= 4s+3);
    // refill them: quads up to s-1+NQ (the next R steps need quads <= s+R+1).
    if (--cd == 0 || s == nsteps - 1) {
      cd = R;
      __syncthreads();
      const int to = min(s - 1 + NQ, last_quad);
      issue_quads(next_quad, to);
      next_quad = max(next_quad, to + 1);
    }
  }
  // every issued quad is consumed before the barriers are re-initialised
  for (int qq = min(nsteps, last_quad) + 1; qq <= last_quad; ++qq) wait_next();
}

// Warp 0: the first RING/4 quads of a band's colour pass (= gs_colour_pass_t's
// own first issue), for a caller that puts them in flight early.
template <int RING>
__device__ __forceinline__ void gs_issue_first(MarchSmem<RING>& sm, int slot_len, const Band& b,
                                               const double* __restrict__ ub) {
  constexpr int NQ = RING / 4;
  const int last_plane = b.kmax + 1;
  const int q1 = min(NQ, last_plane / 4 + 1) - 1;
  if (threadIdx.x < 32) {
    for (int p = (int)threadIdx.x; p <= 4 * q1 + 3; p += 32) {
      uint64_t* bar = &sm.bars[(p >> 2) % NQ];
      if (p <= last_plane) {
        const int g0 = sm.po[p] + b.c_lo;
        const int a0 = g0 & ~1;
        const int a1 = (g0 + b.ncols + 1) & ~1;
        const uint32_t bytes = (uint32_t)((a1 - a0) * 8);
        mbar_expect_tx(bar, bytes);
        tma_load_1d(sm.ring + (p % RING) * slot_len, ub + a0, bytes, bar);
      } else {
        mbar_arrive(bar);
      }
    }
  }
}

// thread 0: fresh quad barriers for the next colour pass (every thread is past
// the previous pass's last wait); made visible by the caller's next bar.sync
template <int RING>
__device__ __forceinline__ void gs_quad_bars_init(MarchSmem<RING>& sm) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < RING / 4; ++s) mbar_init(&sm.bars[s], 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// Shared-memory tables of a band (plane offsets, ring offsets, C_w), then a
// CTA barrier.
template <int OP, int RING>
__device__ __forceinline__ void band_tables(MarchSmem<RING>& sm, int N, const Band& b, int64_t T, int slot_len,
                                            const double* __restrict__ coef10) {
  if (threadIdx.x < 15) sm.Cw[threadIdx.x] = (OP == HHG_OP_SURROGATE) ? coef10[T * 150 + threadIdx.x * 10 + 9] : 0.0;
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) {
    const int pof = (int)plane_off(N, p);
    sm.po[p] = pof;
    sm.roff[p] = (p % RING) * slot_len + ((pof + b.c_lo) & 1);
  }
  __syncthreads();
}

template <int OP, int RING = kRing>
__device__ __forceinline__ void band_setup(MarchSmem<RING>& sm, int N, const Band& b, int64_t T, int slot_len,
                                           const double* __restrict__ coef10, const double* __restrict__ cons,
                                           Column& q, double (&A)[15], double (&B)[15]) {
  q = make_column(b, N);
  column_coeffs<OP>(coef10, cons, T, q.i, q.j, A, B);
  if (threadIdx.x < 15) sm.Cw[threadIdx.x] = (OP == HHG_OP_SURROGATE) ? coef10[T * 150 + threadIdx.x * 10 + 9] : 0.0;
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) {
    const int pof = (int)plane_off(N, p);
    sm.po[p] = pof;
    // ring slot of plane p + the 16-byte alignment shift of its bulk copy
    sm.roff[p] = (p % RING) * slot_len + ((pof + b.c_lo) & 1);
  }
  __syncthreads();
}

// One colour pass, one CTA per (macro, band).
template <int OP>
__global__ void __launch_bounds__(kMarchThreads, 2)
    k_gs_march(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
               const double* __restrict__ coef10, const double* __restrict__ cons, int colour,
               double* __restrict__ u, const double* __restrict__ f, int64_t T0) {
  extern __shared__ __align__(16) double smem[];
  MarchSmem<> sm(smem, slot_len, N);
  const int64_t Tr = blockIdx.x / n_bands;
  const int64_t T = T0 + Tr;
  const Band b = bands[blockIdx.x - Tr * n_bands];
  Column q;
  double A[15], B[15];
  band_setup<OP>(sm, N, b, T, slot_len, coef10, cons, q, A, B);
  gs_colour_pass<OP>(sm, slot_len, N, b, q, A, B, colour, u + T * S, f + T * S + q.c, u + T * S + q.c);
}

// ---------------------------------------------------------------------------
// Whole volume GS (4 colours) as ONE persistent launch.  Work item = (macro,
// band): the CTA runs the band's four colour passes in order; before colour c
// it waits until bands b-1, b+1 of the same macro have finished colour c-1
// (completion flags = sweep epoch).  That is exactly the colour order of the
// 4-colour GS: colour c of band b reads only bands b-1..b+1, and colour-c nodes
// are never neighbours of each other.  Items are handed out in (macro, band)
// order by an atomic counter, so the ~8 macros in flight keep u and f
// L2-resident across their four colours (HBM sees ~1x u, f, u instead of 4x).
// Only the single partially handed-out macro can wait on an item that is not
// running yet; every other running item's neighbours run too => no deadlock
// while the grid has more CTAs than a macro has bands.
// ---------------------------------------------------------------------------
// Items come from an atomic counter; C_w through shared memory.
// CWC: the macro's C_w from the constant bank g_cC (chunk [T0, T0 + ntl),
// ntl <= kCMax, uploaded by the launcher) as uniform-register DFMA operands
// (the item index is made warp-uniform by a shuffle); else from shared memory.
template <int OP, int NT, int RING, bool CWC, bool PROF>
__global__ void __launch_bounds__(NT, 512 / NT)
    k_gs_items(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
               const double* __restrict__ coef10, const double* __restrict__ cons, double* __restrict__ u,
               const double* __restrict__ f, int64_t ntl, int64_t T0, int* __restrict__ counter,
               int* __restrict__ flags, int epoch, int stress, unsigned long long* __restrict__ prof) {
  static_assert(RING % 8 == 0 && RING >= 16, "quad ring: RING / 4 slots, refill period RING / 4 - 3 >= 1");
  extern __shared__ __align__(16) double smem[];
  MarchSmem<RING> sm(smem, slot_len, N);
  __shared__ int s_item;
  const int64_t total = ntl * n_bands;
  // optional cycle accounting (PROF, tools/gsprof.py): thread 0's
  // cycles in [0] item fetch + band setup, [1] flag wait, [2] pass-start
  // barrier, [3] colour pass, [4] pass-end barrier; [6] steps, [7] items
  long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tq = PROF ? clock64() : 0;
  auto tick = [&](int slot, long long& t) {
    if (PROF) {
      const long long now = clock64();
      pacc[slot] += now - t;
      t = now;
    }
  };
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int64_t item = s_item;  // rewritten only after band_tables' CTA barrier
    if (item >= total) break;
    const int64_t Tr = item / n_bands;  // macro within the launch's range [T0, T0 + ntl)
    const int64_t T = T0 + Tr;
    // stress test (HHG_GS_STRESS): bands of a macro handed out in reverse order
    // (macro-major order kept: still deadlock-free) and random delays below
    const int band = (stress & 1) ? n_bands - 1 - (int)(item - Tr * n_bands) : (int)(item - Tr * n_bands);
    const Band b = bands[band];
    Column q;
    double A[15], B[15];
    // tables, then colour 0's first quads go in flight (colour 0 waits for no
    // neighbour), then the column coefficients: their L2 latency overlaps the
    // bulk copies
    gs_quad_bars_init(sm);  // visible after band_tables' CTA barrier
    band_tables<OP, RING>(sm, N, b, T, slot_len, coef10);
    if (threadIdx.x < 32) asm volatile("fence.proxy.async.global;" ::: "memory");
    gs_issue_first<RING>(sm, slot_len, b, u + T * S);
    q = make_column(b, N);
    column_coeffs<OP>(coef10, cons, T, q.i, q.j, A, B);
    tick(0, tq);
    pacc[7] += 1;
    for (int colour = 0; colour < 4; ++colour) {
      if (threadIdx.x == 0 && colour > 0) {
        for (int bb = band - 1; bb <= band + 1; bb += 2) {
          if (bb < 0 || bb >= n_bands) continue;
          const int* fl = flags + ((T * n_bands + bb) * 4 + colour - 1);
          // bounded wait: a protocol fault traps (sticky launch error,
          // HHG_ERR_CUDA) instead of hanging the device
          for (long long spin = 0; ld_acquire_gpu(fl) != epoch; ++spin) {
            if (spin > kSpinLimit) __trap();
            __nanosleep(32);
          }
        }
      }
      if (stress && threadIdx.x == 0) __nanosleep(stress_hash(stress, (uint32_t)(T * n_bands + band), colour) & 8191);
      tick(1, tq);
      if (colour > 0) {
        __syncthreads();
        // the lanes of warp 0 issue the pass's bulk copies: order this CTA's and the
        // neighbours' generic global writes before their async-proxy reads
        if (threadIdx.x < 32) asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      tick(2, tq);
      if (CWC) {
        const int cwb = __shfl_sync(0xffffffffu, (int)Tr, 0) * 15;
        gs_colour_pass_t<OP, RING>(sm, slot_len, b, q, A, B, colour, u + T * S, f + T * S + q.c, u + T * S + q.c,
                                   [&](int w) { return g_cC[cwb + w]; }, colour == 0);
      } else {
        const double* const Cw = sm.Cw;
        gs_colour_pass_t<OP, RING>(sm, slot_len, b, q, A, B, colour, u + T * S, f + T * S + q.c, u + T * S + q.c,
                                   [&](int w) { return Cw[w]; }, colour == 0);
      }
      tick(3, tq);
      pacc[6] += (b.kmax + 4) / 4;
      __syncthreads();
      tick(4, tq);
      // bar.sync orders every thread's stores before the gpu-scope release
      // (cumulative); the neighbours' acquire loads pair with it
      // (by warp 1: its fence overlaps thread 0's poll of the next pass's
      // flags; colour 3's flag is never awaited, so it is not released)
      if (threadIdx.x == 32 && colour < 3) st_release_gpu(flags + ((T * n_bands + band) * 4 + colour), epoch);
      if (colour < 3) gs_quad_bars_init(sm);
    }
  }
  if (PROF && threadIdx.x == 0)
    for (int x = 0; x < 8; ++x) atomicAdd(prof + x, (unsigned long long)pacc[x]);
}

}  // namespace hhg
