// Multicolour Gauss-Seidel volume sweep as ONE persistent, continuously
// pipelined kernel (eq. iteration-scheme; colour order
// (i+2j+3k) mod 4 = 0,1,2,3, R13/R14).
//
// Work item = (macro T, band b of diagonals).  A CTA runs the item's four
// colour passes back to back over ONE continuous stream of planes (pass 0
// planes 0..kmax+1, pass 1 planes 0..kmax+1, ...): the TMA ring never drains
// between passes or between items.  Every plane is (re)loaded from global
// memory for each pass, so the halo diagonals always carry the neighbours'
// latest colours; the macro's u and f stay L2-resident across the four passes
// (a few macros are in flight at any time), so HBM sees ~1x u, f and u-write.
//
// Ordering (the GS dependency DAG): colour c at plane p of band b reads
// colour c-1 nodes at planes p-1..p+1 of bands b-1, b, b+1.  Each item
// publishes its progress (epoch, pass, planes done) in global memory; the
// producer of a plane of pass c checks that the three predecessor bands have
// finished pass c-1 up to that plane + 1 (read-after-write).  Write-after-read
// is implied: a neighbour overwrites a colour-c' node only after our colour c
// < c' pass passed it (it waits for our progress the same way).  Items are
// handed out in (macro, band) order and a CTA takes its next item only after
// its current item issued its last dependent plane, so the oldest unfinished
// item can always run (no deadlock while #CTAs > bands per macro).
//
// Inside a pass a thread owns one lattice column (i,j); its colour-c nodes
// sit at planes k = delta (mod 4), delta = 3 (c - (i + 2j)) mod 4, so the pass
// marches in plane quads [4q, 4q+3] and every thread updates exactly one node
// per quad (all lanes busy).  Node update u = (f - sum_{w != mc} s_w u_w)/s_mc
// with the weight polynomial expanded per column (A_w + k B_w + k^2 C_w, three
// independent FMA chains) and 1/s_mc by rcp + 2 Newton steps (R16).
#pragma once
#include "pair.cuh"

namespace hhg {

constexpr int kGThreads = 256;
constexpr int kGWarps = kGThreads / 32;
constexpr int kGRQ = 6;               // ring slots, each a QUAD of planes (4q .. 4q+3)
constexpr int kGAhead = kGRQ - 3;     // quads a warp issues ahead of its own position
constexpr int kGPassStride = 1024;    // progress encoding: pass * 1024 + planes done
constexpr int kGEpoch = 8 * 1024;     // ... + epoch * 8192
#ifndef HHG_GS_PUB
#define HHG_GS_PUB 3
#endif
constexpr int kGPubMask = HHG_GS_PUB;  // publish progress every (mask+1) quads

struct GSmem {
  double* ring;      // [kGRQ][4][slot_len]
  double* coef;      // [2][160] coefficients of the current / next item
  uint64_t* full;    // [kGRQ]
  uint64_t* empty;   // [kGRQ]
  uint64_t* cfull;   // [2]
  uint64_t* cempty;  // [2]
  int* po;           // [N+2]
  int* qitem;        // [4] items of this CTA (ring by sequence number); -1 = done
  int* qcount;       // [1] items fetched
  int* own;          // [1] own progress: item sequence * 8192 + pass * 1024 + planes done
  __device__ GSmem(double* smem, int slot_len, int N) {
    ring = smem;
    coef = ring + (size_t)kGRQ * 4 * slot_len;
    full = (uint64_t*)(coef + 2 * 160);
    empty = full + kGRQ;
    cfull = empty + kGRQ;
    cempty = cfull + 2;
    po = (int*)(cempty + 2);
    qitem = po + (N + 2);
    qcount = qitem + 4;
    own = qcount + 1;
  }
};

__host__ __device__ inline size_t gsq_smem_bytes(int slot_len, int N) {
  return (size_t)kGRQ * 4 * slot_len * 8 + 2 * 160 * 8 + (2 * kGRQ + 4) * 8 + (size_t)(N + 2) * 4 + 6 * 4;
}

struct GArgs {
  int N;
  int64_t S;
  const Band* bands;
  int n_bands;
  int slot_len;
  const double* coef10;
  const double* u;
  int* prog;        // [ntl * n_bands] progress words
  int epoch;
  int64_t total;    // items
  int* counter;
};

// Issue cursor of one warp (lane 0): the next quad g (g mod 8 == warp) of the
// CTA's quad stream; n = item sequence number, c = pass, p = quad in pass.
struct GCursor {
  int g, n, c, p;
  int T, b, np;    // item of sequence n; np = quads per pass (0 = item unknown)
  int nplanes;     // kmax + 2 planes per pass
  int need;        // quad g whose dependencies were already found satisfied
  int seen;        // cached min progress of the two neighbour bands of item n
  unsigned tpoll;  // clock of the last global poll (throttle)
};

__device__ __forceinline__ int gs_item(const GSmem& sm, int n) {
  if (*(volatile int*)sm.qcount <= n) return -2;
  return ((volatile int*)sm.qitem)[n & 3];
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Predecessors of quad p of pass c (c >= 1) of band b have finished pass c-1
// up to plane 4p+4 inclusive (progress >= (c-1)*1024 + 4p + 5).  Own band: the
// CTA's own progress word in shared memory (tagged with the item sequence
// number).  Neighbour bands b-1, b+1: their global progress words; `seen`
// caches the smaller as last observed; re-read (two relaxed loads + one
// acquire fence) only when insufficient, at most once per ~2k cycles per warp.
__device__ __forceinline__ bool gs_deps_ok(const GArgs& a, const GSmem& sm, GCursor& cu) {
  if (cu.c == 0) return true;
  const int rel = (cu.c - 1) * kGPassStride + 4 * cu.p + 5;
  if (*(volatile int*)sm.own < cu.n * kGEpoch + rel) return false;
  const int want = a.epoch * kGEpoch + rel;
  if (cu.seen >= want) return true;
  const unsigned now = (unsigned)clock();
  if (cu.tpoll != 0u && now - cu.tpoll < 2048u) return false;
  cu.tpoll = now | 1u;
  const int* base = a.prog + (int64_t)cu.T * a.n_bands;
  const int big = 0x7fffffff;
  const int v0 = cu.b > 0 ? ld_relaxed(base + cu.b - 1) : big;
  const int v2 = cu.b + 1 < a.n_bands ? ld_relaxed(base + cu.b + 1) : big;
  cu.seen = min(v0, v2);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  return cu.seen >= want;
}

__device__ __forceinline__ bool gs_cursor_settle(GCursor& cu, const GArgs& a, const GSmem& sm) {
  for (;;) {
    if (cu.np == 0) {
      const int it = gs_item(sm, cu.n);
      if (it == -2) return false;
      if (it < 0) {
        cu.T = -1;
        return false;
      }
      cu.T = it / a.n_bands;
      cu.b = it - cu.T * a.n_bands;
      cu.nplanes = a.bands[cu.b].kmax + 2;
      cu.np = (cu.nplanes + 3) / 4;
    }
    if (cu.T < 0) return false;
    if (cu.p < cu.np) return true;
    cu.p -= cu.np;
    if (++cu.c == 4) {
      cu.c = 0;
      ++cu.n;
      cu.np = 0;
      cu.seen = -1;
    }
  }
}

// Fetch the next item of this CTA (called by the warp that issued the last
// quad of the current item's pass 3: from then on the item waits on nobody).
__device__ __forceinline__ void gs_fetch(GSmem& sm, const GArgs& a) {
  const int qc = *(volatile int*)sm.qcount;
  const int it = atomicAdd(a.counter, 1);
  ((volatile int*)sm.qitem)[qc & 3] = it < a.total ? (int)it : -1;
  __threadfence_block();
  *(volatile int*)sm.qcount = qc + 1;
}

template <int OP>
__device__ __forceinline__ void gs_try_issue(GCursor& cu, const GArgs& a, GSmem& sm, int limit) {
  while (cu.g < limit) {
    if (!gs_cursor_settle(cu, a, sm)) return;
    const int slot = cu.g % kGRQ;
    if (cu.g >= kGRQ && !mbar_test(&sm.empty[slot], ((cu.g / kGRQ) - 1) & 1)) return;
    if (cu.need != cu.g) {
      if (!gs_deps_ok(a, sm, cu)) return;
      cu.need = cu.g;
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (cu.c == 0 && cu.p == 0) {  // first quad of the item: its coefficients
      const int e = cu.n & 1;
      if (cu.n >= 2 && !mbar_test(&sm.cempty[e], ((cu.n / 2) - 1) & 1)) return;
      if (OP == HHG_OP_SURROGATE) {
        mbar_expect_tx(&sm.cfull[e], 150 * 8);
        tma_load_1d(sm.coef + e * 160, a.coef10 + (int64_t)cu.T * 150, 150 * 8, &sm.cfull[e]);
      } else {
        mbar_arrive(&sm.cfull[e]);
      }
    }
    const Band& b = a.bands[cu.b];
    const int p0 = 4 * cu.p, p1 = min(p0 + 4, cu.nplanes);
    uint32_t nbytes[4];
    int src0[4];
    uint32_t total = 0;
    for (int p = p0; p < p1; ++p) {
      const int g0 = sm.po[p] + b.c_lo;
      const int a0 = g0 & ~1;
      nbytes[p - p0] = (uint32_t)((((g0 + b.ncols + 1) & ~1) - a0) * 8);
      src0[p - p0] = a0;
      total += nbytes[p - p0];
    }
    mbar_expect_tx(&sm.full[slot], total);
    const double* src = a.u + (int64_t)cu.T * a.S;
    double* dst = sm.ring + (size_t)slot * 4 * a.slot_len;
    for (int p = p0; p < p1; ++p)
      tma_load_1d(dst + (size_t)(p - p0) * a.slot_len, src + src0[p - p0], nbytes[p - p0], &sm.full[slot]);
    const bool last = cu.c == 3 && cu.p == cu.np - 1;
    cu.g += kGWarps;
    cu.p += kGWarps;
    if (last) gs_fetch(sm, a);
  }
}

template <int OP>
__device__ __forceinline__ void gs_wait(uint64_t* bar, uint32_t parity, GCursor& cu, const GArgs& a, GSmem& sm,
                                        int limit) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    if (lane == 0 && cu.g < limit) gs_try_issue<OP>(cu, a, sm, limit);
    __syncwarp();
    if (__all_sync(0xffffffffu, mbar_try(bar, parity))) break;
  }
}


template <int OP>
__global__ void __launch_bounds__(kGThreads, 2)
    k_gs_quad(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
              const double* __restrict__ coef10, const double* __restrict__ cons, double* __restrict__ u,
              const double* __restrict__ f, int64_t ntl, int* __restrict__ counter, int* __restrict__ prog,
              int epoch) {
  extern __shared__ __align__(16) double smem[];
  GSmem sm(smem, slot_len, N);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const GArgs a{N, S, bands, n_bands, slot_len, coef10, u, prog, epoch, ntl * n_bands, counter};
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGRQ; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kGWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.cfull[s], 1);
      mbar_init(&sm.cempty[s], kGWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    *sm.qcount = 0;
    *sm.own = 0;
    gs_fetch(sm, a);
  }
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) sm.po[p] = (int)plane_off(N, p);
  __syncthreads();

  GCursor cu;
  cu.g = warp;
  cu.n = 0;
  cu.c = 0;
  cu.p = warp;
  cu.np = 0;
  cu.nplanes = 0;
  cu.T = 0;
  cu.b = 0;
  cu.need = -1;
  cu.seen = -1;
  cu.tpoll = 0u;
  if (lane == 0) gs_try_issue<OP>(cu, a, sm, kGAhead);

  int gq = 0;  // stream number of quad 0 of the current pass
#ifdef HHG_GS_PROF
  const long long tk0 = clock64();
#endif
  for (int n = 0;; ++n) {
    int it;
    GPROF_T0
    for (;;) {  // item n of this CTA (fetched by whichever warp finished issuing item n-1)
      if (lane == 0 && cu.g < gq + kGAhead) gs_try_issue<OP>(cu, a, sm, gq + kGAhead);
      __syncwarp();
      it = gs_item(sm, n);
      if (__all_sync(0xffffffffu, it != -2)) break;
      __nanosleep(32);
    }
    if (it < 0) break;
    const int T = it / n_bands;
    const int bi = it - T * n_bands;
    const Band b = bands[bi];
    const int e = n & 1;
    gs_wait<OP>(&sm.cfull[e], (n / 2) & 1, cu, a, sm, gq + kGAhead);
    GPROF_ADD(2)
    const QCol q = qcolumn(b, N);
    const double* cf = sm.coef + e * 160;
    double A[15], B[15];
    pcolumn_coeffs<OP>(cf, cons, T, q.i, q.j, A, B);
    const int clo = b.c_lo;
    const int kmax = b.kmax;
    const int np = kmax + 2;           // planes per pass
    const int nq = (np + 3) / 4;       // stream quads per pass
    const int nquads = kmax / 4 + 1;   // compute quads per pass
    const int xcol = q.i + 2 * q.j;
    double* const ucol = u + (int64_t)T * S + q.c;
    const double* const fcol = f + (int64_t)T * S + q.c;
    int* const myprog = prog + (int64_t)T * n_bands + bi;

    for (int c = 0; c < 4; ++c) {
      const int delta = ((c - xcol) * 3) & 3;
      auto sptr = [&](int p) -> const double* {
        const int g = gq + (p >> 2);
        return sm.ring + ((size_t)(g % kGRQ) * 4 + (p & 3)) * slot_len + ((sm.po[p] + clo) & 1);
      };
      int waited = -1;  // quads <= waited are resident
      auto wait_upto = [&](int qq) {
        qq = min(qq, nq - 1);
        for (; waited < qq;) {
          ++waited;
          const int g = gq + waited;
          gs_wait<OP>(&sm.full[g % kGRQ], (g / kGRQ) & 1, cu, a, sm, g + kGAhead);
        }
      };
      int released = -1;  // quads <= released are given back
      auto release_upto = [&](int qq) {
        qq = min(qq, nq - 1);
        __syncwarp();
        for (; released < qq;) {
          ++released;
          if (lane == 0) mbar_arrive(&sm.empty[(gq + released) % kGRQ]);
        }
      };
      double fnext = 0.0;
      if (q.active && delta >= 1 && delta <= q.len) fnext = __ldg(fcol + sm.po[delta]);
      for (int qd = 0; qd < nquads; ++qd) {
        const int k = 4 * qd + delta;
        {
          GPROF_T0
          wait_upto(qd + 1);  // planes 4qd-1 .. 4qd+4
          GPROF_ADD(0)
        }
        const double fv = fnext;
        if (q.active && k + 4 >= 1 && k + 4 <= q.len) fnext = __ldg(fcol + sm.po[k + 4]);
        if (q.active && k >= 1 && k <= q.len) {
          const double* Pb = sptr(k - 1);
          const double* Pm = sptr(k);
          const double* Pt = sptr(k + 1);
          const double uu[15] = {Pb[q.o_c], Pb[q.o_e], Pb[q.o_n], Pb[q.o_nw], Pm[q.o_s],
                                 Pm[q.o_se], Pm[q.o_w], 0.0, Pm[q.o_e], Pm[q.o_nw],
                                 Pm[q.o_n], Pt[q.o_se], Pt[q.o_s], Pt[q.o_w], Pt[q.o_c]};
          const double kd = (double)k;
          double x = 0.0, y = 0.0, z = 0.0, smc;
          if (OP == HHG_OP_SURROGATE) {
#pragma unroll
            for (int w = 0; w < 15; ++w) {
              if (w == kMC) continue;
              x = fma(A[w], uu[w], x);
              y = fma(B[w], uu[w], y);
              z = fma(cf[w * 10 + 9], uu[w], z);
            }
            smc = fma(fma(cf[kMC * 10 + 9], kd, B[kMC]), kd, A[kMC]);
          } else {
#pragma unroll
            for (int w = 0; w < 15; ++w) {
              if (w == kMC) continue;
              x = fma(A[w], uu[w], x);
            }
            smc = A[kMC];
          }
          const double r = fma(fma(z, kd, y), kd, x);
          ucol[sm.po[k]] = (fv - r) * rcp_nr(smc);
        }
        release_upto(qd - 1);  // quad qd-1 (planes 4qd-4 .. 4qd-1) is no longer needed
        if (kGPubMask == 0 || (qd & kGPubMask) == kGPubMask || qd == nquads - 1) {
          // publish: colour c done on planes < 4 qd + 4 (all threads' stores of this pass so far;
          // bar.sync orders them before thread 0's release store)
          GPROF_T0
          __syncthreads();
          GPROF_ADD(1)
          if (threadIdx.x == 0) {
            const int done = qd == nquads - 1 ? (c + 1) * kGPassStride : c * kGPassStride + min(4 * qd + 4, np);
            *(volatile int*)sm.own = n * kGEpoch + done;
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(myprog), "r"(epoch * kGEpoch + done)
                         : "memory");
          }
        }
      }
      wait_upto(nq - 1);  // quads past the last compute window still hold a TMA phase
      release_upto(nq - 1);
      gq += nq;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.cempty[e]);
#ifdef HHG_GS_PROF
    if (threadIdx.x == 0) atomicAdd(&g_gsprof[4], (unsigned long long)(4 * nquads));
#endif
  }
#ifdef HHG_GS_PROF
  if (threadIdx.x == 0) atomicAdd(&g_gsprof[3], (unsigned long long)(clock64() - tk0));
#endif
}

}  // namespace hhg
