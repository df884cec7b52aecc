// Persistent 4-colour volume GS with a PRODUCER warp (warp-specialised
// variant of march.cuh::k_gs_items; HHG_GS_KERNEL=prod).
//
// Same work items (macro, band), same four colour passes per item, same
// per-node arithmetic (gs_node_value_acc) and the same colour order -- the
// sweep is bit-identical to k_gs_items and to the four colour launches.  What
// changes is who waits for what:
//
// * NCW compute warps march the band's columns and never meet at a CTA barrier
//   inside an item: they wait only for their ring quads (mbarriers, phases
//   running continuously over passes and items) and, every R steps, ARRIVE
//   (bar.arrive, non-blocking) on a named barrier to release the quads they
//   are done with.
// * 1 producer warp syncs on that named barrier, publishes the band's
//   progress, checks the neighbour bands' progress and issues the bulk copies
//   of the next quads.
// * Cross-band ordering is per plane instead of per pass: progress word of
//   (macro, band) = 1 + c K + p once colour c is complete on planes <= p
//   (K = 1024 > any plane index; pass complete: p = K - 1).  Before loading
//   planes <= P for colour c >= 1 the producer needs both neighbours at
//   >= 1 + (c-1) K + min(P, K-1): their colour c-1 values on those planes are
//   final (read-after-write), and they have finished every colour c-1 node
//   that reads our planes <= P - 1 (write-after-read: we write a plane-k node
//   only after loading plane k+1).  Waits only ever point at colour c-1, so
//   the wait graph is acyclic in colour; with every band of the partially
//   handed-out macro resident (grid > bands per macro) it cannot deadlock.
//   Neighbour words are read relaxed one refill ahead and confirmed with an
//   acquire fence, so the producer rarely waits a round trip.
//
// Measured on the bench workload (tools/kbench.py, r02): 2.75 ms ("prodw": 15
// compute warps, one CTA per SM) and 3.60 ms ("prod": 7 compute warps, two
// CTAs per SM) against 2.57 ms for k_gs_items.  Each mid-pass progress
// release is a gpu-scope fence that waits for the CTA's outstanding stores
// (~1 us); publishing only at pass ends ("prod": 2.84 ms) removes that but
// also the per-plane early start; and the producer warp costs 1/16 of the
// compute warps.  Kept opt-in, bit-identical and stress-tested.
#pragma once
#include "march.cuh"

namespace hhg {

// mbarrier wait that traps instead of hanging the device (protocol fault)
__device__ __forceinline__ void mbar_wait_bounded(uint32_t bar, uint32_t parity) {
  for (long long n = 0;; ++n) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) return;
    if (n > (kSpinLimit >> 4)) __trap();
  }
}

// named barriers 1 / 2 (immediate ids: ptxas then reserves only those)
template <int N>
__device__ __forceinline__ void nbar_arrive(int which) {
  if (which) asm volatile("bar.arrive 2, %0;" ::"n"(N) : "memory");
  else asm volatile("bar.arrive 1, %0;" ::"n"(N) : "memory");
}

template <int N>
__device__ __forceinline__ void nbar_sync(int which) {
  if (which) asm volatile("bar.sync 2, %0;" ::"n"(N) : "memory");
  else asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kProgK = 1024;  // progress encoding: 1 + colour * kProgK + plane

// NCW compute warps (bands of <= 32 NCW columns) + 1 producer warp; 16 warps
// per SM either way (7: two CTAs per SM, 15: one), so 128 registers per thread.
template <int OP, int RING, bool CWC, int NCW>
__global__ void __launch_bounds__(32 * NCW + 32, NCW <= 7 ? 2 : 1)
    k_gs_prod(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
              const double* __restrict__ coef10, const double* __restrict__ cons, double* __restrict__ u,
              const double* __restrict__ f, int64_t ntl, int64_t T0, int* __restrict__ counter,
              int* __restrict__ prog, int stress) {
  static_assert(RING % 8 == 0 && RING >= 24, "quad ring with refill period RING / 4 - 3 >= 3");
  constexpr int NT = 32 * NCW;  // compute threads; the producer is warp NCW
  constexpr int NQ = RING / 4;
  constexpr int R = NQ - 3;
  constexpr int FPD = 2;
  extern __shared__ __align__(16) double smem[];
  MarchSmem<RING> sm(smem, slot_len, N);
  __shared__ int s_item;
  const bool producer = threadIdx.x >= NT;
  const int lane = (int)(threadIdx.x & 31);
  const int64_t total = ntl * n_bands;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NQ; ++s) mbar_init(&sm.bars[s], 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) sm.po[p] = (int)plane_off(N, p);
  __syncthreads();
  const uint32_t bar0 = smem_u32(sm.bars);
  // the quad sequence runs on over passes and items: gq = quads of all
  // earlier passes (both roles count the same passes)
  uint32_t gq = 0;
  int wslot = 0;  // compute warps: barrier slot / phase of their next quad
  uint32_t wph = 0;
  int seen_lo = 0, seen_hi = 0, pf_lo = 0, pf_hi = 0;  // producer lane 0: neighbour progress
  // release points alternate between named barriers 1 and 2: a compute warp
  // cannot reach the release point after next before the producer has synced
  // on this one (it needs the quads that sync releases), so no barrier phase
  // ever sees a warp twice
  int nbid = 0;
  if (producer) {
  for (;;) {
    if (threadIdx.x == NT) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= total) break;
    const int64_t Tr = item / n_bands;
    const int64_t T = T0 + Tr;
    const int band = (stress & 1) ? n_bands - 1 - (int)(item - Tr * n_bands) : (int)(item - Tr * n_bands);
    const Band b = bands[band];
    const int last_plane = b.kmax + 1;
    const int last_quad = last_plane / 4;
    const int nsteps = (b.kmax + 4) / 4;
    double* const ub = u + T * S;
    for (int p = lane; p <= N + 1; p += 32) sm.roff[p] = (p % RING) * slot_len + ((sm.po[p] + b.c_lo) & 1);
    if (!CWC && lane < 15) sm.Cw[lane] = OP == HHG_OP_SURROGATE ? coef10[T * 150 + lane * 10 + 9] : 0.0;
    seen_lo = seen_hi = pf_lo = pf_hi = 0;
    __syncthreads();  // roff / Cw of this item; every thread is past the previous item
      // ------------------------------------------------------------ producer
      const int* nlo = band > 0 ? prog + T * n_bands + band - 1 : nullptr;
      const int* nhi = band + 1 < n_bands ? prog + T * n_bands + band + 1 : nullptr;
      int* own = prog + T * n_bands + band;
      for (int colour = 0; colour < 4; ++colour) {
        const uint32_t gq0 = gq;
        // planes <= P of this colour may be loaded once both neighbours are at
        // colour - 1 on them (lane 0 checks; the warp then fences and issues)
        auto ensure = [&](int P) {
          if (colour > 0 && lane == 0) {
            const int need = 1 + (colour - 1) * kProgK + min(P, kProgK - 1);
            if (nlo) {
              seen_lo = max(seen_lo, pf_lo);
              for (long long n = 0; seen_lo < need; ++n) {
                if (n > kSpinLimit) __trap();
                __nanosleep(32);
                seen_lo = ld_relaxed_gpu(nlo);
              }
            }
            if (nhi) {
              seen_hi = max(seen_hi, pf_hi);
              for (long long n = 0; seen_hi < need; ++n) {
                if (n > kSpinLimit) __trap();
                __nanosleep(32);
                seen_hi = ld_relaxed_gpu(nhi);
              }
            }
            asm volatile("fence.acquire.gpu;" ::: "memory");
          }
          if (stress && lane == 0) __nanosleep(stress_hash(stress, (uint32_t)(T * n_bands + band), colour * 64 + P) & 4095);
          __syncwarp();
          // order the neighbours' (acquired) and this CTA's (named barrier)
          // generic writes before the async-proxy reads of the bulk copies
          asm volatile("fence.proxy.async.global;" ::: "memory");
        };
        auto issue = [&](int q0, int q1) {  // quads [q0, q1] of this pass
          for (int p = 4 * q0 + lane; p <= 4 * q1 + 3; p += 32) {
            uint64_t* bar = &sm.bars[(gq0 + (uint32_t)(p >> 2)) % NQ];
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
        };
        auto prefetch = [&]() {  // neighbour words for the next check (relaxed, one refill ahead)
          if (lane == 0 && nlo) pf_lo = ld_relaxed_gpu(nlo);
          if (lane == 0 && nhi) pf_hi = ld_relaxed_gpu(nhi);
        };
        int next_q = min(NQ, last_quad + 1);
        ensure(min(4 * next_q - 1, last_plane));
        issue(0, next_q - 1);
        prefetch();
        int cd = R;
        for (int s = 0; s < nsteps; ++s) {
          if (--cd == 0 || s == nsteps - 1) {
            cd = R;
            nbar_sync<NT + 32>(nbid);  // compute warps are done with steps <= s
            nbid ^= 1;
            const int to = min(s - 1 + NQ, last_quad);
            if (to >= next_q) {
              ensure(min(4 * to + 3, last_plane));
              issue(next_q, to);
              next_q = to + 1;
              prefetch();
            }
            // publish after the refill: the release fence waits for the CTA's
            // stores, the compute warps meanwhile march on the refilled quads
            if (s < nsteps - 1 && lane == 0) st_release_gpu(own, 1 + colour * kProgK + min(4 * s + 3, kProgK - 1));
          }
        }
        if (lane == 0) st_release_gpu(own, 1 + colour * kProgK + (kProgK - 1));  // pass complete
        gq = gq0 + (uint32_t)(last_quad + 1);
      }
  }
  } else {
  for (;;) {
    if (threadIdx.x == NT) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= total) break;
    const int64_t Tr = item / n_bands;
    const int64_t T = T0 + Tr;
    const int band = (stress & 1) ? n_bands - 1 - (int)(item - Tr * n_bands) : (int)(item - Tr * n_bands);
    const Band b = bands[band];
    const int last_plane = b.kmax + 1;
    const int last_quad = last_plane / 4;
    const int nsteps = (b.kmax + 4) / 4;
    double* const ub = u + T * S;
    Column q = make_column(b, N);
    double A[15], B[15];
    column_coeffs<OP>(coef10, cons, T, q.i, q.j, A, B);
    __syncthreads();  // roff / Cw of this item; every thread is past the previous item
      // ------------------------------------------------------ compute warps
      const double* const rc = sm.ring + q.o_c;
      const int d1 = q.d + 1;
      const unsigned lenu = q.active ? (unsigned)q.len : 0u;
      const double* const fb = f + T * S + q.c;
      double* const wb = ub + q.c;
      const int cwb = CWC ? __shfl_sync(0xffffffffu, (int)Tr, 0) * 15 : 0;
      auto Cw = [&](int w) { return CWC ? g_cC[cwb + w] : sm.Cw[w]; };
      auto wait_next = [&]() {
        mbar_wait_bounded(bar0 + 8u * (uint32_t)wslot, wph);
        if (++wslot == NQ) {
          wslot = 0;
          wph ^= 1u;
        }
      };
      for (int colour = 0; colour < 4; ++colour) {
        const int delta = (3 * ((((colour - q.d - q.j) % 4) + 4) % 4)) % 4;
        wait_next();  // quad 0
        double fq[FPD];
#pragma unroll
        for (int x = 0; x < FPD; ++x) {
          const int kk = 4 * x + delta;
          fq[x] = ((unsigned)(kk - 1) < lenu) ? __ldg(fb + (unsigned)sm.po[kk]) : 0.0;
        }
        int cd = R;
#pragma unroll(R)
        for (int s = 0; s < nsteps; ++s) {
          if (s + 1 <= last_quad) wait_next();
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
            const double* Pbh = Pb + d1;
            const double* Pmh = Pm + d1;
            const double* Pml = Pm - d1;
            const double* Ptl = Pt - d1;
            const double uu[15] = {Pb[0],  Pbh[0], Pbh[1], Pb[1],  Pml[0], Pm[-1], Pml[1], 0.0,
                                   Pmh[0], Pm[1],  Pmh[1], Pt[-1], Ptl[0], Ptl[1], Pt[0]};
            wb[(unsigned)sm.po[k]] = gs_node_value_acc<OP>(A, B, Cw, k, uu, fv);
          }
          if (--cd == 0 || s == nsteps - 1) {
            cd = R;
            __syncwarp();
            nbar_arrive<NT + 32>(nbid);
            nbid ^= 1;
          }
        }
        gq += (uint32_t)(last_quad + 1);
      }
  }
  }
}

}  // namespace hhg
