// Experimental single-pass 4-colour GS sweep (HHG_GS_KERNEL=wave).
//
// Inside a band the four colour passes run as one lagged wavefront: at step t
// the node of column (i, j) at plane p = t - 6c is updated, where c is the one
// colour with (i + 2j + 3p) mod 4 = c, i.e. c = 3 (i + 2j + 3t) mod 4 -- every
// column updates exactly one node per step, as in the apply.  With the lag of
// 6 planes per colour every lower-colour neighbour of a node is updated >= 5
// steps before it and every higher-colour neighbour >= 5 steps after it, so
// the in-place ring (updated by the compute threads) reproduces the
// colour-by-colour order exactly.
//
// Across bands: the values of the two neighbouring diagonals (owned by bands
// b-1, b+1) enter the ring by TMA (old values) and are refreshed from global
// memory 5 steps after the neighbour updated them (one node per halo column
// per step).  Every band publishes its completed step count; a band refreshes
// the neighbour's step-s updates only once the neighbour has published s + 1,
// which also keeps neighbours within 4 steps of each other (no write-after-read
// hazard on the TMA-loaded old values, which are loaded 6 steps ahead).
//
// Warp specialisation: warps 0-7 compute (one column per thread); warp 8 does
// the per-step synchronisation (ring refills, halo refresh, progress flags) and
// signals the compute warps through mbarriers, off their critical path.
#pragma once
#include "march.cuh"

namespace hhg {

constexpr int kWL = 6;           // colour lag in planes
constexpr int kWRing = 26;       // plane slots: planes t-20 .. t+5 live at step t
constexpr int kWPre = 5;         // plane t + 1 + kWPre issued at step t
constexpr int kWThreads = 288;   // 8 compute warps + 1 synchronisation warp
constexpr int kWHalo = 8;        // halo columns per sync lane (2 diagonals <= 256 columns)

// Bounded waits: a synchronisation bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ bool wave_wait_dbg(uint64_t* bar, uint32_t parity, int, int, int) {
  uint32_t ok = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return false;
    if (it > (1u << 26)) __trap();
  }
}

__device__ __forceinline__ bool wave_timeout(int, int, int, int, int) {
  __trap();
  return true;
}

__device__ __forceinline__ void wave_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (it > (1u << 26)) __trap();  // a bug, not a hang
  }
}

__device__ __forceinline__ int wave_colour(int i, int j, int t) { return (3 * ((i + 2 * j + 3 * t) & 3)) & 3; }

template <int OP>
__global__ void __launch_bounds__(kWThreads, 2)
    k_gs_wave(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
              const double* __restrict__ coef10, const double* __restrict__ cons, double* __restrict__ u,
              const double* __restrict__ f, int64_t ntl, int* __restrict__ counter, int* __restrict__ prog) {
  extern __shared__ __align__(16) double smem[];
  double* ring = smem;
  uint64_t* full = (uint64_t*)(ring + (size_t)kWRing * slot_len);
  uint64_t* ready = full + kWRing;
  uint64_t* done = ready + 2;
  double* Cw = (double*)(done + 2);
  int* po = (int*)(Cw + 16);
  __shared__ int s_item;
  const int64_t total = ntl * n_bands;
  const bool sync_warp = threadIdx.x >= 256;
  const int lane = threadIdx.x & 31;

  bool first_item = true;
  for (;; first_item = false) {
    if (threadIdx.x == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= total) break;
    const int64_t T = item / n_bands;
    const int bi = (int)(item - T * n_bands);
    const Band b = bands[bi];
    const int clo = b.c_lo;
    const int last_plane = b.kmax + 1;
    const int nsteps = b.kmax + 3 * kWL + 1;
    double* const ub = u + T * S;
    if (threadIdx.x < 15) Cw[threadIdx.x] = (OP == HHG_OP_SURROGATE) ? coef10[T * 150 + threadIdx.x * 10 + 9] : 0.0;
    for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) po[p] = (int)plane_off(N, p);
    if (threadIdx.x == 256) {
      if (!first_item) {  // a previous item used the barriers: invalidate before re-use
        for (int s = 0; s < kWRing + 4; ++s)
          asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
      }
      for (int s = 0; s < kWRing; ++s) mbar_init(&full[s], 1);
      mbar_init(&ready[0], 1);
      mbar_init(&ready[1], 1);
      mbar_init(&done[0], 8);
      mbar_init(&done[1], 8);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (sync_warp) {
      // ---------------- synchronisation warp ----------------
      auto issue = [&](int p) {  // plane p -> slot p % R (lane 0)
        if (lane == 0 && p <= last_plane) {
          const int g0 = po[p] + clo;
          const int a0 = g0 & ~1;
          const int a1 = (g0 + b.ncols + 1) & ~1;
          const uint32_t bytes = (uint32_t)((a1 - a0) * 8);
          uint64_t* bar = &full[p % kWRing];
          mbar_expect_tx(bar, bytes);
          tma_load_1d(ring + (p % kWRing) * slot_len, ub + a0, bytes, bar);
        }
      };
      // the previous item's generic ring writes before this item's bulk copies
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int p = 0; p <= kWPre; ++p) issue(p);  // then plane t + 1 + kWPre at step t
      // halo columns of this lane: interior columns of diagonals d0-1 (band b-1)
      // and d1 (band b+1)
      const int nlo = (bi > 0 && b.d0 - 1 >= 2) ? b.d0 - 2 : 0;
      const int nhi = (bi < n_bands - 1 && b.d1 <= N - 2) ? b.d1 - 1 : 0;
      const int* plo = prog + (T * n_bands + bi - 1);
      const int* phi = prog + (T * n_bands + bi + 1);
      // halo refresh: the neighbours' updates of their step t - 4 are loaded at
      // iteration t and written into the ring at iteration t + 1 (before step
      // t + 1, the first one that reads them)
      double pend_v[kWHalo];
      int pend_o[kWHalo];  // ring index (slot * slot_len + offset + shift), -1: none
#pragma unroll
      for (int h = 0; h < kWHalo; ++h) pend_o[h] = -1;
      int seen_lo = 0, seen_hi = 0;  // last observed neighbour progress
      for (int t = 0; t < nsteps; ++t) {
        if (t >= 1 && wave_wait_dbg(&done[(t - 1) & 1], ((t - 1) >> 1) & 1, 1, (int)item, t)) return;
#pragma unroll
        for (int h = 0; h < kWHalo; ++h)
          if (pend_o[h] >= 0) ring[pend_o[h]] = pend_v[h];
        __syncwarp();
        if (t == 0 && wave_wait_dbg(&full[0], 0, 2, (int)item, t)) return;
        if (t + 1 <= last_plane && wave_wait_dbg(&full[(t + 1) % kWRing], ((t + 1) / kWRing) & 1, 3, (int)item, t))
          return;
        if (lane == 0) mbar_arrive(&ready[t & 1]);
        // ---- work overlapping the compute of step t ----
        if (t >= 1 && lane == 0) st_release_gpu(prog + (T * n_bands + bi), t);  // steps 0..t-1 done
        issue(t + 1 + kWPre);  // its slot held plane t - 20, last read at step t - 1
        const int s = t + 1 - 5;
#pragma unroll
        for (int h = 0; h < kWHalo; ++h) pend_o[h] = -1;
        if (s >= 0 && nlo + nhi > 0) {
          if (nlo && seen_lo < s + 1) {
            for (uint32_t it = 0; (seen_lo = ld_acquire_gpu(plo)) < s + 1; ++it) {
              __nanosleep(64);
              if (it > (1u << 22) && wave_timeout(4, (int)item, t, seen_lo, s + 1)) return;
            }
          }
          if (nhi && seen_hi < s + 1) {
            for (uint32_t it = 0; (seen_hi = ld_acquire_gpu(phi)) < s + 1; ++it) {
              __nanosleep(64);
              if (it > (1u << 22) && wave_timeout(5, (int)item, t, seen_hi, s + 1)) return;
            }
          }
          __syncwarp();
#pragma unroll
          for (int h = 0; h < kWHalo; ++h) {
            const int x = lane + 32 * h;
            if (x >= nlo + nhi) continue;
            const int d = x < nlo ? b.d0 - 1 : b.d1;
            const int j = x < nlo ? x + 1 : x - nlo + 1;
            const int i = d - j;
            const int c = wave_colour(i, j, s);
            const int p = s - kWL * c;
            if (c > 2 || p < 1 || p > N - 1 - d) continue;  // colour-3 values are never read as new
            const int o = (int)col_idx(i, j) - clo;
            const int64_t gp = (int64_t)po[p] + col_idx(i, j);
            pend_v[h] = __ldcg(ub + gp);
            pend_o[h] = (p % kWRing) * slot_len + o + ((po[p] + clo) & 1);
          }
        }
      }
      if (wave_wait_dbg(&done[(nsteps - 1) & 1], ((nsteps - 1) >> 1) & 1, 7, (int)item, nsteps)) return;
      if (lane == 0) st_release_gpu(prog + (T * n_bands + bi), 1 << 30);  // done
      __syncwarp();
    } else {
      // ---------------- compute warps ----------------
      const Column q = make_column(b, N);
      double A[15], B[15];
      column_coeffs<OP>(coef10, cons, T, q.i, q.j, A, B);
      const double* fb = f + T * S + q.c;
      double* wb = ub + q.c;
      // f of the node of step t + 1, loaded one step ahead
      int c1 = wave_colour(q.i, q.j, 0), p1 = -kWL * c1;
      double fnext = (q.active && p1 >= 1 && p1 <= q.len) ? __ldg(fb + po[p1]) : 0.0;
      for (int t = 0; t < nsteps; ++t) {
        const int p = p1;
        const double fv = fnext;
        c1 = wave_colour(q.i, q.j, t + 1);
        p1 = t + 1 - kWL * c1;
        if (q.active && p1 >= 1 && p1 <= q.len) fnext = __ldg(fb + po[p1]);
        if (wave_wait_dbg(&ready[t & 1], (t >> 1) & 1, 6, (int)item, t)) return;
        if (q.active && p >= 1 && p <= q.len) {
          const double kd = (double)p;
          const double smc = (OP == HHG_OP_SURROGATE) ? fma(fma(Cw[kMC], kd, B[kMC]), kd, A[kMC]) : A[kMC];
          const double rinv = rcp_nr(smc);
          const double* Pb = ring + ((p - 1) % kWRing) * slot_len + ((po[p - 1] + clo) & 1);
          double* Pm = ring + (p % kWRing) * slot_len + ((po[p] + clo) & 1);
          const double* Pt = ring + ((p + 1) % kWRing) * slot_len + ((po[p + 1] + clo) & 1);
          const double uu[15] = {Pb[q.o_c],  Pb[q.o_e],  Pb[q.o_n],  Pb[q.o_nw], Pm[q.o_s],
                                 Pm[q.o_se], Pm[q.o_w],  0.0,        Pm[q.o_e],  Pm[q.o_nw],
                                 Pm[q.o_n],  Pt[q.o_se], Pt[q.o_s],  Pt[q.o_w],  Pt[q.o_c]};
          double r;
          if (OP == HHG_OP_SURROGATE) {
            double x = 0.0, y = 0.0, z = 0.0;
#pragma unroll
            for (int w = 0; w < 15; ++w) {
              if (w == kMC) continue;
              x = fma(A[w], uu[w], x);
              y = fma(B[w], uu[w], y);
              z = fma(Cw[w], uu[w], z);
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
          const double nv = (fv - r) * rinv;
          Pm[q.o_c] = nv;
          wb[po[p]] = nv;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[t & 1]);
      }
    }
    __syncthreads();  // item done: ring and barriers are re-initialised for the next one
  }
}

}  // namespace hhg
