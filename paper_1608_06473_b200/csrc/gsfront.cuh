// Single-pass 4-colour volume GS: a lagged colour wavefront per band, one
// node per thread per step, bands coupled through flag-carrying ("LL") halo
// words in global memory -- no fences, no colour passes.
//
// Semantics (R13/R14; eq. iteration-scheme):
// the volume step of the hybrid GS updates colour 0 = (i+2j+3k) mod 4 nodes
// from the values before it, then colour 1, 2, 3.  Colour c at plane k is
// processed at wavefront time t = k + LAG c.  A colour-c node reads its 14
// neighbours in planes k-1..k+1; a neighbour of colour c' < c was updated at
// t' = k' + LAG c' <= t - (LAG - 1), one of colour c' > c is updated at
// t' >= t + (LAG - 1): with LAG >= 2 every read sees exactly the value the
// sequential colour order gives (the node arithmetic is gs_node_value, the
// same as the colour-pass kernels', so the sweep is bit-identical to them).
// For LAG even, (i + 2j + 3t) fixes ONE colour per lattice column and step,
// so every thread (= lattice column) updates one node per step, like the
// apply march.
//
// A CTA owns a band of diagonals [d0, d1) of one macro (march.cuh layout);
// its planes arrive by 1-D TMA bulk copies into a RING-slot shared-memory
// ring (halo diagonals d0-1 and d1 included) and are updated in place.  The
// halo diagonals belong to the neighbour bands: their new values come from
// the neighbour's LL words -- every node on a band's boundary diagonal is
// also stored as {lo32 | tag, hi32 | tag} (tag = the sweep epoch; 8-byte
// halves are single-copy atomic), and the reader polls until both tags
// match.  A halo node updated at neighbour time t_X is patched into the ring
// at this band's step t_X + DELTA, DELTA = LAG - 2: after its last old-value
// read (<= t_X - LAG + 1) and before its first new-value read
// (>= t_X + LAG - 1).  Plane p is written back to HBM at step p + 3 LAG + 1
// (every node of it final, its slot refilled after that step), and only
// after both neighbour bands have loaded plane p (their progress words) --
// the neighbours read the pre-sweep halo from HBM.  Items (macro, band) come
// from an atomic counter, macro-major; all bands of a macro progress
// together (deadlock-free while the grid holds more CTAs than a macro has
// bands: only the last handed-out macro can wait on a band not yet running).
#pragma once
#include "march.cuh"

namespace hhg {

__device__ __forceinline__ void ll_store(uint64_t* p, double v, uint32_t tag) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const uint64_t w0 = (b & 0xffffffffull) | ((uint64_t)tag << 32);
  const uint64_t w1 = (b >> 32) | ((uint64_t)tag << 32);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}

__device__ __forceinline__ void ll_load_raw(const uint64_t* p, uint64_t& w0, uint64_t& w1) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}

__device__ __forceinline__ bool ll_ready(uint64_t w0, uint64_t w1, uint32_t tag) {
  return (uint32_t)(w0 >> 32) == tag && (uint32_t)(w1 >> 32) == tag;
}

__device__ __forceinline__ double ll_value(uint64_t w0, uint64_t w1) {
  return __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32)));
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// progress word of a band: (epoch << 12) | completed steps; kFrontDone = finished
constexpr uint32_t kFrontDone = 0xfff;

// Colour processed by column (i,j) at wavefront time t: (i + 2j + 3k) = c
// (mod 4) with k = t - LAG c  <=>  c (1 + 3 LAG) = i + 2j + 3t (mod 4); for
// LAG even, 1 + 3 LAG is 1 (LAG = 0 mod 4) or 3 (LAG = 2 mod 4), its own
// inverse mod 4.
template <int LAG>
__device__ __forceinline__ int front_colour(int i, int j, int t) {  // (i, j) may be (i + 2j, 0)
  const int m = (LAG % 4 == 0) ? 1 : 3;
  return (m * (i + 2 * j + 3 * t)) & 3;
}

#ifndef HHG_FRONT_FD
#define HHG_FRONT_FD 3
#endif
constexpr int kFrontFD = HHG_FRONT_FD;  // f prefetch distance (steps)
constexpr int kFrontFS = kFrontFD < 4 ? 4 : 8;  // cp.async ring slots (power of 2 > FD: the slot
                                                  // refilled at a step is never the one read at it)

template <int RING, int NT>
__host__ __device__ inline size_t front_smem_bytes(int slot_len, int N) {
  return (size_t)RING * slot_len * 8 + RING * 8 + 16 * 8 + (size_t)kFrontFS * NT * 8 + 8 * 8 +
         (size_t)2 * (N + 2) * 4 + 16;
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Per-item state, uniform across the CTA (shared memory: keeps it out of the
// 128 registers the column needs -- A_w, B_w alone take 60).
struct FrontItem {
  int64_t TS;                // macro block offset T * S
  const uint32_t* prog_lo;   // neighbour bands' progress words (nullptr: none)
  const uint32_t* prog_hi;
  uint32_t* my_prog;
  int last_plane, last_lo, last_hi, clo, ncols, tend;
  uint32_t known_lo, known_hi;  // thread 0: neighbour progress seen so far
  uint32_t seqbase;             // planes issued by this CTA before this item
  int next_issue;
};

template <int OP, int LAG, int RING, int NT, bool PROF>
__global__ void __launch_bounds__(NT, 512 / NT)
    k_gs_front(int N, int64_t S, const Band* __restrict__ bands, int n_bands, int slot_len,
               const double* __restrict__ coef10, const double* __restrict__ cons, double* __restrict__ u,
               const double* __restrict__ f, int64_t ntl, int* __restrict__ counter,
               const uint32_t* __restrict__ epoch_ptr, uint32_t* __restrict__ prog, uint64_t* __restrict__ ex,
               unsigned long long* __restrict__ gprof, int stress) {
  static_assert(LAG % 2 == 0 && LAG >= 4, "LAG even, >= 4 (DELTA = LAG - 2 >= 2 steps of slack)");
  // plane t + 1 + DELTA is waited at step t and issued at the end of step
  // t + 1 + DELTA - RING + 3 LAG + 1: at least one step earlier
  static_assert(RING >= 4 * LAG + 2, "ring too short for the wavefront window");
  constexpr int DELTA = LAG - 2;
  constexpr int FD = kFrontFD;
  constexpr int FS = kFrontFS;
  extern __shared__ __align__(16) double smem[];
  double* ring = smem;
  uint64_t* bars = (uint64_t*)(ring + RING * slot_len);
  double* Cw = (double*)(bars + RING);
  double* fbuf = Cw + 16;                                                  // [FS][NT]
  unsigned long long* spf = (unsigned long long*)(fbuf + FS * NT);  // [8] profiling
  int* po = (int*)(spf + 8);
  int* roff = po + (N + 2);
  __shared__ FrontItem it;
  __shared__ int s_item;
  const uint32_t epoch = *epoch_ptr;
  const uint32_t ptag = (epoch & 0xfffff) << 12;
  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    it.seqbase = 0;
  }
  if (PROF && threadIdx.x < 8) spf[threadIdx.x] = 0;
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) po[p] = (int)plane_off(N, p);
  // optional cycle accounting (PROF; tools/gsprof.py): thread 0's time per phase of a step
  long long tp = 0;
  auto mark = [&](int x) {
    if (PROF && threadIdx.x == 0) {
      const long long now = clock64();
      spf[x] += (unsigned long long)(now - tp);
      tp = now;
    }
  };
  unsigned fails = 0;
  auto issue = [&](int p) {  // bulk copy of plane p into its ring slot (one thread)
    const uint32_t sq = it.seqbase + p;
    const int g0 = po[p] + it.clo;
    const int a0 = g0 & ~1;
    const int a1 = (g0 + it.ncols + 1) & ~1;
    const uint32_t bytes = (uint32_t)((a1 - a0) * 8);
    mbar_expect_tx(&bars[sq % RING], bytes);
    tma_load_1d(ring + (sq % RING) * slot_len, u + it.TS + a0, bytes, &bars[sq % RING]);
  };
  auto wait_plane = [&](int p) {
    const uint32_t sq = it.seqbase + p;
    mbar_wait(&bars[sq % RING], (sq / RING) & 1);
  };
  const int64_t total = ntl * n_bands;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= total) break;
    const int64_t T = item / n_bands;
    // stress test (HHG_GS_STRESS): bands of a macro in reverse order, random delays
    const int band = (stress & 1) ? n_bands - 1 - (int)(item - T * n_bands) : (int)(item - T * n_bands);
    const Band b = bands[band];
    if (threadIdx.x == 0) {
      it.TS = T * S;
      it.prog_lo = band > 0 ? prog + T * n_bands + band - 1 : nullptr;
      it.prog_hi = band + 1 < n_bands ? prog + T * n_bands + band + 1 : nullptr;
      it.my_prog = prog + T * n_bands + band;
      it.last_plane = b.kmax + 1;
      it.last_lo = band > 0 ? bands[band - 1].kmax + 1 : 0;
      it.last_hi = band + 1 < n_bands ? bands[band + 1].kmax + 1 : 0;
      it.clo = b.c_lo;
      it.ncols = b.ncols;
      it.tend = b.kmax + 3 * LAG + 1;
      it.known_lo = band > 0 ? 0u : kFrontDone;
      it.known_hi = band + 1 < n_bands ? 0u : kFrontDone;
      it.next_issue = min(RING - 1, b.kmax + 1) + 1;
    }
    if (threadIdx.x < 15) Cw[threadIdx.x] = (OP == HHG_OP_SURROGATE) ? coef10[T * 150 + threadIdx.x * 10 + 9] : 0.0;
    __syncthreads();
    for (int p = threadIdx.x; p <= it.last_plane; p += blockDim.x)
      roff[p] = (int)((it.seqbase + p) % RING) * slot_len + ((po[p] + it.clo) & 1);
    // first RING planes in flight (every slot is free: the previous item consumed all it issued)
    if ((int)threadIdx.x < it.next_issue) issue(threadIdx.x);
    if (threadIdx.x == 0) st_volatile_u32(it.my_prog, ptag | 0u);
    // this thread's column (overlaps the first bulk copies)
    const Column q = make_column(b, N);
    double A[15], B[15];
    column_coeffs<OP>(coef10, cons, T, q.i, q.j, A, B);
    const int csum = q.i + 2 * q.j;   // colour of (i,j,k) = (csum + 3k) & 3
    const bool pub = q.active && ((q.d == b.d0 && band > 0) || (q.d == b.d1 - 1 && band + 1 < n_bands));
    const int o_c = q.c - b.c_lo;     // ring offset of this column; neighbours at o_c + {+-1, d+1, d+2, -d, -d-1}
    const int dd = q.d;
    double* const fslot = fbuf + threadIdx.x;
    // halo patch job: one interior column of diagonal d0-1 or d1
    int h_sum = 0, h_len = -1, h_col = 0;
    {
      const int x = threadIdx.x;
      const int n_lo = band > 0 ? b.d0 - 2 : 0;
      const int n_hi = band + 1 < n_bands ? b.d1 - 1 : 0;
      int hi_ = 0, hj = 0;
      if (x < n_lo) {
        hj = x + 1;
        hi_ = b.d0 - 1 - hj;
      } else if (x < n_lo + n_hi) {
        hj = x - n_lo + 1;
        hi_ = b.d1 - hj;
      }
      if (x < n_lo + n_hi) {
        h_len = N - 1 - (hi_ + hj);
        h_col = (int)col_idx(hi_, hj);
        h_sum = hi_ + 2 * hj;
      }
    }
    // f of this column's node at step t: cp.async into fbuf[t % FS] at step t - FD
    // (one commit group per step; a register shift ring would stall on the loads)
#pragma unroll
    for (int x = 0; x < FD; ++x) {
      const int tt = 1 + x;
      const int kk = tt - LAG * front_colour<LAG>(csum, 0, tt);
      if (q.active && kk >= 1 && kk <= q.len) cp_async8(fslot + (tt & (FS - 1)) * NT, f + it.TS + q.c + po[kk]);
      cp_async_commit();
    }
    for (int p = 0; p <= min(1 + DELTA, it.last_plane); ++p) wait_plane(p);
    if (PROF && threadIdx.x == 0) tp = clock64();
    const int tend = it.tend;
    for (int t = 1; t <= tend; ++t) {
      mark(5);
      // halo patch: the neighbour's node updated at its step t - DELTA (new value
      // needed from step t - DELTA + LAG - 1 = t + 1 on; colour 3 is read by no
      // one).  Issued first: it is the step's longest-latency load.
      int hk = -1;
      uint64_t h0 = 0, h1 = 0;
      if (h_len > 0) {
        const int tt = t - DELTA;
        const int c = front_colour<LAG>(h_sum, 0, tt);
        const int kk = tt - LAG * c;
        if (c < 3 && kk >= 1 && kk <= h_len) {
          hk = kk;
          ll_load_raw(ex + 2 * (it.TS + h_col + po[kk]), h0, h1);
        }
      }
      // planes <= t + 1 + DELTA present (the neighbours' write-back waits on this, see below)
      if (t + 1 + DELTA <= it.last_plane) wait_plane(t + 1 + DELTA);
      mark(0);
      // f of this step's node (its cp.async group landed; waited before the
      // halo and progress loads are issued, so the wait does not cover them)
      const int k = t - LAG * front_colour<LAG>(csum, 0, t);
      const bool mine = q.active && k >= 1 && k <= q.len;
      cp_async_wait<FD - 1>();
      const double fv = mine ? fslot[(t & (FS - 1)) * NT] : 0.0;
      {
        const int tt = t + FD;
        const int kk = tt - LAG * front_colour<LAG>(csum, 0, tt);
        if (q.active && kk >= 1 && kk <= q.len)
          cp_async8(fslot + (tt & (FS - 1)) * NT, f + it.TS + q.c + po[kk]);
        cp_async_commit();
      }
      // thread 0: the next step writes back plane pn = t - 3 LAG; a neighbour
      // that loads pn must have completed step pn - 1 - DELTA (it waits for
      // planes <= step + 1 + DELTA at each step).  The progress words are
      // re-read (issued here, consumed after the node update: the L2 latency
      // hides behind it) only when the known value gets within 8 steps of the need.
      const int pn = t - 3 * LAG;
      uint32_t r_lo = 0, r_hi = 0;
      bool rd_lo = false, rd_hi = false;
      if (threadIdx.x == 0 && pn >= 1) {
        const uint32_t need = (uint32_t)max(pn - 1 - DELTA, 0);
        rd_lo = pn <= it.last_lo && it.known_lo < need + 8;
        rd_hi = pn <= it.last_hi && it.known_hi < need + 8;
        if (rd_lo) r_lo = ld_volatile_u32(it.prog_lo);
        if (rd_hi) r_hi = ld_volatile_u32(it.prog_hi);
      }
      // this column's node
      if (mine) {
        const double* Pb = ring + roff[k - 1] + o_c;
        double* Pm = ring + roff[k] + o_c;
        const double* Pt = ring + roff[k + 1] + o_c;
        const double* Pbe = Pb + dd + 1;  // (i+1, j) and (i, j+1)
        const double* Pme = Pm + dd + 1;
        const double* Pmw = Pm - dd;      // (i-1, j) and (i, j-1)
        const double* Ptw = Pt - dd;
        const double uu[15] = {Pb[0],  Pbe[0], Pbe[1], Pb[1],  Pmw[-1], Pm[-1], Pmw[0], 0.0,
                               Pme[0], Pm[1],  Pme[1], Pt[-1], Ptw[-1], Ptw[0], Pt[0]};
        const double v = gs_node_value<OP>(A, B, Cw, k, uu, fv);
        Pm[0] = v;
        if (pub) ll_store(ex + 2 * (it.TS + q.c + po[k]), v, epoch);
      }
      mark(1);
      if (hk >= 0) {
        for (long long spin = 0; !ll_ready(h0, h1, epoch); ++spin) {
          if (spin > kSpinLimit) __trap();
          if (PROF) ++fails;
          ll_load_raw(ex + 2 * (it.TS + h_col + po[hk]), h0, h1);
        }
        ring[roff[hk] + h_col - it.clo] = ll_value(h0, h1);
      }
      // write-back of plane t - 3 LAG - 1 (final since step t - 1); the
      // neighbours loaded it (checked by thread 0 at the previous step)
      {
        const int p = t - 3 * LAG - 1;
        if (q.active && p >= 1 && p <= q.len) u[it.TS + po[p] + q.c] = ring[roff[p] + o_c];
      }
      mark(2);
      if (threadIdx.x == 0 && pn >= 1) {
        const uint32_t need = (uint32_t)max(pn - 1 - DELTA, 0);
        auto decode = [&](uint32_t v) -> uint32_t { return (v & ~0xfffu) == ptag ? (v & 0xfffu) : 0u; };
        uint32_t klo = it.known_lo, khi = it.known_hi;
        if (rd_lo) klo = max(klo, decode(r_lo));
        if (rd_hi) khi = max(khi, decode(r_hi));
        for (long long spin = 0; pn <= it.last_lo && klo < need; ++spin) {
          if (spin > kSpinLimit) __trap();
          klo = max(klo, decode(ld_volatile_u32(it.prog_lo)));
        }
        for (long long spin = 0; pn <= it.last_hi && khi < need; ++spin) {
          if (spin > kSpinLimit) __trap();
          khi = max(khi, decode(ld_volatile_u32(it.prog_hi)));
        }
        it.known_lo = klo;
        it.known_hi = khi;
      }
      if (stress) {
        const uint32_t h = stress_hash(stress, (uint32_t)(it.TS + t), threadIdx.x);
        if ((h & 63) == 0) __nanosleep((h >> 8) & 4095);
      }
      mark(3);
      __syncthreads();
      mark(4);
      if (threadIdx.x == 0) {
        st_volatile_u32(it.my_prog, ptag | (uint32_t)t);
        // refill the slot of the plane written back at this step
        const int p = t + RING - 3 * LAG - 1;
        if (p >= it.next_issue && p <= it.last_plane) {
#ifdef HHG_FRONT_PROXY_FENCE
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
          issue(p);
          it.next_issue = p + 1;
        }
      }
    }
    cp_async_wait<0>();  // no copy in flight into fbuf across items
    __syncthreads();
    if (threadIdx.x == 0) {
      st_volatile_u32(it.my_prog, ptag | kFrontDone);
      it.seqbase += (uint32_t)(it.last_plane + 1);
      if (PROF) spf[6] += (unsigned long long)tend, spf[7] += 1;
    }
  }
  if (PROF) {
    if (fails) atomicAdd(&gprof[8], (unsigned long long)fails);
    if (threadIdx.x == 0)
      for (int x = 0; x < 8; ++x) atomicAdd(&gprof[x], spf[x]);
  }
}

// counter <- 0, epoch <- epoch + 1 (device-side, so a captured graph replays correctly)
__global__ void k_front_begin(int* counter, uint32_t* epoch) {
  *counter = 0;
  uint32_t e = *epoch + 1;
  if ((e & 0xfffff) == 0) e += 1;  // the progress words carry 20 bits of it; 0 = never written
  *epoch = e;
}

}  // namespace hhg
