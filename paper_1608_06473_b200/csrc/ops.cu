// Operator entry points: apply, residual, multicolour GS, gather/scatter,
// stencil export.  Baseline ("v1") volume kernels: one thread per lattice node.
//
// PAPER.md:618-636 (L~: volume rows from the surrogate, lower primitives from
// exact FEM), PAPER.md:654-657 (15 polynomials evaluated per node),
// PAPER.md:862-871 (residual), PAPER.md:1306-1315 (eq. iteration-scheme:
// u_I = (f_I - sum_{w != mc} s_w u_{I_w}) / s_mc).
#include <cstring>
#include <map>

#include "fem_device.cuh"
#include "hhg_internal.h"
#include "vol_kernels.cuh"
#include "march.cuh"
#include "gsfront.cuh"
#include "gsprod.cuh"
#include "gslex.cuh"
#include "femew.cuh"

namespace hhg {

// ---------------------------------------------------------------------------
// Lower-primitive rows (stored exact FEM rows, CSR; entry 0 = centre)
// ---------------------------------------------------------------------------
__global__ void k_lp_apply(int64_t r0, int64_t r1, const uint64_t* __restrict__ rp,
                           const uint32_t* __restrict__ col, const double* __restrict__ val,
                           const uint64_t* __restrict__ cp, const uint32_t* __restrict__ copy,
                           const double* __restrict__ u, const double* __restrict__ f,
                           double* __restrict__ out, int mode) {
  int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= r1) return;
  double acc = 0.0;
  const uint64_t e0 = rp[r], e1 = rp[r + 1];
  for (uint64_t e = e0; e < e1; ++e) acc += val[e] * u[col[e]];
  double res = mode == kModeResid ? f[col[e0]] - acc : acc;
  for (uint64_t c = cp[r]; c < cp[r + 1]; ++c) out[copy[c]] = res;
}

__global__ void k_lp_gs_compute(int64_t r0, int64_t r1, const uint64_t* __restrict__ rp,
                                const uint32_t* __restrict__ col, const double* __restrict__ val,
                                const double* __restrict__ u, const double* __restrict__ f,
                                double* __restrict__ tmp) {
  int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= r1) return;
  const uint64_t e0 = rp[r], e1 = rp[r + 1];
  double acc = f[col[e0]];
  for (uint64_t e = e0 + 1; e < e1; ++e) acc -= val[e] * u[col[e]];
  tmp[r] = acc / val[e0];
}

__global__ void k_lp_write(int64_t r0, int64_t r1, const uint64_t* __restrict__ cp,
                           const uint32_t* __restrict__ copy, const double* __restrict__ tmp,
                           double* __restrict__ u) {
  int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= r1) return;
  double v = tmp[r];
  for (uint64_t c = cp[r]; c < cp[r + 1]; ++c) u[copy[c]] = v;
}

__global__ void k_lp_sync(int64_t n_rows, const uint64_t* __restrict__ cp,
                          const uint32_t* __restrict__ copy, double* __restrict__ u) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  uint64_t c0 = cp[r];
  double v = u[copy[c0]];
  for (uint64_t c = c0 + 1; c < cp[r + 1]; ++c) u[copy[c]] = v;
}

__global__ void k_zero_slots(int64_t n, const uint32_t* __restrict__ slots, double* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) out[slots[t]] = 0.0;
}

// gather / scatter ------------------------------------------------------------
__global__ void k_vol_gather(int N, int64_t S, int64_t P, const MacroTopo* __restrict__ topo,
                             GidInfo gi, const double* __restrict__ local, double* __restrict__ glob,
                             int dir) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t T = blockIdx.y;
  if (p >= P) return;
  int i, j, k;
  decode_pos(N, p, i, j, k);
  if (i < 1 || j < 1 || k < 1 || i + j + k > N - 1) return;
  int64_t g = gi.base_v + topo[T].gT * gi.nvi + vol_index(N, i, j, k);
  if (dir == 0) glob[g] = local[T * S + p];
  else ((double*)local)[T * S + p] = glob[g];
}

__global__ void k_lp_gather(int64_t n_rows, const uint64_t* __restrict__ cp,
                            const uint32_t* __restrict__ copy, const int64_t* __restrict__ gid,
                            const double* __restrict__ local, double* __restrict__ glob, int dir) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  if (dir == 0) {
    glob[gid[r]] = local[copy[cp[r]]];
  } else {
    double v = glob[gid[r]];
    for (uint64_t c = cp[r]; c < cp[r + 1]; ++c) ((double*)local)[copy[c]] = v;
  }
}

// sum of squares over unique unknowns (fixed grid => deterministic) ----------
constexpr int kRedBlocks = 1184;
__device__ inline double block_sum(double v) {
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  }
  return v;
}

// sum over unique unknowns of a*b: volume interiors + CSR rows at their owner
// copy (face rows: faces.cu::k_face_dot)
// sum over the interior volume nodes (column march: thread = (macro, lattice
// column (i, j)), k = 1 .. N-1-i-j; consecutive threads read consecutive
// columns of a plane) and the owned lower-primitive rows.  Fixed grid and
// mapping: deterministic.
__global__ void k_dot(int N, int64_t S, int64_t P, int64_t ntl, const double* __restrict__ a,
                      const double* __restrict__ b, int64_t n_rows, const uint32_t* __restrict__ lp_owner_col,
                      const uint64_t* __restrict__ rp, double* __restrict__ part) {
  __shared__ int64_t po_s[258];
  for (int k = threadIdx.x; k <= N; k += blockDim.x) po_s[k] = plane_off(N, k);
  __syncthreads();
  (void)P;
  double acc = 0.0;
  const int64_t ncol = (int64_t)(N + 1) * (N + 2) / 2;  // columns of plane 0
  const int64_t tot = ntl * ncol;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t T = t / ncol;
    const int c = (int)(t - T * ncol);
    int d = (int)((sqrt(8.0 * (double)c + 1.0) - 1.0) * 0.5);
    while ((d + 1) * (d + 2) / 2 <= c) ++d;
    while (d * (d + 1) / 2 > c) --d;
    const int j = c - d * (d + 1) / 2, i = d - j;
    if (i < 1 || j < 1) continue;
    const double* pa = a + T * S + c;
    const double* pb = b + T * S + c;
    for (int k = 1; k <= N - 1 - d; ++k) acc = fma(pa[po_s[k]], pb[po_s[k]], acc);
  }
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_rows;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t s = lp_owner_col[rp[q]];
    acc += a[s] * b[s];
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// CSR rows: every copy <- sum of all copies (ascending macro order)
__global__ void k_lp_sumcopies(int64_t n_rows, const uint64_t* __restrict__ cp, const uint32_t* __restrict__ copy,
                               double* __restrict__ v) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  double s = 0.0;
  for (uint64_t c = cp[r]; c < cp[r + 1]; ++c) s += v[copy[c]];
  for (uint64_t c = cp[r]; c < cp[r + 1]; ++c) v[copy[c]] = s;
}

__global__ void k_final_sum(const double* __restrict__ part, int n, double* __restrict__ out) {
  double acc = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) acc += part[t];
  acc = block_sum(acc);
  if (threadIdx.x == 0) out[0] = acc;
}

// eval stencils export ---------------------------------------------------------
__global__ void k_eval_stencils(int N, int64_t P, const double* __restrict__ geo,
                                const double* __restrict__ coef, int mq, const double* __restrict__ cons,
                                int op, bool blended, double* __restrict__ out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  int i, j, k;
  decode_pos(N, p, i, j, k);
  if (i < 1 || j < 1 || k < 1 || i + j + k > N - 1) return;
  double s[15];
  node_weights(op, N, i, j, k, geo, coef, mq, cons, blended, s);
  int64_t idx = vol_index(N, i, j, k);
  for (int w = 0; w < 15; ++w) out[idx * 15 + w] = s[w];
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct Staged {
  double* dev = nullptr;
  const void* host = nullptr;
  bool staged = false;
};

static hhg_status stage(Ctx* c, int slot, const void* p, int64_t n, bool copy_in, Staged& s) {
  s.host = p;
  if (is_device_ptr(p)) {
    s.dev = (double*)p;
    s.staged = false;
    return HHG_OK;
  }
  if (c->stage_n < n) {
    for (auto*& b : c->d_stage)
      if (b) { cudaFree(b); b = nullptr; }
    c->stage_n = n;
  }
  if (!c->d_stage[slot]) HHG_CK(c, cudaMalloc(&c->d_stage[slot], c->stage_n * sizeof(double)));
  s.dev = c->d_stage[slot];
  s.staged = true;
  if (copy_in)
    HHG_CK(c, cudaMemcpyAsync(s.dev, p, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  return HHG_OK;
}

static hhg_status unstage(Ctx* c, Staged& s, int64_t n) {
  if (!s.staged) return HHG_OK;
  HHG_CK(c, cudaMemcpyAsync((void*)s.host, s.dev, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  { hhg_status st_sync__ = ctx_sync(c); if (st_sync__ != HHG_OK) return st_sync__; }
  return HHG_OK;
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// The GS update divides by the centre weight (eq. iteration-scheme,
// PAPER.md:1306-1315): a level whose fitted surrogate has a non-positive
// centre weight somewhere (hhg_fit_surrogates' check) cannot be smoothed.
hhg_status check_centre_ok(Ctx* c, const Level& lv, int op) {
  if ((op == HHG_OP_SURROGATE || op == HHG_OP_SURROGATE_FACES) && lv.centre_bad)
    return set_err(c, HHG_ERR_NUMERIC, "non-positive surrogate centre weight on level " + std::to_string(lv.L));
  if (op == HHG_OP_SURROGATE_FACES && lv.fcentre_bad)
    return set_err(c, HHG_ERR_NUMERIC, "non-positive face-surrogate centre weight on level " + std::to_string(lv.L));
  return HHG_OK;
}

static hhg_status check_call(Ctx* c, int L, int op, bool smoother) {
  if (!c) return HHG_ERR_INVALID;
  if (c->poisoned) return HHG_ERR_CUDA;
  if (c->host_only) return set_err(c, HHG_ERR_STATE, "plan-only context (hhg_set_host_transport host_only)");
  if (L < 2 || L > c->L_max) return set_err(c, HHG_ERR_INVALID, "L out of range");
  if (op < 0 || op > 3) return set_err(c, HHG_ERR_INVALID, "bad op");
  const Level& lv = c->levels[L];
  if ((op == HHG_OP_SURROGATE || op == HHG_OP_SURROGATE_FACES) && !lv.fitted)
    return set_err(c, HHG_ERR_STATE, "hhg_fit_surrogates must be called before using the surrogate operator");
  if (op == HHG_OP_SURROGATE_FACES && L >= 3 && lv.n_flp > 0 && !lv.d_fcoef)
    return set_err(c, HHG_ERR_STATE, "no face surrogates on this level (fitted from planted samples)");
  return smoother ? check_centre_ok(c, lv, op) : HHG_OK;
}

// Per-macro k^2 coefficients C_w (coefficient 9 of each weight polynomial),
// contiguous [T][15], the source of the constant-memory chunks (g_cC).
static hhg_status ensure_cC(Ctx* c, Level& lv, int op) {
  if (op != HHG_OP_SURROGATE || lv.d_cC) return HHG_OK;
  HHG_CK(c, cudaMalloc(&lv.d_cC, (size_t)c->nt_local * 15 * sizeof(double)));
  HHG_CK(c, cudaMemcpy2DAsync(lv.d_cC, sizeof(double), lv.d_coef10 + 9, 10 * sizeof(double), sizeof(double),
                              (size_t)c->nt_local * 15, cudaMemcpyDeviceToDevice, c->stream));
  return HHG_OK;
}

// Opt-in dynamic shared memory for a kernel, once per context (a context is
// bound to one device; the attribute is per device).
static hhg_status smem_attr(Ctx* c, const void* fn) {
  if (c->smem_attr_done.count(fn)) return HHG_OK;
  HHG_CK(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  c->smem_attr_done.insert(fn);
  return HHG_OK;
}

// Co-resident grid of a persistent kernel (SMs x resident CTAs per SM), per
// context and (kernel, dynamic shared memory).
static hhg_status resident_grid(Ctx* c, const void* fn, int threads, size_t smem, int& grid) {
  auto key = std::make_pair(fn, smem);
  auto it = c->grid_cache.find(key);
  if (it != c->grid_cache.end()) {
    grid = it->second;
    return HHG_OK;
  }
  int dev = 0, sms = 0, per_sm = 0;
  HHG_CK(c, cudaGetDevice(&dev));
  HHG_CK(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  HHG_CK(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  grid = sms * per_sm;
  c->grid_cache[key] = grid;
  return HHG_OK;
}

template <int OP, int MODE>
static hhg_status launch_march(Ctx* c, Level& lv, const double* u, const double* f, double* out, int64_t Tb,
                               int64_t Te) {
  const size_t smem = march_smem_bytes(lv.slot_len, lv.N);
  hhg_status st = smem_attr(c, (const void*)k_vol_march<OP, MODE>);
  if (st != HHG_OK) return st;
  const int nb = (int)lv.bands.size();
  if ((st = ensure_cC(c, lv, OP)) != HHG_OK) return st;
  ProfScope ps(c, 0);
  for (int64_t T0 = Tb; T0 < Te; T0 += kCMax) {
    const int64_t nt = std::min<int64_t>(kCMax, Te - T0);
    if (OP == HHG_OP_SURROGATE)
      HHG_CK(c, cudaMemcpyToSymbolAsync(g_cC, lv.d_cC + T0 * 15, nt * 15 * sizeof(double), 0,
                                        cudaMemcpyDeviceToDevice, c->stream));
    k_vol_march<OP, MODE><<<dim3((unsigned)nb, (unsigned)nt), kMarchThreads, smem, c->stream>>>(
        lv.N, lv.S, lv.d_bands, nb, lv.slot_len, lv.d_coef10, lv.d_cons, u, f, out, (int)T0);
    HHG_LAUNCHED(c);
  }
  return HHG_OK;
}

// One GS colour pass over every band (the fallback of the persistent sweep).
template <int OP>
static hhg_status launch_gs_march(Ctx* c, Level& lv, int colour, double* u, const double* f, int64_t Tb,
                                  int64_t Te) {
  const size_t smem = march_smem_bytes(lv.slot_len, lv.N);
  hhg_status st = smem_attr(c, (const void*)k_gs_march<OP>);
  if (st != HHG_OK) return st;
  const int nb = (int)lv.bands.size();
  ProfScope ps(c, 1);
  if (Te <= Tb) return HHG_OK;
  k_gs_march<OP><<<(unsigned)(nb * (Te - Tb)), kMarchThreads, smem, c->stream>>>(
      lv.N, lv.S, lv.d_bands, nb, lv.slot_len, lv.d_coef10, lv.d_cons, colour, u, f, Tb);
  HHG_LAUNCHED(c);
  return HHG_OK;
}

// HHG_OVERLAP=0 (read per call): no exchange / interior-compute overlap on multi-rank
static bool overlap_on() {
  const char* e = getenv("HHG_OVERLAP");
  return !(e && atoi(e) == 0);
}

// HHG_GS_STRESS=<seed> (tests): the persistent GS kernels hand out the bands of
// a macro in reverse order and insert random delays (read per call).
static int gs_stress() {
  const char* e = getenv("HHG_GS_STRESS");
  return e ? atoi(e) : 0;
}

// The whole volume GS (4 colours) as one persistent launch (march.cuh::k_gs_items).
template <int OP, int RING>
static hhg_status launch_gs_items_r(Ctx* c, Level& lv, double* u, const double* f, int64_t Tb, int64_t Te) {
  constexpr int NT = kMarchThreads;
  // HHG_GS_CW=smem: C_w from shared memory; default: the constant bank (surrogate op)
  const char* ce = getenv("HHG_GS_CW");
  const bool cwc = OP == HHG_OP_SURROGATE && !(ce && std::string(ce) == "smem");
  // cycle accounting (hhg_gs_prof enabled): the instrumented instantiation
  const bool prof = cwc && c->d_gsprof != nullptr;
  const size_t smem = march_smem_bytes(lv.slot_len, lv.N, RING);
  if (smem > (size_t)kMaxDynSmem) return HHG_ERR_STATE;
  auto kern = prof ? k_gs_items<OP, NT, RING, true, true>
                   : cwc ? k_gs_items<OP, NT, RING, true, false> : k_gs_items<OP, NT, RING, false, false>;
  const void* fn = (const void*)kern;
  hhg_status st = smem_attr(c, fn);
  if (st != HHG_OK) return st;
  int grid = 0;
  if ((st = resident_grid(c, fn, NT, smem, grid)) != HHG_OK) return st;
  const int nb = (int)lv.bands.size();
  // deadlock freedom needs every band of the partially handed-out macro
  // resident at once (an item waits on its neighbour bands): otherwise use the
  // colour-pass kernels (no cross-CTA waits)
  if (grid <= nb) return HHG_ERR_STATE;
  if (Te <= Tb) return HHG_OK;
  if (cwc && (st = ensure_cC(c, lv, OP)) != HHG_OK) return st;
  // completion flags cleared per sweep (epoch 1): the launch is replayable from
  // a CUDA graph (hhg_vcycle)
  HHG_CK(c, cudaMemsetAsync(lv.d_gs_flags + Tb * nb * 4, 0, (size_t)(Te - Tb) * nb * 4 * sizeof(int), c->stream));
  lv.gs_epoch = 1;
  ProfScope ps(c, 1);
  // macro chunks of <= kCMax (the constant-bank C_w table), run in order
  for (int64_t T0 = Tb; T0 < Te; T0 += (cwc ? kCMax : Te - Tb)) {
    const int64_t ntr = std::min<int64_t>(cwc ? kCMax : Te - Tb, Te - T0);
    if (cwc)
      HHG_CK(c, cudaMemcpyToSymbolAsync(g_cC, lv.d_cC + T0 * 15, ntr * 15 * sizeof(double), 0,
                                        cudaMemcpyDeviceToDevice, c->stream));
    HHG_CK(c, cudaMemsetAsync(lv.d_gs_counter, 0, sizeof(int), c->stream));
    const int64_t items = ntr * nb;
    kern<<<(unsigned)std::min<int64_t>(grid, items), NT, smem, c->stream>>>(
        lv.N, lv.S, lv.d_bands, nb, lv.slot_len, lv.d_coef10, lv.d_cons, u, f, ntr, T0, lv.d_gs_counter,
        lv.d_gs_flags, lv.gs_epoch, gs_stress(), c->d_gsprof);
    HHG_LAUNCHED(c);
  }
  return HHG_OK;
}

// The persistent 4-colour sweep with a producer warp and per-plane
// cross-band progress (gsprod.cuh; HHG_GS_KERNEL=prod: 7 compute warps, two
// CTAs per SM; prodw: 15 compute warps, one CTA per SM).
template <int OP, int RING, int NCW>
static hhg_status launch_gs_prod(Ctx* c, Level& lv, double* u, const double* f, int64_t Tb, int64_t Te) {
  constexpr int NT = 32 * NCW + 32;
  const int x = NCW <= 7 ? 0 : 1;
  if (lv.bands_p[x].empty()) return HHG_ERR_STATE;
  const bool cwc = OP == HHG_OP_SURROGATE;
  const size_t smem = march_smem_bytes(lv.slot_len_p[x], lv.N, RING);
  if (smem > (size_t)(NCW <= 7 ? 113 * 1024 : kMaxDynSmem)) return HHG_ERR_STATE;
  auto kern = cwc ? k_gs_prod<OP, RING, true, NCW> : k_gs_prod<OP, RING, false, NCW>;
  const void* fn = (const void*)kern;
  hhg_status st = smem_attr(c, fn);
  if (st != HHG_OK) return st;
  int grid = 0;
  if ((st = resident_grid(c, fn, NT, smem, grid)) != HHG_OK) return st;
  const int nb = (int)lv.bands_p[x].size();
  if (grid <= nb) return HHG_ERR_STATE;  // every band of the partially handed-out macro resident
  if ((size_t)nb > lv.bands.size() * 4) return HHG_ERR_STATE;  // progress words fit d_gs_flags
  if (Te <= Tb) return HHG_OK;
  if (cwc && (st = ensure_cC(c, lv, OP)) != HHG_OK) return st;
  // progress words (one per (macro, band)) cleared per sweep: replayable from a CUDA graph
  HHG_CK(c, cudaMemsetAsync(lv.d_gs_flags + Tb * nb, 0, (size_t)(Te - Tb) * nb * sizeof(int), c->stream));
  ProfScope ps(c, 1);
  for (int64_t T0 = Tb; T0 < Te; T0 += (cwc ? kCMax : Te - Tb)) {
    const int64_t ntr = std::min<int64_t>(cwc ? kCMax : Te - Tb, Te - T0);
    if (cwc)
      HHG_CK(c, cudaMemcpyToSymbolAsync(g_cC, lv.d_cC + T0 * 15, ntr * 15 * sizeof(double), 0,
                                        cudaMemcpyDeviceToDevice, c->stream));
    HHG_CK(c, cudaMemsetAsync(lv.d_gs_counter, 0, sizeof(int), c->stream));
    const int64_t items = ntr * nb;
    kern<<<(unsigned)std::min<int64_t>(grid, items), NT, smem, c->stream>>>(
        lv.N, lv.S, lv.d_bands_p[x], nb, lv.slot_len_p[x], lv.d_coef10, lv.d_cons, u, f, ntr, T0, lv.d_gs_counter,
        lv.d_gs_flags, gs_stress());
    HHG_LAUNCHED(c);
  }
  return HHG_OK;
}

template <int OP>
static hhg_status launch_gs_items(Ctx* c, Level& lv, double* u, const double* f, int64_t Tb, int64_t Te) {
  // 24-plane ring only while two CTAs fit an SM (N = 256: 768-double slots -> 16)
  if (march_smem_bytes(lv.slot_len, lv.N, 24) > 113 * 1024) return launch_gs_items_r<OP, 16>(c, lv, u, f, Tb, Te);
  return launch_gs_items_r<OP, 24>(c, lv, u, f, Tb, Te);
}

// The whole volume GS (4 colours) as one single-pass wavefront launch
// (gsfront.cuh): NT threads per CTA over bands of <= NT columns.
template <int OP, int LAG, int RING, int NT>
static hhg_status launch_gs_front_r(Ctx* c, Level& lv, double* u, const double* f) {
  const bool wide = NT > kMarchThreads;
  const std::vector<Band>& bands = wide ? lv.bands_w : lv.bands;
  const int slot_len = wide ? lv.slot_len_w : lv.slot_len;
  const size_t smem = front_smem_bytes<RING, NT>(slot_len, lv.N);
  if (smem > (size_t)kMaxDynSmem) return HHG_ERR_STATE;
  const bool prof = c->d_gsprof != nullptr;
  const void* fn = prof ? (const void*)k_gs_front<OP, LAG, RING, NT, true>
                        : (const void*)k_gs_front<OP, LAG, RING, NT, false>;
  hhg_status st = smem_attr(c, fn);
  if (st != HHG_OK) return st;
  int grid = 0;
  if ((st = resident_grid(c, fn, NT, smem, grid)) != HHG_OK) return st;
  const int nb = (int)bands.size();
  // every band of the last handed-out macro must be resident (bands of a macro wait on each other)
  if (grid <= nb) return HHG_ERR_STATE;
  if (!lv.d_gs_ex) {
    const size_t np = (size_t)std::max<int64_t>(c->nt_local * (int64_t)lv.bands.size(), 1);
    HHG_CK(c, cudaMalloc(&lv.d_gs_ex, (size_t)lv.n_local * 2 * sizeof(uint64_t)));
    HHG_CK(c, cudaMemsetAsync(lv.d_gs_ex, 0, (size_t)lv.n_local * 2 * sizeof(uint64_t), c->stream));
    HHG_CK(c, cudaMalloc(&lv.d_gs_prog, np * sizeof(uint32_t)));
    HHG_CK(c, cudaMemsetAsync(lv.d_gs_prog, 0, np * sizeof(uint32_t), c->stream));
    HHG_CK(c, cudaMalloc(&lv.d_gs_epoch, sizeof(uint32_t)));
    HHG_CK(c, cudaMemsetAsync(lv.d_gs_epoch, 0, sizeof(uint32_t), c->stream));
  }
  const int64_t items = c->nt_local * nb;
  ProfScope ps(c, 1);
  k_front_begin<<<1, 1, 0, c->stream>>>(lv.d_gs_counter, lv.d_gs_epoch);
  HHG_LAUNCHED(c);
  auto kern = prof ? k_gs_front<OP, LAG, RING, NT, true> : k_gs_front<OP, LAG, RING, NT, false>;
  kern<<<(unsigned)std::min<int64_t>(grid, items), NT, smem, c->stream>>>(
      lv.N, lv.S, wide ? lv.d_bands_w : lv.d_bands, nb, slot_len, lv.d_coef10, lv.d_cons, u, f, c->nt_local,
      lv.d_gs_counter, lv.d_gs_epoch, lv.d_gs_prog, lv.d_gs_ex, c->d_gsprof, gs_stress());
  HHG_LAUNCHED(c);
  return HHG_OK;
}

// variant: 0 = 256 threads, LAG 4; 1 = 256, LAG 6; 2 = 512, LAG 4; 3 = 512, LAG 6
template <int OP>
static hhg_status launch_gs_front(Ctx* c, Level& lv, double* u, const double* f, int variant) {
  switch (variant) {
    case 1: return launch_gs_front_r<OP, 6, 32, kMarchThreads>(c, lv, u, f);
    case 2: return launch_gs_front_r<OP, 4, 24, 2 * kMarchThreads>(c, lv, u, f);
    case 3: return launch_gs_front_r<OP, 6, 32, 2 * kMarchThreads>(c, lv, u, f);
    default:
      // two CTAs per SM while the 24-slot ring fits half the shared memory
      if (front_smem_bytes<24, kMarchThreads>(lv.slot_len, lv.N) <= 113 * 1024)
        return launch_gs_front_r<OP, 4, 24, kMarchThreads>(c, lv, u, f);
      return launch_gs_front_r<OP, 4, 20, kMarchThreads>(c, lv, u, f);
  }
}

// Whether the volume pass of (op, mode) runs the column-march kernels, which
// take a macro range (the overlapped exchange splits boundary / interior macros).
static bool march_path(const Level& lv, int op) {
  if (op == HHG_OP_SURROGATE_FACES) op = HHG_OP_SURROGATE;
  return !lv.bands.empty() && ((op == HHG_OP_SURROGATE && lv.d_coef10) || op == HHG_OP_CONST_AFFINE);
}

static hhg_status volume_pass(Ctx* c, Level& lv, int op, int mode, int colour, const double* u,
                              const double* f, double* out, int64_t Tb = 0, int64_t Te = -1) {
  if (Te < 0) Te = c->nt_local;
  if (op == HHG_OP_SURROGATE_FACES) op = HHG_OP_SURROGATE;  // volume rows: the surrogate
  // column-march kernels: q <= 2 surrogate (s_w quadratic along a column) and the constant stencil
  const bool march = march_path(lv, op);
  if (!march && (Tb != 0 || Te != c->nt_local)) return set_err(c, HHG_ERR_STATE, "macro range on a full-grid kernel");
  if (march && mode == kModeGS)
    return op == HHG_OP_SURROGATE ? launch_gs_march<HHG_OP_SURROGATE>(c, lv, colour, out, f, Tb, Te)
                                  : launch_gs_march<HHG_OP_CONST_AFFINE>(c, lv, colour, out, f, Tb, Te);
  if (march) {
    if (op == HHG_OP_SURROGATE)
      return mode == kModeApply ? launch_march<HHG_OP_SURROGATE, kModeApply>(c, lv, u, f, out, Tb, Te)
                                : launch_march<HHG_OP_SURROGATE, kModeResid>(c, lv, u, f, out, Tb, Te);
    return mode == kModeApply ? launch_march<HHG_OP_CONST_AFFINE, kModeApply>(c, lv, u, f, out, Tb, Te)
                              : launch_march<HHG_OP_CONST_AFFINE, kModeResid>(c, lv, u, f, out, Tb, Te);
  }
  if (op == HHG_OP_FEM_ELEMENTWISE && mode != kModeGS && !lv.bands.empty()) {
    // plane range per band (the first band's also holds diagonal 0)
    int need = 0;
    for (const Band& bb : lv.bands_fem) need = std::max(need, bb.ncols + (bb.d0 == 2 ? bb.c_lo : 0));
    const int slot = std::max(lv.slot_len, (need + 3 + 3) / 4 * 4);
    const size_t smem = ew_smem_bytes(slot, lv.N);
    if (need + 1 > kFPosPerThread * kMarchThreads || smem > (size_t)kMaxDynSmem)
      return set_err(c, HHG_ERR_INVALID, "fem: band ring wider than the element-wise kernel");
    hhg_status st = smem_attr(c, (const void*)k_vol_fem_ew<kModeApply>);
    if (st == HHG_OK) st = smem_attr(c, (const void*)k_vol_fem_ew<kModeResid>);
    if (st != HHG_OK) return st;
    if (!lv.d_ew_lo) {
      HHG_CK(c, cudaMalloc(&lv.d_ew_lo, lv.n_local * sizeof(double)));
      HHG_CK(c, cudaMalloc(&lv.d_ew_hi, lv.n_local * sizeof(double)));
    }
    const int nb = (int)lv.bands_fem.size();
    ProfScope ps(c, 0);
    const unsigned grid = (unsigned)(nb * c->nt_local);
    if (mode == kModeApply)
      k_vol_fem_ew<kModeApply><<<grid, kMarchThreads, smem, c->stream>>>(
          lv.N, lv.S, lv.d_bands_fem, nb, slot, c->d_geo, c->blended, u, f, out, lv.d_ew_lo, lv.d_ew_hi);
    else
      k_vol_fem_ew<kModeResid><<<grid, kMarchThreads, smem, c->stream>>>(
          lv.N, lv.S, lv.d_bands_fem, nb, slot, c->d_geo, c->blended, u, f, out, lv.d_ew_lo, lv.d_ew_hi);
    HHG_LAUNCHED(c);
    if (nb > 1) {
      int maxcol = 0;
      for (const Band& bb : lv.bands_fem) maxcol = std::max(maxcol, bb.d1 + bb.d0);
      const dim3 fg(nblk((int64_t)maxcol * (lv.N - 1), 128), (unsigned)c->nt_local, (unsigned)nb);
      if (mode == kModeApply)
        k_fem_ew_fixup<kModeApply><<<fg, 128, 0, c->stream>>>(lv.N, lv.S, lv.d_bands_fem, nb, lv.d_ew_lo, lv.d_ew_hi, out);
      else
        k_fem_ew_fixup<kModeResid><<<fg, 128, 0, c->stream>>>(lv.N, lv.S, lv.d_bands_fem, nb, lv.d_ew_lo, lv.d_ew_hi, out);
      HHG_LAUNCHED(c);
    }
    return HHG_OK;
  }
  // one thread per lattice node: q = 3, 4 (the weights are not quadratic along
  // a column) and the level with no march band
  dim3 grid(nblk(lv.P, 128), (unsigned)c->nt_local);
  ProfScope ps(c, mode == kModeGS ? 1 : 0);
  k_vol_v1<<<grid, 128, 0, c->stream>>>(lv.N, lv.S, lv.P, c->d_geo, lv.d_coef, lv.mq, lv.d_cons, op,
                                        c->blended, mode, colour, u, f, out);
  HHG_LAUNCHED(c);
  return HHG_OK;
}

static hhg_status lp_pass(Ctx* c, Level& lv, int op, int mode, const double* u, const double* f,
                          double* out) {
  hhg_status stf = face_apply(c, lv, op, mode, u, f, out);
  if (stf != HHG_OK) return stf;
  if (lv.n_rows == 0) return HHG_OK;
  const double* val = op == HHG_OP_CONST_AFFINE ? lv.d_val_cons : lv.d_val;
  ProfScope ps(c, 2);
  k_lp_apply<<<nblk(lv.n_rows, 128), 128, 0, c->stream>>>(0, lv.n_rows, lv.d_row_ptr, lv.d_col, val,
                                                         lv.d_copy_ptr, lv.d_copy, u, f, out, mode);
  HHG_LAUNCHED(c);
  return HHG_OK;
}

static hhg_status zero_dir(Ctx* c, Level& lv, double* out) {
  if (lv.n_dir == 0) return HHG_OK;
  ProfScope ps(c, 3);
  k_zero_slots<<<nblk(lv.n_dir, 256), 256, 0, c->stream>>>(lv.n_dir, lv.d_dir_slot, out);
  HHG_LAUNCHED(c);
  return HHG_OK;
}

hhg_status zero_dir_slots(Ctx* c, Level& lv, double* out) { return zero_dir(c, lv, out); }

// a.b over the unique unknowns into the device scalar d_out (fixed grids: deterministic)
static hhg_status ensure_red(Ctx* c) {
  if (c->red_n < 2 * kRedBlocks + 1) {
    HHG_CK(c, cudaMalloc(&c->d_red, (2 * kRedBlocks + 1) * sizeof(double)));
    HHG_CK(c, cudaMallocHost(&c->h_red, 2 * sizeof(double)));
    c->red_n = 2 * kRedBlocks + 1;
  }
  return HHG_OK;
}

hhg_status dot_dev(Ctx* c, Level& lv, const double* a, const double* b, double* d_out) {
  hhg_status st0 = ensure_red(c);
  if (st0 != HHG_OK) return st0;
  ProfScope ps(c, 3);
  k_dot<<<kRedBlocks, 256, 0, c->stream>>>(lv.N, lv.S, lv.P, c->nt_local, a, b, lv.n_rows, lv.d_col,
                                           lv.d_row_ptr, c->d_red);
  HHG_LAUNCHED(c);
  hhg_status stf = face_dot(c, lv, a, b, c->d_red + kRedBlocks, kRedBlocks);
  if (stf != HHG_OK) return stf;
  k_final_sum<<<1, 1024, 0, c->stream>>>(c->d_red, 2 * kRedBlocks, d_out);
  HHG_LAUNCHED(c);
  return dist_allreduce_sum(c, d_out);
}

// Multi-rank: a kernel that updates only the local blocks (prolongation)
// leaves the ghost-block copies of this rank's OWN lower-primitive nodes stale
// (no peer sends them: the rank is their owner), and stored rows may read
// them.  Refresh them from the owner-macro copy.
hhg_status lp_sync_own_copies(Ctx* c, Level& lv, double* v) {
  if (lv.n_rows) {
    k_lp_sync<<<nblk(lv.n_rows, 128), 128, 0, c->stream>>>(lv.n_rows, lv.d_copy_ptr, lv.d_copy, v);
    HHG_LAUNCHED(c);
  }
  return face_sync(c, lv, v);
}

hhg_status lp_sum_copies(Ctx* c, Level& lv, double* v) {
  if (lv.n_rows) {
    k_lp_sumcopies<<<nblk(lv.n_rows, 128), 128, 0, c->stream>>>(lv.n_rows, lv.d_copy_ptr, lv.d_copy, v);
    HHG_LAUNCHED(c);
  }
  return face_sum_copies(c, lv, v);
}

hhg_status norm2_of(Ctx* c, Level& lv, const double* r, double* out) {
  hhg_status st = ensure_red(c);
  if (st != HHG_OK) return st;
  if ((st = dot_dev(c, lv, r, r, c->d_red + 2 * kRedBlocks)) != HHG_OK) return st;
  HHG_CK(c, cudaMemcpyAsync(c->h_red, c->d_red + 2 * kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  { hhg_status st_sync__ = ctx_sync(c); if (st_sync__ != HHG_OK) return st_sync__; }
  *out = std::sqrt(c->h_red[0]);
  return HHG_OK;
}

// lexicographic volume GS (gslex.cuh): one CTA per macro
static hhg_status launch_gs_lex(Ctx* c, Level& lv, int op, double* u, const double* f) {
  const size_t smem = lex_smem_bytes(lv.N);
  static bool attr = false;
  if (!attr) {
    HHG_CK(c, cudaFuncSetAttribute(k_gs_lex<HHG_OP_SURROGATE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    HHG_CK(c, cudaFuncSetAttribute(k_gs_lex<HHG_OP_CONST_AFFINE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kMaxDynSmem));
    attr = true;
  }
  if (lv.N < 4) return HHG_OK;  // no interior nodes
  if (op == HHG_OP_SURROGATE && !lv.d_coef10) return set_err(c, HHG_ERR_STATE, "gs_lex: surrogate not fitted");
  ProfScope ps(c, 1);
  for (int64_t T0 = 0; T0 < c->nt_local; T0 += 65535) {
    const unsigned nt = (unsigned)std::min<int64_t>(65535, c->nt_local - T0);
    if (op == HHG_OP_SURROGATE)
      k_gs_lex<HHG_OP_SURROGATE><<<nt, kLexThreads, smem, c->stream>>>(lv.N, lv.S, lv.d_coef10, lv.d_cons, u, f,
                                                                       (int)T0);
    else
      k_gs_lex<HHG_OP_CONST_AFFINE><<<nt, kLexThreads, smem, c->stream>>>(lv.N, lv.S, lv.d_coef10, lv.d_cons, u,
                                                                          f, (int)T0);
    HHG_LAUNCHED(c);
  }
  return HHG_OK;
}

hhg_status gs_sweep_dev(Ctx* c, Level& lv, int op, double* u, const double* f, bool lex) {
  const double* val = op == HHG_OP_CONST_AFFINE ? lv.d_val_cons : lv.d_val;
  for (int s = 0; s < kNumLpSteps; ++s) {
    if (s >= kStepFace0) {  // face colours: structured face rows
      hhg_status stf = face_gs_step(c, lv, op, s - kStepFace0, u, f);
      if (stf != HHG_OK) return stf;
    }
    int64_t r0 = lv.step_start[s], r1 = lv.step_start[s + 1];
    if (r1 > r0) {
      ProfScope ps(c, 2);
      k_lp_gs_compute<<<nblk(r1 - r0, 128), 128, 0, c->stream>>>(r0, r1, lv.d_row_ptr, lv.d_col, val, u, f,
                                                                 lv.d_tmp);
      HHG_LAUNCHED(c);
      k_lp_write<<<nblk(r1 - r0, 128), 128, 0, c->stream>>>(r0, r1, lv.d_copy_ptr, lv.d_copy, lv.d_tmp, u);
      HHG_LAUNCHED(c);
    }
    // the next class step reads this step's values on every rank -- except
    // after the vertex step: the next step (edge colour 0, even positions
    // m >= 2 along an edge) has no vertex in its stencils (lattice distance
    // >= 2), so the vertex values travel with the edge-colour-0 exchange and
    // reach every rank before edge colour 1 (positions 1 and N-1) reads them.
    // 6 exchanges per sweep instead of 7; results unchanged (bitwise
    // rank-count test, tests/test_gpu_dist.py).
    if (s == kStepVertex) continue;
    hhg_status sts = dist_sync(c, lv, u);
    if (sts != HHG_OK) return sts;
  }
  if (op == HHG_OP_SURROGATE_FACES) op = HHG_OP_SURROGATE;  // volume rows: the surrogate
  if (lex) {  // the paper's lexicographic volume ordering
    hhg_status st = launch_gs_lex(c, lv, op, u, f);
    if (st != HHG_OK) return st;
    return dist_sync(c, lv, u);
  }
  // HHG_GS_KERNEL (read per call, so tests can compare the variants):
  // default = the persistent 4-pass sweep k_gs_items; the single-pass wavefront
  // k_gs_front as "front" (256 threads, LAG 4), "front6" (LAG 6), "wide4" /
  // "wide6" (512 threads); the producer-warp sweep k_gs_prod as "prod" (7
  // compute warps) / "prodw" (15); "passes" = 4 colour launches
  const char* e = getenv("HHG_GS_KERNEL");
  const std::string ks = e ? e : "";
  const int mode = ks == "passes" ? 1 : ks == "front" ? 3 : ks == "front6" ? 4 : ks == "wide4" ? 5 : ks == "wide6" ? 6 : ks == "prod" ? 7 : ks == "prodw" ? 8 : 2;
  const bool march_ok = march_path(lv, op);
  auto sweep = [&](int64_t Tb, int64_t Te) -> hhg_status {
    hhg_status st = HHG_ERR_STATE;
    if (march_ok && mode == 2)
      st = op == HHG_OP_SURROGATE ? launch_gs_items<HHG_OP_SURROGATE>(c, lv, u, f, Tb, Te)
                                  : launch_gs_items<HHG_OP_CONST_AFFINE>(c, lv, u, f, Tb, Te);
    if (march_ok && mode == 7)
      st = op == HHG_OP_SURROGATE ? launch_gs_prod<HHG_OP_SURROGATE, 24, 7>(c, lv, u, f, Tb, Te)
                                  : launch_gs_prod<HHG_OP_CONST_AFFINE, 24, 7>(c, lv, u, f, Tb, Te);
    if (march_ok && mode == 8)
      st = op == HHG_OP_SURROGATE ? launch_gs_prod<HHG_OP_SURROGATE, 32, 15>(c, lv, u, f, Tb, Te)
                                  : launch_gs_prod<HHG_OP_CONST_AFFINE, 32, 15>(c, lv, u, f, Tb, Te);
    if (march_ok && mode >= 3 && mode <= 6 && Tb == 0 && Te == c->nt_local) {
      const int variant = mode - 3;
      st = op == HHG_OP_SURROGATE ? launch_gs_front<HHG_OP_SURROGATE>(c, lv, u, f, variant)
                                  : launch_gs_front<HHG_OP_CONST_AFFINE>(c, lv, u, f, variant);
    }
    if (st != HHG_OK) {
      if (c->poisoned) return HHG_ERR_CUDA;
      for (int col = 0; col < 4; ++col)
        if ((st = volume_pass(c, lv, op, kModeGS, col, u, f, u, march_ok ? Tb : 0, march_ok ? Te : -1)) != HHG_OK)
          return st;
    }
    return HHG_OK;
  };
  // multi-rank: the ghost exchange of the swept volume values overlaps the
  // sweep of the interior macros (HHG_OVERLAP=0 disables)
  if (c->nranks > 1 && march_ok && (mode == 1 || mode == 2 || mode >= 7) && overlap_on()) {
    hhg_status st = sweep(0, c->nt_bnd);
    if (st != HHG_OK) return st;
    return dist_sync_overlapped(c, lv, u, [&]() { return sweep(c->nt_bnd, c->nt_local); });
  }
  hhg_status st = sweep(0, c->nt_local);
  if (st != HHG_OK) return st;
  return dist_sync(c, lv, u);  // ghost volume values for the other ranks
}

hhg_status apply_dev(Ctx* c, Level& lv, int op, int mode, const double* u, const double* f, double* y) {
  hhg_status st;
  if (c->nranks > 1 && march_path(lv, op) && overlap_on()) {
    // boundary macros and the lower-primitive rows first; the exchange of the
    // rows' owner values and of the boundary volume values then overlaps the
    // interior macros' volume pass (they send and receive nothing)
    if ((st = volume_pass(c, lv, op, mode, 0, u, f, y, 0, c->nt_bnd)) != HHG_OK) return st;
    if ((st = lp_pass(c, lv, op, mode, u, f, y)) != HHG_OK) return st;
    st = dist_sync_overlapped(c, lv, y, [&]() { return volume_pass(c, lv, op, mode, 0, u, f, y, c->nt_bnd, c->nt_local); });
    if (st != HHG_OK) return st;
    return zero_dir(c, lv, y);
  }
  if ((st = volume_pass(c, lv, op, mode, 0, u, f, y)) != HHG_OK) return st;
  if ((st = lp_pass(c, lv, op, mode, u, f, y)) != HHG_OK) return st;
  if ((st = dist_sync(c, lv, y)) != HHG_OK) return st;  // owners' rows -> every copy / ghost
  return zero_dir(c, lv, y);
}

}  // namespace hhg

using namespace hhg;

extern "C" hhg_status hhg_apply(hhg_ctx ctx, int L, hhg_op op, const double* u, double* y) {
  Ctx* c = (Ctx*)ctx;
  hhg_status st = check_call(c, L, op, false);
  if (st != HHG_OK) return st;
  if (!u || !y || u == y) return set_err(c, HHG_ERR_INVALID, "u, y must be non-NULL and distinct");
  Level& lv = c->levels[L];
  Staged su, sy;
  if ((st = stage(c, 0, u, lv.n_local, true, su)) != HHG_OK) return st;
  if ((st = stage(c, 1, y, lv.n_local, false, sy)) != HHG_OK) return st;
  if ((st = apply_dev(c, lv, op, kModeApply, su.dev, nullptr, sy.dev)) != HHG_OK) return st;
  return unstage(c, sy, lv.n_local);
}

extern "C" hhg_status hhg_residual(hhg_ctx ctx, int L, hhg_op op, const double* u, const double* f,
                                   double* r, double* norm2) {
  Ctx* c = (Ctx*)ctx;
  hhg_status st = check_call(c, L, op, false);
  if (st != HHG_OK) return st;
  if (!u || !f || !r || r == u || r == f) return set_err(c, HHG_ERR_INVALID, "bad vectors");
  Level& lv = c->levels[L];
  Staged su, sf, sr;
  if ((st = stage(c, 0, u, lv.n_local, true, su)) != HHG_OK) return st;
  if ((st = stage(c, 1, f, lv.n_local, true, sf)) != HHG_OK) return st;
  if ((st = stage(c, 2, r, lv.n_local, false, sr)) != HHG_OK) return st;
  if ((st = apply_dev(c, lv, op, kModeResid, su.dev, sf.dev, sr.dev)) != HHG_OK) return st;
  if (norm2 && (st = norm2_of(c, lv, sr.dev, norm2)) != HHG_OK) return st;
  return unstage(c, sr, lv.n_local);
}

static hhg_status gs_sweep_api(hhg_ctx ctx, int L, hhg_op op, double* u, const double* f, int n, bool lex) {
  Ctx* c = (Ctx*)ctx;
  hhg_status st = check_call(c, L, op, true);
  if (st != HHG_OK) return st;
  if (!u || !f || (const double*)u == f || n < 0) return set_err(c, HHG_ERR_INVALID, "bad vectors");
  Level& lv = c->levels[L];
  Staged su, sf;
  if ((st = stage(c, 0, u, lv.n_local, true, su)) != HHG_OK) return st;
  if ((st = stage(c, 1, f, lv.n_local, true, sf)) != HHG_OK) return st;
  for (int s = 0; s < n; ++s)
    if ((st = gs_sweep_dev(c, lv, op, su.dev, sf.dev, lex)) != HHG_OK) return st;
  return unstage(c, su, lv.n_local);
}

extern "C" hhg_status hhg_gs_sweep(hhg_ctx ctx, int L, hhg_op op, double* u, const double* f, int n) {
  return gs_sweep_api(ctx, L, op, u, f, n, false);
}

extern "C" hhg_status hhg_gs_sweep_lex(hhg_ctx ctx, int L, hhg_op op, double* u, const double* f, int n) {
  Ctx* c = (Ctx*)ctx;
  if (c && op == HHG_OP_FEM_ELEMENTWISE) return set_err(c, HHG_ERR_INVALID, "FEM is not a smoother");
  return gs_sweep_api(ctx, L, op, u, f, n, true);
}

namespace hhg {

hhg_status gather_owned_dev(Ctx* c, Level& lv, const double* local, double* dglob) {
  HHG_CK(c, cudaMemsetAsync(dglob, 0, lv.gi.n_total * sizeof(double), c->stream));
  dim3 grid(nblk(lv.P, 128), (unsigned)c->nt_local);
  k_vol_gather<<<grid, 128, 0, c->stream>>>(lv.N, lv.S, lv.P, c->d_topo, lv.gi, local, dglob, 0);
  HHG_LAUNCHED(c);
  if (lv.n_rows) {
    k_lp_gather<<<nblk(lv.n_rows, 128), 128, 0, c->stream>>>(lv.n_rows, lv.d_copy_ptr, lv.d_copy,
                                                            lv.d_row_gid, local, dglob, 0);
    HHG_LAUNCHED(c);
  }
  return face_gather(c, lv, local, dglob, 0);
}

hhg_status scatter_global_dev(Ctx* c, Level& lv, const double* dglob, double* local) {
  hhg_status st;
  HHG_CK(c, cudaMemsetAsync(local, 0, lv.n_local * sizeof(double), c->stream));
  dim3 grid(nblk(lv.P, 128), (unsigned)c->nt_blocks);  // ghost interiors too
  k_vol_gather<<<grid, 128, 0, c->stream>>>(lv.N, lv.S, lv.P, c->d_topo, lv.gi, local, (double*)dglob, 1);
  HHG_LAUNCHED(c);
  if (lv.n_rows) {
    k_lp_gather<<<nblk(lv.n_rows, 128), 128, 0, c->stream>>>(lv.n_rows, lv.d_copy_ptr, lv.d_copy,
                                                            lv.d_row_gid, local, (double*)dglob, 1);
    HHG_LAUNCHED(c);
  }
  if ((st = face_gather(c, lv, local, (double*)dglob, 1)) != HHG_OK) return st;
  if ((st = dist_sync(c, lv, local)) != HHG_OK) return st;
  return zero_dir(c, lv, local);
}

}  // namespace hhg

using namespace hhg;

extern "C" hhg_status hhg_gather_global(hhg_ctx ctx, int L, const double* local, double* glob) {
  Ctx* c = (Ctx*)ctx;
  if (!c || L < 2 || L > c->L_max || !local || !glob) return HHG_ERR_INVALID;
  if (c->host_only) return HHG_ERR_STATE;
  // multi-rank: writes the entries this rank owns, 0 elsewhere (sum over ranks = global vector)
  Level& lv = c->levels[L];
  hhg_status st;
  Staged sl;
  if ((st = stage(c, 0, local, lv.n_local, true, sl)) != HHG_OK) return st;
  // global may be larger than n_local: use a dedicated allocation if host
  double* dglob = glob;
  bool host_glob = !is_device_ptr(glob);
  if (host_glob) HHG_CK(c, cudaMalloc(&dglob, lv.gi.n_total * sizeof(double)));
  if ((st = gather_owned_dev(c, lv, sl.dev, dglob)) != HHG_OK) return st;
  if (host_glob) {
    HHG_CK(c, cudaMemcpyAsync(glob, dglob, lv.gi.n_total * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    { hhg_status st_sync__ = ctx_sync(c); if (st_sync__ != HHG_OK) return st_sync__; }
    cudaFree(dglob);
  }
  return HHG_OK;
}

extern "C" hhg_status hhg_scatter_global(hhg_ctx ctx, int L, const double* glob, double* local) {
  Ctx* c = (Ctx*)ctx;
  if (!c || L < 2 || L > c->L_max || !local || !glob) return HHG_ERR_INVALID;
  if (c->host_only) return HHG_ERR_STATE;
  // multi-rank: every rank passes the full global vector; owned rows fill their
  // copies here and the sync fills the mirrors of nodes owned elsewhere
  Level& lv = c->levels[L];
  hhg_status st;
  Staged sl;
  if ((st = stage(c, 0, local, lv.n_local, false, sl)) != HHG_OK) return st;
  const double* dglob = glob;
  double* tmp = nullptr;
  if (!is_device_ptr(glob)) {
    HHG_CK(c, cudaMalloc(&tmp, lv.gi.n_total * sizeof(double)));
    HHG_CK(c, cudaMemcpyAsync(tmp, glob, lv.gi.n_total * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    dglob = tmp;
  }
  if ((st = scatter_global_dev(c, lv, dglob, sl.dev)) != HHG_OK) return st;
  if ((st = unstage(c, sl, lv.n_local)) != HHG_OK) return st;
  if (tmp) {
    { hhg_status st_sync__ = ctx_sync(c); if (st_sync__ != HHG_OK) return st_sync__; }
    cudaFree(tmp);
  }
  return HHG_OK;
}

extern "C" hhg_status hhg_sync_copies(hhg_ctx ctx, int L, double* local) {
  Ctx* c = (Ctx*)ctx;
  if (!c || L < 2 || L > c->L_max || !local) return HHG_ERR_INVALID;
  Level& lv = c->levels[L];
  hhg_status st;
  Staged sl;
  if ((st = stage(c, 0, local, lv.n_local, true, sl)) != HHG_OK) return st;
  if (lv.n_rows) {
    k_lp_sync<<<nblk(lv.n_rows, 128), 128, 0, c->stream>>>(lv.n_rows, lv.d_copy_ptr, lv.d_copy, sl.dev);
    HHG_LAUNCHED(c);
  }
  if ((st = face_sync(c, lv, sl.dev)) != HHG_OK) return st;
  if ((st = dist_sync(c, lv, sl.dev)) != HHG_OK) return st;
  if ((st = zero_dir(c, lv, sl.dev)) != HHG_OK) return st;
  return unstage(c, sl, lv.n_local);
}

extern "C" hhg_status hhg_eval_stencils(hhg_ctx ctx, int L, hhg_op op, int64_t macro, double* out) {
  Ctx* c = (Ctx*)ctx;
  hhg_status st = check_call(c, L, op, false);
  if (st != HHG_OK) return st;
  if (macro < 0 || macro >= c->nt_local || !out) return set_err(c, HHG_ERR_INVALID, "bad macro/out");
  Level& lv = c->levels[L];
  int64_t n = n_interior(lv.N) * 15;
  Staged so;
  if ((st = stage(c, 3, out, std::max<int64_t>(n, lv.n_local), false, so)) != HHG_OK) return st;
  const double* coef = lv.d_coef ? lv.d_coef + macro * 15 * lv.mq : nullptr;
  k_eval_stencils<<<nblk(lv.P, 128), 128, 0, c->stream>>>(lv.N, lv.P, c->d_geo + macro * 16, coef, lv.mq,
                                                         lv.d_cons + macro * 15, op, c->blended, so.dev);
  HHG_LAUNCHED(c);
  if (so.staged) {
    HHG_CK(c, cudaMemcpyAsync(out, so.dev, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    { hhg_status st_sync__ = ctx_sync(c); if (st_sync__ != HHG_OK) return st_sync__; }
  }
  return HHG_OK;
}

// Cycle accounting of the wavefront GS kernel (development): enable != 0
// allocates and zeroes the counters, later sweeps accumulate; read copies the
// 16 counters out (thread 0's cycles in mbar wait / compute / halo wait /
// progress check / barrier / post-barrier, steps, items, failed halo polls).
extern "C" hhg_status hhg_gs_prof(hhg_ctx ctx, int enable, unsigned long long* out16) {
  Ctx* c = (Ctx*)ctx;
  if (!c) return HHG_ERR_INVALID;
  if (enable && !c->d_gsprof) HHG_CK(c, cudaMalloc(&c->d_gsprof, 16 * sizeof(unsigned long long)));
  if (out16 && c->d_gsprof) {
    HHG_CK(c, cudaStreamSynchronize(c->stream));
    HHG_CK(c, cudaMemcpy(out16, c->d_gsprof, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  }
  if (c->d_gsprof) HHG_CK(c, cudaMemsetAsync(c->d_gsprof, 0, 16 * sizeof(unsigned long long), c->stream));
  if (!enable && c->d_gsprof) {
    HHG_CK(c, cudaStreamSynchronize(c->stream));
    cudaFree(c->d_gsprof);
    c->d_gsprof = nullptr;
  }
  return HHG_OK;
}

extern "C" hhg_status hhg_profile(hhg_ctx ctx, int enable) {
  Ctx* c = (Ctx*)ctx;
  if (!c) return HHG_ERR_INVALID;
  c->prof = enable != 0;
  return HHG_OK;
}

extern "C" hhg_status hhg_profile_read(hhg_ctx ctx, int kind, double* total_ms, int64_t* launches) {
  Ctx* c = (Ctx*)ctx;
  if (!c || kind < 0 || kind > 3) return HHG_ERR_INVALID;
  { hhg_status st_sync__ = ctx_sync(c); if (st_sync__ != HHG_OK) return st_sync__; }
  double tot = 0.0;
  for (auto& p : c->ev_rec[kind]) {
    float ms = 0.f;
    HHG_CK(c, cudaEventElapsedTime(&ms, p.first, p.second));
    tot += ms;
    c->ev_pool.push_back(p.first);
    c->ev_pool.push_back(p.second);
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = (int64_t)c->ev_rec[kind].size();
  c->ev_rec[kind].clear();
  return HHG_OK;
}


