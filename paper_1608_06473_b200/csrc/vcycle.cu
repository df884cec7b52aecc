// Geometric multigrid V(nu1,nu2) cycle, grid transfers and
// the coarse CG solver (R18, R19).
//
// Transfers live in index space per macro: P interpolates linearly -- a fine
// node 2C coincides with coarse node C, every other fine node is the midpoint
// of exactly one coarse edge whose direction is fixed by its parity class
// (pinned by brute force in tests/test_oracle_solvers.py) -- and R = P^T.
// P is evaluated for every copy of a shared fine node (identical arithmetic =>
// copies stay consistent).  R sums over fine nodes: each macro adds the fine
// nodes it OWNS (lowest macro id containing the node's primitive) into partial
// sums at its copies of the coarse nodes, then the copies of shared coarse
// nodes are summed (hhg::lp_sum_copies), so every fine node counts once.
// Multi-rank: each rank restricts its own macros; copies on other ranks reach
// the owner through dist_sum_to_owner (the reverse of the ghost sync), and
// prolongation re-syncs the ghost slots it cannot compute.
#include <cmath>
#include <cstdlib>

#include "fem_device.cuh"
#include "hhg_internal.h"

namespace hhg {

// parity class (i%2, j%2, k%2) -> coarse edge direction
__device__ __constant__ static const int kParityDir[8][3] = {
    {0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {-1, 1, 0}, {0, 0, 1}, {-1, 0, 1}, {0, -1, 1}, {1, -1, 1}};

// does macro (own mask) own fine lattice node (i,j,k) at level N?
__device__ __forceinline__ bool owns(uint16_t own, int N, int i, int j, int k) {
  const int w[4] = {N - i - j - k, i, j, k};
  int sup[4], ns = 0, zero = 0;
  for (int v = 0; v < 4; ++v) {
    if (w[v] > 0) sup[ns++] = v;
    else zero = v;
  }
  if (ns == 4) return true;
  if (ns == 3) return (own >> zero) & 1;
  if (ns == 2) return (own >> (4 + local_edge(sup[0], sup[1]))) & 1;
  return (own >> (10 + sup[0])) & 1;
}

// Lattice position of (i, j, k) from a shared-memory plane-offset table.
__device__ __forceinline__ int64_t lpos(const int64_t* po, int i, int j, int k) { return po[k] + col_idx(i, j); }

__device__ __forceinline__ void col_of(int c, int& i, int& j) {
  int d = (int)((sqrt(8.0 * (double)c + 1.0) - 1.0) * 0.5);
  while ((d + 1) * (d + 2) / 2 <= c) ++d;
  while (d * (d + 1) / 2 > c) --d;
  j = c - d * (d + 1) / 2;
  i = d - j;
}

// partial restriction at every coarse lattice node of every macro: thread =
// coarse lattice column (i, j) of macro blockIdx.y, marching k (no per-node
// position decode; plane offsets from shared memory)
__global__ void k_restrict_partial(int Nf, int64_t Sf, int64_t Sc, int64_t Pc, const uint16_t* __restrict__ own,
                                   const double* __restrict__ rf, double* __restrict__ fc) {
  __shared__ int64_t pof[258], poc[130];
  const int Nc = Nf / 2;
  for (int k = threadIdx.x; k <= Nf; k += blockDim.x) pof[k] = plane_off(Nf, k);
  for (int k = threadIdx.x; k <= Nc; k += blockDim.x) poc[k] = plane_off(Nc, k);
  __syncthreads();
  (void)Pc;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (Nc + 1) * (Nc + 2) / 2) return;
  const int64_t T = blockIdx.y;
  int i, j;
  col_of(c, i, j);
  const uint16_t om = own[T];
  const double* r = rf + T * Sf;
  double* out = fc + T * Sc + c;
  const int fi = 2 * i, fj = 2 * j;
  for (int k = 0; k <= Nc - i - j; ++k) {
    const int fk = 2 * k;
    double acc = owns(om, Nf, fi, fj, fk) ? r[lpos(pof, fi, fj, fk)] : 0.0;
    double half = 0.0;
    for (int w = 0; w < 15; ++w) {
      if (w == kMC) continue;
      const int a = fi + kDir[w][0], b = fj + kDir[w][1], cc = fk + kDir[w][2];
      if (a < 0 || b < 0 || cc < 0 || a + b + cc > Nf) continue;
      if (owns(om, Nf, a, b, cc)) half += r[lpos(pof, a, b, cc)];
    }
    out[poc[k]] = acc + 0.5 * half;
  }
}

// u_f += P u_c at every fine lattice node of every macro: thread = fine lattice
// column (i, j) of macro blockIdx.y, marching k
__global__ void k_prolong_add(int Nf, int64_t Sf, int64_t Sc, int64_t Pf, const double* __restrict__ uc,
                              double* __restrict__ uf) {
  __shared__ int64_t pof[258], poc[130];
  const int Nc = Nf / 2;
  for (int k = threadIdx.x; k <= Nf; k += blockDim.x) pof[k] = plane_off(Nf, k);
  for (int k = threadIdx.x; k <= Nc; k += blockDim.x) poc[k] = plane_off(Nc, k);
  __syncthreads();
  (void)Pf;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= (Nf + 1) * (Nf + 2) / 2) return;
  const int64_t T = blockIdx.y;
  int i, j;
  col_of(col, i, j);
  const double* cu = uc + T * Sc;
  double* out = uf + T * Sf + col;
  for (int k = 0; k <= Nf - i - j; ++k) {
    const int par = (i & 1) | ((j & 1) << 1) | ((k & 1) << 2);
    double v;
    if (par == 0) {
      v = cu[lpos(poc, i / 2, j / 2, k / 2)];
    } else {
      const int* d = kParityDir[par];
      v = 0.5 * (cu[lpos(poc, (i - d[0]) / 2, (j - d[1]) / 2, (k - d[2]) / 2)] +
                 cu[lpos(poc, (i + d[0]) / 2, (j + d[1]) / 2, (k + d[2]) / 2)]);
    }
    out[pof[k]] += v;
  }
}

// CG vector updates with device scalars s[0] = rr, s[1] = pAp, s[2] = rr_new
__global__ void k_cg_update1(int64_t n, const double* __restrict__ s, double* __restrict__ x,
                             double* __restrict__ r, const double* __restrict__ p, const double* __restrict__ Ap) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double alpha = s[1] != 0.0 ? s[0] / s[1] : 0.0;
  x[t] += alpha * p[t];
  r[t] -= alpha * Ap[t];
}

__global__ void k_cg_update2(int64_t n, const double* __restrict__ s, const double* __restrict__ r,
                             double* __restrict__ p) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double beta = s[0] != 0.0 ? s[2] / s[0] : 0.0;
  p[t] = r[t] + beta * p[t];
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

static hhg_status ensure_mg(Ctx* c) {
  if (!c->d_own) {
    HHG_CK(c, cudaMalloc(&c->d_own, std::max<size_t>(c->own.size(), 1) * sizeof(uint16_t)));
    HHG_CK(c, cudaMemcpy(c->d_own, c->own.data(), c->own.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
  }
  if ((int)c->vc_u.size() <= c->L_max) {
    c->vc_u.assign(c->L_max + 1, nullptr);
    c->vc_f.assign(c->L_max + 1, nullptr);
    c->vc_r.assign(c->L_max + 1, nullptr);
  }
  if (!c->d_scal) HHG_CK(c, cudaMalloc(&c->d_scal, 8 * sizeof(double)));
  return HHG_OK;
}

static hhg_status level_vec(Ctx* c, std::vector<double*>& v, int L) {
  if (!v[L]) {
    HHG_CK(c, cudaMalloc(&v[L], c->levels[L].n_local * sizeof(double)));
    HHG_CK(c, cudaMemsetAsync(v[L], 0, c->levels[L].n_local * sizeof(double), c->stream));
  }
  return HHG_OK;
}

// Coarse solver selection: the replicated CSR solve (coarse.cu, default) or CG
// through the library's operator calls (one apply, three dot products and two
// updates per iteration; the same recurrence) -- for coarse levels too large to
// replicate (coarse_replicable), or forced with HHG_COARSE=ops.
static bool coarse_ops() {
  const char* e = getenv("HHG_COARSE");  // read per call (tests compare both solvers)
  return e && std::string(e) == "ops";
}

// x = A^-1 b by `iters` CG iterations from x = 0 on the exact FEM operator
// (surrogate at L = 2 is the exact stencil; above, the node-wise FEM operator).
static hhg_status coarse_cg_ops(Ctx* c, int L, int iters, double* x, const double* b) {
  Level& lv = c->levels[L];
  const int64_t n = lv.n_local;
  const int op = L == 2 ? HHG_OP_SURROGATE : HHG_OP_FEM_ELEMENTWISE;
  if (!c->d_cg || c->cg_n < n) {
    if (c->d_cg) cudaFree(c->d_cg);
    HHG_CK(c, cudaMalloc(&c->d_cg, 3 * n * sizeof(double)));
    HHG_CK(c, cudaMemsetAsync(c->d_cg, 0, 3 * n * sizeof(double), c->stream));
    c->cg_n = n;
  }
  double *r = c->d_cg, *p = c->d_cg + n, *Ap = c->d_cg + 2 * n;
  double* s = c->d_scal;
  hhg_status st;
  HHG_CK(c, cudaMemsetAsync(x, 0, n * sizeof(double), c->stream));
  HHG_CK(c, cudaMemcpyAsync(r, b, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  HHG_CK(c, cudaMemcpyAsync(p, b, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  if ((st = dot_dev(c, lv, r, r, s + 0)) != HHG_OK) return st;
  for (int it = 0; it < iters; ++it) {
    if ((st = apply_dev(c, lv, op, 0, p, nullptr, Ap)) != HHG_OK) return st;
    if ((st = dot_dev(c, lv, p, Ap, s + 1)) != HHG_OK) return st;
    k_cg_update1<<<nblk(n, 256), 256, 0, c->stream>>>(n, s, x, r, p, Ap);
    HHG_LAUNCHED(c);
    if ((st = dot_dev(c, lv, r, r, s + 2)) != HHG_OK) return st;
    k_cg_update2<<<nblk(n, 256), 256, 0, c->stream>>>(n, s, r, p);
    HHG_LAUNCHED(c);
    HHG_CK(c, cudaMemcpyAsync(s + 0, s + 2, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  }
  return HHG_OK;
}

static hhg_status restrict_to(Ctx* c, int Lf, const double* rf, double* fc) {
  Level& F = c->levels[Lf];
  Level& C = c->levels[Lf - 1];
  dim3 grid(nblk((int64_t)(C.N + 1) * (C.N + 2) / 2, 128), (unsigned)c->nt_local);  // coarse columns
  hhg_status st;
  if (c->nt_blocks > c->nt_local)  // ghost blocks hold no partial sums
    HHG_CK(c, cudaMemsetAsync(fc + c->nt_local * C.S, 0, (c->nt_blocks - c->nt_local) * C.S * sizeof(double),
                              c->stream));
  k_restrict_partial<<<grid, 128, 0, c->stream>>>(F.N, F.S, C.S, C.P, c->d_own, rf, fc);
  HHG_LAUNCHED(c);
  // multi-rank: the partials at the copies of shared coarse nodes on other
  // ranks are added into the owner's slot first, then every rank sums its own
  // rows' local copies, then the owners' totals go back to every copy
  if ((st = dist_sum_to_owner(c, C, fc)) != HHG_OK) return st;
  if ((st = lp_sum_copies(c, C, fc)) != HHG_OK) return st;
  if ((st = zero_dir_slots(c, C, fc)) != HHG_OK) return st;
  return dist_sync(c, C, fc);
}

static hhg_status prolong_add(Ctx* c, int Lf, const double* uc, double* uf) {
  Level& F = c->levels[Lf];
  Level& C = c->levels[Lf - 1];
  dim3 grid(nblk((int64_t)(F.N + 1) * (F.N + 2) / 2, 128), (unsigned)c->nt_local);  // fine columns
  k_prolong_add<<<grid, 128, 0, c->stream>>>(F.N, F.S, C.S, F.P, uc, uf);
  HHG_LAUNCHED(c);
  if (c->nranks > 1) {  // ghost-block copies of this rank's own nodes, then the other ranks' values
    hhg_status st = lp_sync_own_copies(c, F, uf);
    if (st != HHG_OK) return st;
  }
  return dist_sync(c, F, uf);  // ghost-block slots of the other ranks' macros
}

// op: smoother; rop: residual operator (= op, or the exact FEM operator for
// double discretisation)
static hhg_status vcycle_rec(Ctx* c, int L, int Lc, int nu1, int nu2, int cg_iters, int op, int rop, bool lex,
                             double* u, const double* f) {
  hhg_status st;
  if (L == Lc)
    return coarse_ops() || !coarse_replicable(c->levels[L]) ? coarse_cg_ops(c, L, cg_iters, u, f)
                                                            : coarse_solve(c, c->levels[L], cg_iters, u, f);
  Level& lv = c->levels[L];
  for (int s = 0; s < nu1; ++s)
    if ((st = gs_sweep_dev(c, lv, op, u, f, lex)) != HHG_OK) return st;
  if ((st = level_vec(c, c->vc_r, L)) != HHG_OK) return st;
  if ((st = level_vec(c, c->vc_u, L - 1)) != HHG_OK) return st;
  if ((st = level_vec(c, c->vc_f, L - 1)) != HHG_OK) return st;
  if ((st = apply_dev(c, lv, rop, 1 /*residual*/, u, f, c->vc_r[L])) != HHG_OK) return st;
  if ((st = restrict_to(c, L, c->vc_r[L], c->vc_f[L - 1])) != HHG_OK) return st;
  HHG_CK(c, cudaMemsetAsync(c->vc_u[L - 1], 0, c->levels[L - 1].n_local * sizeof(double), c->stream));
  if ((st = vcycle_rec(c, L - 1, Lc, nu1, nu2, cg_iters, op, rop, lex, c->vc_u[L - 1], c->vc_f[L - 1])) != HHG_OK)
    return st;
  if ((st = prolong_add(c, L, c->vc_u[L - 1], u)) != HHG_OK) return st;
  for (int s = 0; s < nu2; ++s)
    if ((st = gs_sweep_dev(c, lv, op, u, f, lex)) != HHG_OK) return st;
  return HHG_OK;
}

}  // namespace hhg

using namespace hhg;

static hhg_status vcycle_impl(Ctx* c, int L, int nu1, int nu2, int L_coarse, int coarse_cg_iters, hhg_op op,
                              hhg_op rop, bool lex, double* u, const double* f, int n_cycles, double* res_hist);

extern "C" hhg_status hhg_vcycle(hhg_ctx ctx, int L, int nu1, int nu2, int L_coarse, int coarse_cg_iters,
                                 hhg_op op, double* u, const double* f, int n_cycles, double* res_hist) {
  return vcycle_impl((Ctx*)ctx, L, nu1, nu2, L_coarse, coarse_cg_iters, op, op, false, u, f, n_cycles, res_hist);
}

extern "C" hhg_status hhg_vcycle_dd(hhg_ctx ctx, int L, int nu1, int nu2, int L_coarse, int coarse_cg_iters,
                                    hhg_op smoother_op, hhg_op residual_op, double* u, const double* f,
                                    int n_cycles, double* res_hist) {
  Ctx* c = (Ctx*)ctx;
  if (c && residual_op != HHG_OP_SURROGATE && residual_op != HHG_OP_FEM_ELEMENTWISE &&
      residual_op != HHG_OP_CONST_AFFINE && residual_op != HHG_OP_SURROGATE_FACES)
    return set_err(c, HHG_ERR_INVALID, "hhg_vcycle_dd: residual_op");
  return vcycle_impl(c, L, nu1, nu2, L_coarse, coarse_cg_iters, smoother_op, residual_op, false, u, f, n_cycles,
                     res_hist);
}

extern "C" hhg_status hhg_vcycle_ex(hhg_ctx ctx, int L, int nu1, int nu2, int L_coarse, int coarse_cg_iters,
                                    hhg_op smoother_op, hhg_op residual_op, int lexicographic, double* u,
                                    const double* f, int n_cycles, double* res_hist) {
  Ctx* c = (Ctx*)ctx;
  if (c && residual_op != HHG_OP_SURROGATE && residual_op != HHG_OP_FEM_ELEMENTWISE &&
      residual_op != HHG_OP_CONST_AFFINE && residual_op != HHG_OP_SURROGATE_FACES)
    return set_err(c, HHG_ERR_INVALID, "hhg_vcycle_ex: residual_op");
  return vcycle_impl(c, L, nu1, nu2, L_coarse, coarse_cg_iters, smoother_op, residual_op, lexicographic != 0, u,
                     f, n_cycles, res_hist);
}

static hhg_status vcycle_impl(Ctx* c, int L, int nu1, int nu2, int L_coarse, int coarse_cg_iters, hhg_op op,
                              hhg_op rop, bool lex, double* u, const double* f, int n_cycles, double* res_hist) {
  if (!c) return HHG_ERR_INVALID;
  if (c->poisoned) return HHG_ERR_CUDA;
  if (L < 2 || L > c->L_max || L_coarse < 2 || L_coarse > L || nu1 < 0 || nu2 < 0 || coarse_cg_iters < 0 ||
      n_cycles < 0 || !u || !f || (const double*)u == f)
    return set_err(c, HHG_ERR_INVALID, "hhg_vcycle: bad arguments");
  if (op != HHG_OP_SURROGATE && op != HHG_OP_CONST_AFFINE && op != HHG_OP_SURROGATE_FACES)
    return set_err(c, HHG_ERR_INVALID, "hhg_vcycle: smoother op must be SURROGATE(_FACES) or CONST_AFFINE");
  if (c->host_only)
    return set_err(c, HHG_ERR_INVALID, "hhg_vcycle: needs device vectors (host_only context)");
  hhg_status st;
  for (int l = L_coarse; l <= L; ++l) {
    if (!c->levels[l].fitted) return set_err(c, HHG_ERR_STATE, "hhg_vcycle: call hhg_fit_surrogates first");
    if (l > L_coarse && (st = check_centre_ok(c, c->levels[l], op)) != HHG_OK) return st;
  }
  st = ensure_mg(c);
  if (st != HHG_OK) return st;
  // the coarse matrix is assembled once per level (collective, synchronising:
  // never inside a graph capture)
  if (!coarse_ops() && coarse_replicable(c->levels[L_coarse]) && (st = coarse_build(c, c->levels[L_coarse])) != HHG_OK)
    return st;
  Level& lv = c->levels[L];
  const int64_t n = lv.n_local;
  // host vectors are staged
  cudaPointerAttributes au, af;
  const bool hu = cudaPointerGetAttributes(&au, u) != cudaSuccess || au.type == cudaMemoryTypeHost ||
                  au.type == cudaMemoryTypeUnregistered;
  cudaGetLastError();
  const bool hf = cudaPointerGetAttributes(&af, f) != cudaSuccess || af.type == cudaMemoryTypeHost ||
                  af.type == cudaMemoryTypeUnregistered;
  cudaGetLastError();
  double* du = u;
  const double* df = f;
  double* stage_u = nullptr;
  double* stage_f = nullptr;
  if (hu) {
    HHG_CK(c, cudaMalloc(&stage_u, n * sizeof(double)));
    HHG_CK(c, cudaMemcpyAsync(stage_u, u, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    du = stage_u;
  }
  if (hf) {
    HHG_CK(c, cudaMalloc(&stage_f, n * sizeof(double)));
    HHG_CK(c, cudaMemcpyAsync(stage_f, f, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    df = stage_f;
  }
  if ((st = level_vec(c, c->vc_r, L)) != HHG_OK) return st;
  double nr = 0.0;
  int grow = 0;
  double prev = 0.0;
  hhg_status result = HHG_OK;
  auto resnorm = [&](double* out) -> hhg_status {
    hhg_status s2 = apply_dev(c, lv, rop, 1, du, df, c->vc_r[L]);
    if (s2 != HHG_OK) return s2;
    return norm2_of(c, lv, c->vc_r[L], out);
  };
  if (res_hist) {
    if ((st = resnorm(&nr)) != HHG_OK) return st;
    res_hist[0] = nr;
    prev = nr;
  }
  // HHG_VCYCLE_GRAPH=1: cycles after the first (which allocates the level
  // vectors and sizes the persistent grids) replay one captured CUDA graph,
  // cached on the ctx for later calls with the same signature.  Measured on the
  // 480-macro L = 7 shell: a replay saves ~2 ms of launch overhead per cycle
  // (coarse levels 4.0 -> 2.6 ms), but capture + instantiation of the ~1050
  // nodes costs ~130 ms, so it pays only across many calls -- off by default.
  // Never with the host transport (host callbacks), while profiling, or with
  // the experimental GS variants.
  const char* ge = getenv("HHG_VCYCLE_GRAPH");
  bool use_graph = ge && atoi(ge) == 1 && c->transport != 2 && !c->prof && !getenv("HHG_COARSE") &&
                   !getenv("HHG_GS_KERNEL");
  // the graph is cached on the ctx and reused by later calls with the same
  // signature (levels, smoother, vectors)
  const std::vector<int64_t> key = {L, L_coarse, nu1, nu2, coarse_cg_iters, (int64_t)op, (int64_t)rop, (int64_t)lex,
                                    (int64_t)(intptr_t)du,
                                    (int64_t)(intptr_t)df};
  if (c->vc_graph && c->vc_graph_key != key) {
    cudaGraphExecDestroy(c->vc_graph);
    c->vc_graph = nullptr;
  }
  cudaGraphExec_t& gexec = c->vc_graph;
  int64_t& graph_launches = c->vc_graph_launches;
  for (int cyc = 0; cyc < n_cycles; ++cyc) {
    if ((cyc == 0 && !gexec) || !use_graph) {
      if ((st = vcycle_rec(c, L, L_coarse, nu1, nu2, coarse_cg_iters, op, rop, lex, du, df)) != HHG_OK) return st;
    } else {
      if (!gexec) {
        cudaGraph_t graph = nullptr;
        const int64_t l0 = c->launches;
        // capture on a private stream (the legacy default stream cannot be
        // captured); nothing executes during capture, the replay goes to c->stream
        if (!c->cap_stream) HHG_CK(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
        cudaStream_t orig = c->stream;
        c->stream = c->cap_stream;
        const cudaError_t eb = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
        if (eb != cudaSuccess) {
          c->stream = orig;
          HHG_CK(c, eb);
        }
        st = vcycle_rec(c, L, L_coarse, nu1, nu2, coarse_cg_iters, op, rop, lex, du, df);
        const cudaError_t ee = cudaStreamEndCapture(c->stream, &graph);
        c->stream = orig;
        if (st != HHG_OK) {
          if (graph) cudaGraphDestroy(graph);
          return st;
        }
        HHG_CK(c, ee);
        graph_launches = c->launches - l0;
        c->launches = l0;
        const cudaError_t ei = cudaGraphInstantiate(&gexec, graph, 0);
        cudaGraphDestroy(graph);
        HHG_CK(c, ei);
        c->vc_graph_key = key;
      }
      HHG_CK(c, cudaGraphLaunch(gexec, c->stream));
      c->launches += graph_launches;
    }
    if (res_hist) {
      if ((st = resnorm(&nr)) != HHG_OK) return st;
      res_hist[cyc + 1] = nr;
      // not for double discretisation: its exact-operator residual stalls and may
      // creep up by design (residual criteria inappropriate)
      grow = (nr > prev && rop == op) ? grow + 1 : 0;
      prev = nr;
      if (grow >= 3) {
        result = set_err(c, HHG_ERR_DIVERGED, "V-cycle residual grew three cycles in a row");
        for (int q = cyc + 2; q <= n_cycles; ++q) res_hist[q] = nr;
        break;
      }
    }
  }
  if (hu) {
    HHG_CK(c, cudaMemcpyAsync(u, stage_u, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
  { hhg_status st_sync__ = ctx_sync(c); if (st_sync__ != HHG_OK) return st_sync__; }
  if (stage_u) cudaFree(stage_u);
  if (stage_f) cudaFree(stage_f);
  return result;
}
