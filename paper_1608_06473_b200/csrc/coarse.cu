// Replicated coarse solve of the V-cycle (BASELINE
// config 5: "coarsest L=2: 50 CG iterations from zero on the exact FEM
// operator", R19).
//
// The coarse operator is assembled ONCE per level into a CSR matrix over the
// canonical global unknown ids (every rank dumps the rows it owns as COO,
// the COO is all-gathered and sorted by (row, column), so every rank holds the
// identical matrix).  A solve is then: owned entries of b into a global vector
// (0 elsewhere), one all-reduce (sum over ranks = b), all CG iterations in ONE
// cooperative kernel (grid-wide barriers between the SpMV, the two updates
// and the direction update; dot products as fixed-order block partials, so the
// iterate is bitwise identical on every rank), and a scatter of x into every
// local copy.  That replaces ~14 launches per CG iteration (~700 per cycle at
// 50 iterations, launch-bound at L = 2) by a handful per solve.
//
// Rows (all exact FEM, blended geometry):
//   volume interior nodes of the local macros: fem_partial (24 tets, one macro);
//   structured face rows: the stored d_fval (both macros summed);
//   vertex/edge rows: the stored CSR (d_val, slot columns).
// Columns of Dirichlet nodes are kept: b, x, r, p are 0 there (no row), so
// they never contribute.
#include <cooperative_groups.h>

#include <algorithm>
#include <numeric>

#include "faces.cuh"

namespace cg = cooperative_groups;

namespace hhg {

struct CooEntry {
  int64_t row, col;
  double val;
};

__device__ __forceinline__ int64_t slot_gid(const GidInfo& g, const MacroTopo* topo, int64_t S, int64_t slot) {
  const int64_t T = slot / S;
  int i, j, k;
  decode_pos(g.N, slot - T * S, i, j, k);
  return node_gid(g, topo[T], i, j, k);
}

__device__ __forceinline__ void coo_push(CooEntry* out, unsigned long long* cnt, const CooEntry* e, int n) {
  if (n == 0) return;
  const unsigned long long o = atomicAdd(cnt, (unsigned long long)n);
  for (int x = 0; x < n; ++x) out[o + x] = e[x];
}

__global__ void k_coarse_vol_coo(int N, int64_t P, const MacroTopo* __restrict__ topo, GidInfo gi,
                                 const double* __restrict__ geo, bool blended, CooEntry* out,
                                 unsigned long long* cnt) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t T = blockIdx.y;
  if (p >= P) return;
  int i, j, k;
  decode_pos(N, p, i, j, k);
  if (i < 1 || j < 1 || k < 1 || i + j + k > N - 1) return;
  double part[15];
  fem_partial(geo + T * 16, N, i, j, k, blended, part);
  const int64_t row = node_gid(gi, topo[T], i, j, k);
  CooEntry e[15];
  for (int w = 0; w < 15; ++w)
    e[w] = CooEntry{row, node_gid(gi, topo[T], i + kDir[w][0], j + kDir[w][1], k + kDir[w][2]), part[w]};
  coo_push(out, cnt, e, 15);
}

__global__ void k_coarse_face_coo(int N, int64_t S, int64_t nfi, int64_t n_frows, const FaceLP* __restrict__ flp,
                                  const uint32_t* __restrict__ fst, const int* __restrict__ fcidx,
                                  const int* __restrict__ po, const MacroTopo* __restrict__ topo, GidInfo gi,
                                  const double* __restrict__ val, CooEntry* out, unsigned long long* cnt) {
  __shared__ int po_s[260];
  load_po(po_s, po, N);
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_frows) return;
  const int64_t fc = r / nfi, q = r - fc * nfi;
  const FaceLP& F = flp[fc];
  const uint32_t st = fst[F.z * nfi + q];
  FaceRowSlots o;
  face_row_slots(F, N, S, po_s, st & 0xffff, st >> 16, o);
  const int64_t row = gi.base_f + F.fid * nfi + fcidx[F.z * nfi + q];
  CooEntry e[15];
  int n = 0;
  e[n++] = CooEntry{row, row, val[r]};
  for (int x = 0; x < 14; ++x)
    if (o.nb[x] >= 0) e[n++] = CooEntry{row, slot_gid(gi, topo, S, o.nb[x]), val[(x + 1) * n_frows + r]};
  coo_push(out, cnt, e, n);
}

__global__ void k_coarse_lp_coo(int64_t n_rows, int64_t S, const uint64_t* __restrict__ rp,
                                const uint32_t* __restrict__ col, const double* __restrict__ val,
                                const int64_t* __restrict__ row_gid, const MacroTopo* __restrict__ topo, GidInfo gi,
                                CooEntry* out, unsigned long long* cnt) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int64_t row = row_gid[r];
  for (uint64_t e = rp[r]; e < rp[r + 1]; ++e) {
    const CooEntry x{row, e == rp[r] ? row : slot_gid(gi, topo, S, col[e]), val[e]};
    coo_push(out, cnt, &x, 1);
  }
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

constexpr int kCgThreads = 256;
#ifndef HHG_CG_ROWS
#define HHG_CG_ROWS 1
#endif
constexpr int kCgRows = HHG_CG_ROWS;  // rows per thread (grid sizing)

// sum of the grid's block partials, fixed order (warp 0), broadcast to the block
__device__ __forceinline__ double grid_total(const double* part, int nparts, double* sh) {
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (int x = threadIdx.x; x < nparts; x += 32) v += part[x];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) sh[0] = v;
  }
  __syncthreads();
  const double t = sh[0];
  __syncthreads();
  return t;
}

__device__ __forceinline__ void block_partial(double v, double* out, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) *out = v;
  }
  __syncthreads();
}

// `iters` CG iterations from x = 0 (alpha = rr / pAp, beta = rr_new / rr, 0 on
// a zero denominator -- the same recurrence as the oracle's cg and the
// operator-based coarse_cg_ops), the whole loop in one cooperative launch.
__global__ void __launch_bounds__(kCgThreads) k_cg_coop(int64_t n, const int* __restrict__ rp,
                                                        const int* __restrict__ col,
                                                        const double* __restrict__ val, double* __restrict__ vec,
                                                        double* __restrict__ part, int iters) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[33];
  const double* b = vec;
  double* x = vec + n;
  double* r = vec + 2 * n;
  double* p = vec + 3 * n;
  double* Ap = vec + 4 * n;
  const int G = gridDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)G * blockDim.x;
  double acc = 0.0;
  for (int64_t i = t0; i < n; i += nth) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    p[i] = bi;
    acc = fma(bi, bi, acc);
  }
  block_partial(acc, part + blockIdx.x, sh);
  grid.sync();
  double rr = grid_total(part, G, sh);
  for (int it = 0; it < iters; ++it) {
    acc = 0.0;
    for (int64_t i = t0; i < n; i += nth) {
      // row in CSR order (one fma chain); the gathers of 4 entries are issued
      // together (the loop is L2-latency-bound otherwise)
      double s = 0.0;
      int e = rp[i];
      const int e1 = rp[i + 1];
      for (; e + 4 <= e1; e += 4) {
        const int c0 = col[e], c1 = col[e + 1], c2 = col[e + 2], c3 = col[e + 3];
        const double v0 = val[e], v1 = val[e + 1], v2 = val[e + 2], v3 = val[e + 3];
        const double p0 = p[c0], p1 = p[c1], p2 = p[c2], p3 = p[c3];
        s = fma(v0, p0, s);
        s = fma(v1, p1, s);
        s = fma(v2, p2, s);
        s = fma(v3, p3, s);
      }
      for (; e < e1; ++e) s = fma(val[e], p[col[e]], s);
      Ap[i] = s;
      acc = fma(p[i], s, acc);
    }
    block_partial(acc, part + G + blockIdx.x, sh);
    grid.sync();
    const double pAp = grid_total(part + G, G, sh);
    const double alpha = pAp != 0.0 ? rr / pAp : 0.0;
    acc = 0.0;
    for (int64_t i = t0; i < n; i += nth) {
      x[i] = fma(alpha, p[i], x[i]);
      const double ri = fma(-alpha, Ap[i], r[i]);
      r[i] = ri;
      acc = fma(ri, ri, acc);
    }
    block_partial(acc, part + 2 * G + blockIdx.x, sh);
    grid.sync();
    const double rrn = grid_total(part + 2 * G, G, sh);
    const double beta = rr != 0.0 ? rrn / rr : 0.0;
    for (int64_t i = t0; i < n; i += nth) p[i] = fma(beta, p[i], r[i]);
    rr = rrn;
    grid.sync();
  }
}

// The replicated solve holds the level's whole CSR matrix on every rank (int32
// row pointers and columns) and sorts its COO on the host: only for levels of
// at most kCoarseMaxUnknowns unknowns (~15 entries per row: <= 63 M entries,
// 1.5 GB of COO); larger coarse levels use the CG through the operator calls
// (vcycle.cu::coarse_cg_ops).
bool coarse_replicable(const Level& lv) { return lv.gi.n_total <= kCoarseMaxUnknowns; }

hhg_status coarse_build(Ctx* c, Level& lv) {
  if (lv.cg_built) return HHG_OK;
  const GidInfo& gi = lv.gi;
  const int64_t n = gi.n_total;
  if (!coarse_replicable(lv)) return set_err(c, HHG_ERR_INVALID, "coarse level too large for the replicated solve");
  const int64_t cap = c->nt_local * gi.nvi * 15 + lv.n_frows * 15 + lv.nnz;
  CooEntry* d_coo = nullptr;
  unsigned long long* d_cnt = nullptr;
  HHG_CK(c, cudaMalloc(&d_coo, std::max<int64_t>(cap, 1) * sizeof(CooEntry)));
  HHG_CK(c, cudaMalloc(&d_cnt, sizeof(unsigned long long)));
  HHG_CK(c, cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), c->stream));
  if (c->nt_local > 0) {
    dim3 grid(nblk(lv.P, 128), (unsigned)c->nt_local);
    k_coarse_vol_coo<<<grid, 128, 0, c->stream>>>(lv.N, lv.P, c->d_topo, gi, c->d_geo, c->blended, d_coo, d_cnt);
    HHG_LAUNCHED(c);
  }
  if (lv.n_frows) {
    k_coarse_face_coo<<<nblk(lv.n_frows, 128), 128, 0, c->stream>>>(
        lv.N, lv.S, gi.nfi, lv.n_frows, lv.d_flp, lv.d_fst, lv.d_fcidx, lv.d_po, c->d_topo, gi, lv.d_fval, d_coo,
        d_cnt);
    HHG_LAUNCHED(c);
  }
  if (lv.n_rows) {
    k_coarse_lp_coo<<<nblk(lv.n_rows, 128), 128, 0, c->stream>>>(lv.n_rows, lv.S, lv.d_row_ptr, lv.d_col, lv.d_val,
                                                                 lv.d_row_gid, c->d_topo, gi, d_coo, d_cnt);
    HHG_LAUNCHED(c);
  }
  unsigned long long cnt = 0;
  HHG_CK(c, cudaMemcpyAsync(&cnt, d_cnt, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
  { hhg_status st_sync__ = ctx_sync(c); if (st_sync__ != HHG_OK) return st_sync__; }
  if ((int64_t)cnt > cap) return set_err(c, HHG_ERR_STATE, "coarse COO overflow");
  std::vector<CooEntry> coo(cnt);
  HHG_CK(c, cudaMemcpy(coo.data(), d_coo, cnt * sizeof(CooEntry), cudaMemcpyDeviceToHost));
  cudaFree(d_coo);
  cudaFree(d_cnt);
  // all-gather the ranks' rows (counts first)
  if (c->nranks > 1) {
    const int nr = c->nranks;
    std::vector<int64_t> cnt_send(nr, (int64_t)cnt), cnt_recv(nr, 0);
    std::vector<int64_t> b8(nr, 8);
    hhg_status st = dist_exchange_bytes(c, b8, cnt_send.data(), b8, cnt_recv.data(), false, c->stream);
    if (st != HHG_OK) return st;
    std::vector<int64_t> sb(nr), rb(nr);
    int64_t tot = 0;
    for (int p = 0; p < nr; ++p) {
      sb[p] = p == c->rank ? 0 : (int64_t)cnt * (int64_t)sizeof(CooEntry);
      rb[p] = p == c->rank ? 0 : cnt_recv[p] * (int64_t)sizeof(CooEntry);
      if (p != c->rank) tot += cnt_recv[p];
    }
    std::vector<CooEntry> sendv((size_t)cnt * (nr - 1)), recvv((size_t)tot);
    for (int q = 0; q < nr - 1; ++q) std::copy(coo.begin(), coo.end(), sendv.begin() + (size_t)q * cnt);
    st = dist_exchange_bytes(c, sb, sendv.data(), rb, recvv.data(), false, c->stream);
    if (st != HHG_OK) return st;
    coo.insert(coo.end(), recvv.begin(), recvv.end());
  }
  if ((int64_t)coo.size() >= (1ll << 31) - 1)
    return set_err(c, HHG_ERR_INVALID, "coarse matrix too large for 32-bit CSR indices");
  std::sort(coo.begin(), coo.end(), [](const CooEntry& a, const CooEntry& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  std::vector<int> rp(n + 1, 0), col;
  std::vector<double> val;
  col.reserve(coo.size());
  val.reserve(coo.size());
  for (size_t x = 0; x < coo.size(); ++x) {
    const CooEntry& e = coo[x];
    if (e.row < 0 || e.row >= n || e.col < 0 || e.col >= n) return set_err(c, HHG_ERR_STATE, "coarse COO index");
    if (x > 0 && coo[x - 1].row == e.row && coo[x - 1].col == e.col) {
      val.back() += e.val;
      continue;
    }
    col.push_back((int)e.col);
    val.push_back(e.val);
    rp[e.row + 1]++;
  }
  for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
  lv.cg_nnz = (int64_t)col.size();
  HHG_CK(c, cudaMalloc(&lv.d_cg_rp, (n + 1) * sizeof(int)));
  HHG_CK(c, cudaMalloc(&lv.d_cg_col, std::max<int64_t>(lv.cg_nnz, 1) * sizeof(int)));
  HHG_CK(c, cudaMalloc(&lv.d_cg_val, std::max<int64_t>(lv.cg_nnz, 1) * sizeof(double)));
  HHG_CK(c, cudaMalloc(&lv.d_cg_vec, 5 * std::max<int64_t>(n, 1) * sizeof(double)));
  HHG_CK(c, cudaMemcpy(lv.d_cg_rp, rp.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice));
  if (lv.cg_nnz) {
    HHG_CK(c, cudaMemcpy(lv.d_cg_col, col.data(), lv.cg_nnz * sizeof(int), cudaMemcpyHostToDevice));
    HHG_CK(c, cudaMemcpy(lv.d_cg_val, val.data(), lv.cg_nnz * sizeof(double), cudaMemcpyHostToDevice));
  }
  int dev = 0, nsm = 0, per_sm = 0;
  HHG_CK(c, cudaGetDevice(&dev));
  HHG_CK(c, cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  HHG_CK(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_coop, kCgThreads, 0));
  // one row per thread while the grid stays co-resident (the SpMV rows are
  // L2-latency-bound; measured: 8 rows per thread, 3 CTAs at L = 2 on the
  // 480-macro shell, 1.83 ms for 50 iterations)
  lv.cg_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * std::max(per_sm, 1),
                                                           (n + kCgRows * kCgThreads - 1) / (kCgRows * kCgThreads)));
  HHG_CK(c, cudaMalloc(&lv.d_cg_part, 3 * lv.cg_grid * sizeof(double)));
  lv.cg_built = true;
  return HHG_OK;
}

hhg_status coarse_solve(Ctx* c, Level& lv, int iters, double* x, const double* b) {
  hhg_status st;
  if ((st = coarse_build(c, lv)) != HHG_OK) return st;
  const int64_t n = lv.gi.n_total;
  double* vb = lv.d_cg_vec;
  if ((st = gather_owned_dev(c, lv, b, vb)) != HHG_OK) return st;
  if ((st = dist_allreduce_vec(c, vb, n)) != HHG_OK) return st;
  int64_t nn = n;
  void* args[] = {&nn, &lv.d_cg_rp, &lv.d_cg_col, &lv.d_cg_val, &lv.d_cg_vec, &lv.d_cg_part, &iters};
  HHG_CK(c, cudaLaunchCooperativeKernel((const void*)k_cg_coop, dim3((unsigned)lv.cg_grid), dim3(kCgThreads), args, 0,
                                        c->stream));
  HHG_LAUNCHED(c);
  return scatter_global_dev(c, lv, lv.d_cg_vec + n, x);
}

}  // namespace hhg
