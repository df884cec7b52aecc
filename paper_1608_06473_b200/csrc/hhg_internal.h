// Internal declarations of libhhg (not part of the ABI; see include/hhg.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <functional>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "../../include/hhg.h"

namespace hhg {

// ---------------------------------------------------------------------------
// Stencil directions (reading R7); opposite(w) = 14 - w.
// ---------------------------------------------------------------------------
constexpr int kMC = 7;
// L~ with surrogate face rows too; the public enum value
// HHG_OP_SURROGATE_FACES lives in include/hhg.h
#define HHG_DIRS_INIT                                                                     \
  {{0, 0, -1}, {1, 0, -1}, {0, 1, -1}, {-1, 1, -1}, {0, -1, 0}, {1, -1, 0}, {-1, 0, 0}, \
   {0, 0, 0},  {1, 0, 0},  {-1, 1, 0}, {0, 1, 0},   {1, -1, 1}, {0, -1, 1}, {-1, 0, 1}, \
   {0, 0, 1}}
extern const int kDirHost[15][3];

// ---------------------------------------------------------------------------
// Lattice layout helpers (host + device).  pos(i,j,k) = planeoff(k) + col(i,j)
// ---------------------------------------------------------------------------
__host__ __device__ inline int64_t tri3(int64_t M) { return (M + 1) * (M + 2) * (M + 3) / 6; }
__host__ __device__ inline int64_t plane_off(int N, int k) { return tri3(N) - tri3(N - k); }
__host__ __device__ inline int64_t col_idx(int i, int j) {
  int64_t d = i + j;
  return d * (d + 1) / 2 + j;
}
__host__ __device__ inline int64_t lattice_pos(int N, int i, int j, int k) {
  return plane_off(N, k) + col_idx(i, j);
}
__host__ __device__ inline int64_t n_lattice(int N) { return tri3(N); }
__host__ __device__ inline int64_t n_interior(int N) {
  return (int64_t)(N - 1) * (N - 2) * (N - 3) / 6;
}
// canonical volume index (k outer, j, i inner) of interior node (DESIGN.md numbering)
__host__ __device__ inline int64_t vol_index(int N, int i, int j, int k) {
  int64_t M = N - 1 - k;
  auto c3 = [](int64_t n) { return n * (n - 1) * (n - 2) / 6; };
  return (c3(N - 1) - c3(M + 1)) + (int64_t)(j - 1) * M - (int64_t)(j - 1) * j / 2 + (i - 1);
}

// Per-level geometry of the canonical numbering.
struct GidInfo {
  int N;
  int64_t nv, n_e, n_f;
  int64_t nfi, nvi;
  int64_t base_e, base_f, base_v, n_total;
};

// Topology tables of one macro (global ids) -- host and device copies.
struct MacroTopo {
  int64_t gv[4];   // global vertex ids of local vertices
  int64_t e[6];    // edge ids of local pairs (0,1),(0,2),(0,3),(1,2),(1,3),(2,3)
  int64_t f[4];    // face ids of faces opposite local vertex 0..3
  int64_t gT;      // global macro index
};

__host__ __device__ inline int local_edge(int a, int b) {
  if (a > b) { int t = a; a = b; b = t; }
  // (0,1)0 (0,2)1 (0,3)2 (1,2)3 (1,3)4 (2,3)5
  return a == 0 ? b - 1 : (a == 1 ? b + 1 : 5);
}

// Canonical global id of lattice node (i,j,k) of a macro (DESIGN.md numbering).
__host__ __device__ inline int64_t node_gid(const GidInfo& g, const MacroTopo& t, int i, int j,
                                            int k) {
  const int N = g.N;
  int w[4] = {N - i - j - k, i, j, k};
  int sup[4];
  int ns = 0;
  for (int v = 0; v < 4; ++v)
    if (w[v] > 0) sup[ns++] = v;
  if (ns == 1) return t.gv[sup[0]];
  if (ns == 2) {
    int p = sup[0], q = sup[1];
    int64_t e = t.e[local_edge(p, q)];
    int m = (t.gv[p] > t.gv[q]) ? w[p] : w[q];  // weight of the larger-id endpoint
    return g.base_e + e * (N - 1) + (m - 1);
  }
  if (ns == 3) {
    int lf = 0;
    for (int v = 0; v < 4; ++v)
      if (w[v] == 0) lf = v;
    // sort the 3 support vertices by global id
    int a = sup[0], b = sup[1], c = sup[2];
    if (t.gv[a] > t.gv[b]) { int x = a; a = b; b = x; }
    if (t.gv[b] > t.gv[c]) { int x = b; b = c; c = x; }
    if (t.gv[a] > t.gv[b]) { int x = a; a = b; b = x; }
    int64_t s = w[b], tt = w[c];
    int64_t idx = (tt - 1) * (N - 1) - (tt - 1) * tt / 2 + (s - 1);
    return g.base_f + t.f[lf] * g.nfi + idx;
  }
  return g.base_v + t.gT * g.nvi + vol_index(N, i, j, k);
}

// Band of diagonals handled by one CTA of the column-march kernels (march.cuh).
struct Band {
  int d0, d1;       // diagonals [d0, d1) computed by this band
  int c_lo;         // first column index loaded (diagonal d0-1, j=0)
  int ncols;        // columns loaded per plane (diagonals d0-1 .. d1)
  int kmax;         // last plane computed (N-1-d0)
  int ncolumns;     // interior columns (threads used)
};
constexpr int kMarchThreads = 256;
// opt-in dynamic shared memory limit of the march kernels (227 KB per block on sm_100, minus static)
constexpr int kMaxDynSmem = 227 * 1024 - 1024;
constexpr int kRing = 16;  // plane slots (power of 2); >= 11 planes in flight ahead of use

// Structured lower-primitive rows of one non-Dirichlet macro face (faces.cu).
// Row entries: 0 centre; 1..6 in-face (ds,dt) = (1,0)(-1,0)(0,1)(0,-1)(-1,1)(1,-1);
// 7..10 into macro A; 11..14 into macro B (zero if the face has no B).
struct FaceLP {
  int TA, TB;           // local macros (TA < TB; TB = -1 for a boundary face)
  int8_t lA[3], lB[3];  // local vertex of the face's sorted vertices a<b<c in A / B
  int8_t off[14][3];    // ijk offsets: [0..5] in-face (A frame), [6..9] into A, [10..13] into B (B frame)
  int8_t mapA[15], mapB[15];  // partial-stencil direction -> entry (-1: not a neighbour)
  int8_t z;             // in-face row mode: node order q -> (s,t) from table fst[z] (setup.cu)
  int8_t bfirst;        // 1: macro B has the lower global id (its entries are summed first)
  int64_t fid;          // canonical face id
};

// ---------------------------------------------------------------------------
// Per-level state
// ---------------------------------------------------------------------------
enum { kStepVertex = 0, kStepEdge0, kStepEdge1, kStepFace0, kStepFace1, kStepFace2, kNumLpSteps };

struct Level {
  int L = 0, N = 0;
  int64_t P = 0;        // lattice nodes per macro
  int64_t S = 0;        // stride (doubles) per macro
  int64_t n_local = 0;  // doubles per local vector
  int64_t n_owned = 0;  // owned unknowns
  GidInfo gi{};
  // lower-primitive rows (owned unknowns on vertices/edges/faces)
  int64_t n_rows = 0, nnz = 0, n_copies = 0, n_dir = 0;
  int64_t step_start[kNumLpSteps + 1] = {0};
  uint64_t* d_row_ptr = nullptr;   // [n_rows+1]
  uint32_t* d_col = nullptr;       // [nnz] local slot; entry 0 of a row = centre
  double* d_val = nullptr;         // [nnz] exact FEM, blended
  double* d_val_cons = nullptr;    // [nnz] exact FEM, affine
  uint64_t* d_copy_ptr = nullptr;  // [n_rows+1]
  uint32_t* d_copy = nullptr;      // [n_copies] slots, ascending (first = owner)
  int64_t* d_row_gid = nullptr;    // [n_rows]
  uint32_t* d_dir_slot = nullptr;  // [n_dir] Dirichlet slots (all copies)
  int64_t* d_dir_gid = nullptr;    // [n_dir]
  double* d_tmp = nullptr;         // [n_rows] GS scratch
  // volume coefficients
  int q = -1;
  int mq = 0;
  double* d_coef = nullptr;        // [nt_local][15][mq] index units, exponent order kExp
  double* d_cons = nullptr;        // [nt_local][15] affine constant stencil
  double* d_coef10 = nullptr;      // [nt_local][15][10] q<=2 coefficients zero-padded to q=2
  double* d_cC = nullptr;          // [nt_local][15] k^2 coefficients (coef10[..][9]), march kernels
  double* d_ew_lo = nullptr;       // [n_local] element-wise FEM: sums for the next band's first diagonal
  double* d_ew_hi = nullptr;       // [n_local] ... for the previous band's last diagonal
  bool fitted = false;
  bool centre_bad = false;         // a surrogate centre weight <= 0 at some interior node (GS refuses: HHG_ERR_NUMERIC)
  bool fcentre_bad = false;        // ... of a fitted face surrogate (SURROGATE_FACES GS refuses)
  // column-march bands (<= kMarchThreads columns)
  std::vector<Band> bands;
  Band* d_bands = nullptr;
  int slot_len = 0;
  std::vector<Band> bands_w;       // <= 2 kMarchThreads columns (single-pass GS, gsfront.cuh)
  Band* d_bands_w = nullptr;
  int slot_len_w = 0;
  // bands of the producer-warp GS (gsprod.cuh): <= 224 / 480 columns (7 / 15 compute warps)
  std::vector<Band> bands_p[2];
  Band* d_bands_p[2] = {nullptr, nullptr};
  int slot_len_p[2] = {0, 0};
  std::vector<Band> bands_fem;  // element-wise FEM: <= kMarchThreads anchor columns per band
  Band* d_bands_fem = nullptr;
  // structured face rows (faces.cu): row r = face * nfi + q, q in colour-major order
  int64_t n_flp = 0, n_frows = 0;
  int fcol[4] = {0, 0, 0, 0};      // colour offsets of q ((s+2t) mod 3 = 0,1,2)
  int fne_len[3] = {0, 0, 0};      // near-edge rows per face and colour (same for every mode z)
  int* d_fne[3] = {nullptr, nullptr, nullptr};  // [colour][3 modes z][fne_len] q of near-edge rows
  FaceLP* d_flp = nullptr;
  uint32_t* d_fst = nullptr;       // [3][nfi] s | t << 16 for q, per row mode z
  int* d_fcidx = nullptr;          // [3][nfi] canonical in-face index of q
  double* d_fval = nullptr;        // [15][n_frows] exact FEM, blended
  double* d_fcoef = nullptr;       // [n_flp][15][(q+1)(q+2)/2] surrogate face polynomials
  double* d_fval_cons = nullptr;   // [15][n_frows] exact FEM, affine
  double* d_ftmp = nullptr;        // [n_frows] GS scratch
  int* d_po = nullptr;             // [N+2] plane offsets
  // replicated coarse solve (coarse.cu): CSR of the exact FEM operator over all
  // canonical unknowns of the level, identical on every rank
  bool cg_built = false;
  int cg_grid = 0;
  int64_t cg_nnz = 0;
  int* d_cg_rp = nullptr;          // [n_total+1]
  int* d_cg_col = nullptr;         // [cg_nnz] canonical ids
  double* d_cg_val = nullptr;      // [cg_nnz]
  double* d_cg_vec = nullptr;      // [5][n_total] b, x, r, p, Ap
  double* d_cg_part = nullptr;     // [3][cg_grid] block partial sums
  double* d_cg_red = nullptr;      // [nranks][n_total] host-transport allreduce scratch
  std::vector<FaceLP> h_flp;       // host copies (exchange plan)
  std::vector<uint32_t> h_fst;
  std::vector<int> h_fcidx;
  // exchange plan (dist.cu): values this rank receives from / sends to each peer
  std::vector<int64_t> send_cnt, recv_cnt;   // [nranks] doubles per peer
  std::vector<uint32_t> h_send_slot, h_recv_slot;
  std::vector<int64_t> h_send_gid, h_recv_gid;  // canonical ids (plan checks)
  uint32_t* d_send_slot = nullptr;
  uint32_t* d_recv_slot = nullptr;
  double* d_sendbuf = nullptr;
  double* d_recvbuf = nullptr;
  int64_t n_send = 0, n_recv = 0;
  // reverse direction (copies -> owner, summed): the send entries grouped by
  // owner slot, entries of a slot in (peer rank, request) order
  int64_t n_rsum = 0;
  uint32_t* d_rsum_ptr = nullptr;   // [n_rsum + 1]
  uint32_t* d_rsum_slot = nullptr;  // [n_rsum]
  uint32_t* d_rsum_idx = nullptr;   // [n_send]
  // persistent GS work queue (k_gs_items)
  int* d_gs_flags = nullptr;   // [nt_local][n_bands][4] sweep epoch of completed colour passes
  int* d_gs_counter = nullptr; // [1]
  // single-pass wavefront GS (gsfront.cuh), allocated on first use
  uint64_t* d_gs_ex = nullptr;    // [n_local][2] LL halo words (value halves + epoch tag)
  uint32_t* d_gs_prog = nullptr;  // [nt_local][n_bands] progress words
  uint32_t* d_gs_epoch = nullptr; // [1] sweep epoch (incremented on the device per sweep)
  int gs_epoch = 0;
};

struct Ctx {
  std::string err;
  bool poisoned = false;
  cudaStream_t stream = nullptr;
  cudaStream_t cap_stream = nullptr;  // graph capture (the ctx stream may be the legacy default stream)
  cudaStream_t comm_stream = nullptr; // ghost exchange overlapped with interior macros (dist.cu)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int64_t nt_bnd = 0;                 // local macros [0, nt_bnd) touch another rank's macros (boundary)
  // cached V-cycle graph (hhg_vcycle): replayed while the call signature matches
  cudaGraphExec_t vc_graph = nullptr;
  int64_t vc_graph_launches = 0;
  std::vector<int64_t> vc_graph_key;
  int rank = 0, nranks = 1;
  int L_max = 0;
  // nt_local macros owned by this rank are blocks [0, nt_local); ghost macros
  // (owned elsewhere, sharing a vertex with a local macro) follow up to nt_blocks
  int64_t nv = 0, nt = 0, nt_local = 0, nt_blocks = 0;
  std::vector<int32_t> owner;         // [nt] rank of every global macro
  std::vector<int64_t> g2b;           // [nt] global macro -> block (-1: absent)
  // transport (dist.cu)
  int transport = 0;                  // 0 none (1 rank), 1 NCCL, 2 host callback
  void* nccl_comm = nullptr;          // ncclComm_t
  void* host_fn = nullptr;            // hhg_host_exchange_fn
  void* host_user = nullptr;
  bool host_only = false;             // plan-only context (no CUDA), tests
  double* h_stage = nullptr;          // pinned staging for the host transport
  int64_t h_stage_n = 0;
  int64_t n_e = 0, n_f = 0;
  bool blended = true;
  std::vector<double> vertices, radius;
  std::vector<int64_t> tets;
  std::vector<uint8_t> dirichlet;
  std::vector<int64_t> local_macros;  // global ids of local macros
  std::vector<MacroTopo> topo;        // [nt_blocks] (local macros, then ghosts)
  MacroTopo* d_topo = nullptr;
  double* d_geo = nullptr;            // [nt_local][4][4]: x,y,z,r per local vertex
  std::vector<Level> levels;          // index L
  int64_t launches = 0;
  // per-context launch caches (a context is bound to one device)
  std::set<const void*> smem_attr_done;                    // kernels with the >48 KB smem attribute set
  std::map<std::pair<const void*, size_t>, int> grid_cache;  // co-resident grid per (kernel, smem)
  // host-vector staging
  double* d_stage[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t stage_n = 0;
  double* d_red = nullptr;            // reduction scratch
  double* h_red = nullptr;            // pinned
  int64_t red_n = 0;
  // multigrid (vcycle.cu)
  std::vector<uint16_t> own;          // [nt_local] owned faces (bits 0-3), edges (4-9), vertices (10-13)
  uint16_t* d_own = nullptr;
  std::vector<double*> vc_u, vc_f, vc_r;  // per-level work vectors
  double* d_cg = nullptr;             // CG work: r p Ap at the coarse level (3 vectors)
  int64_t cg_n = 0;
  double* d_scal = nullptr;           // device scalars
  int* d_flag = nullptr;              // device flag word (fit-time centre-weight check)
  unsigned long long* d_gsprof = nullptr;  // wavefront GS cycle counters (hhg_gs_prof)
  // profiling (hhg_profile)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_rec[4];
};

// RAII event bracket around kernel launches of class `kind` (no-op unless profiling)
struct ProfScope {
  Ctx* c;
  int kind;
  cudaEvent_t a = nullptr, b = nullptr;
  static cudaEvent_t get(Ctx* c) {
    if (!c->ev_pool.empty()) {
      cudaEvent_t e = c->ev_pool.back();
      c->ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  ProfScope(Ctx* c_, int k) : c(c_), kind(k) {
    if (!c->prof) return;
    a = get(c);
    b = get(c);
    cudaEventRecord(a, c->stream);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, c->stream);
    c->ev_rec[kind].push_back({a, b});
  }
};

// error helpers ------------------------------------------------------------
hhg_status set_err(Ctx* c, hhg_status s, const std::string& msg);
hhg_status check_cuda(Ctx* c, cudaError_t e, const char* what);
#define HHG_CK(c, call)                                        \
  do {                                                         \
    cudaError_t e__ = (call);                                  \
    if (e__ != cudaSuccess) return hhg::check_cuda(c, e__, #call); \
  } while (0)
#define HHG_LAUNCHED(c)                                                    \
  do {                                                                     \
    (c)->launches++;                                                       \
    cudaError_t e__ = cudaGetLastError();                                  \
    if (e__ != cudaSuccess) return hhg::check_cuda(c, e__, "kernel launch"); \
  } while (0)

// exponent table for the surrogate basis (index units): for q, m_q entries
int n_coeffs(int q);
void exponents(int q, std::vector<int>& l, std::vector<int>& m, std::vector<int>& n);

// Distributed-memory support (dist.cu)
hhg_status dist_init_transport(Ctx* c, const void* nccl_unique_id);
void dist_destroy(Ctx* c);
hhg_status ctx_sync(Ctx* c);
hhg_status dist_exchange_bytes(Ctx* c, const std::vector<int64_t>& send_bytes, const void* send,
                               const std::vector<int64_t>& recv_bytes, void* recv, bool device,
                               cudaStream_t stream);
hhg_status dist_build_plan(Ctx* c, Level& lv, const std::vector<uint32_t>& recv_slot,
                           const std::vector<int64_t>& recv_gid, const std::vector<int32_t>& recv_rank,
                           const std::vector<std::pair<int64_t, uint32_t>>& serve);
hhg_status dist_sync(Ctx* c, Level& lv, double* v, cudaStream_t stream = nullptr);
hhg_status dist_sync_overlapped(Ctx* c, Level& lv, double* v, const std::function<hhg_status()>& interior);
hhg_status dist_sum_to_owner(Ctx* c, Level& lv, double* v);
hhg_status dist_allreduce_sum(Ctx* c, double* d_scalar);

// Structured face rows (faces.cu)
hhg_status build_face_values(Ctx* c, Level& lv);
hhg_status face_apply(Ctx* c, Level& lv, int op, int mode, const double* u, const double* f, double* out);
hhg_status face_gs_step(Ctx* c, Level& lv, int op, int colour, double* u, const double* f);
hhg_status face_gather(Ctx* c, Level& lv, const double* local, double* glob, int dir);
hhg_status face_sync(Ctx* c, Level& lv, double* u);
hhg_status face_dot(Ctx* c, Level& lv, const double* a, const double* b, double* part, int nblocks);
hhg_status face_sum_copies(Ctx* c, Level& lv, double* v);
hhg_status face_centre_check(Ctx* c, Level& lv, int* d_flag);

// Operator pieces shared by ops.cu and vcycle.cu
hhg_status apply_dev(Ctx* c, Level& lv, int op, int mode, const double* u, const double* f, double* y);
hhg_status gs_sweep_dev(Ctx* c, Level& lv, int op, double* u, const double* f, bool lex = false);
hhg_status norm2_of(Ctx* c, Level& lv, const double* r, double* out);
hhg_status dot_dev(Ctx* c, Level& lv, const double* a, const double* b, double* d_out);
hhg_status zero_dir_slots(Ctx* c, Level& lv, double* out);
hhg_status check_centre_ok(Ctx* c, const Level& lv, int op);
hhg_status lp_sum_copies(Ctx* c, Level& lv, double* v);
hhg_status lp_sync_own_copies(Ctx* c, Level& lv, double* v);
// canonical global vector <-> local layout (ops.cu): owned entries into dglob
// (0 elsewhere; summed over ranks = the global vector) / every local copy from dglob
hhg_status gather_owned_dev(Ctx* c, Level& lv, const double* local, double* dglob);
hhg_status scatter_global_dev(Ctx* c, Level& lv, const double* dglob, double* local);
// replicated coarse solve (coarse.cu)
constexpr int64_t kCoarseMaxUnknowns = 1ll << 22;
bool coarse_replicable(const Level& lv);
hhg_status coarse_build(Ctx* c, Level& lv);
hhg_status coarse_solve(Ctx* c, Level& lv, int iters, double* x, const double* b);
hhg_status dist_allreduce_vec(Ctx* c, double* d_vec, int64_t n);

// Device geometry helpers (fem.cu)
hhg_status launch_fem_partial(Ctx* c, int L, const uint32_t* d_slots, int64_t n, bool blended,
                              double* d_out15);
hhg_status build_lp_values(Ctx* c, Level& lv, const std::vector<uint8_t>& cmap, const std::vector<uint32_t>& cord);

}  // namespace hhg
