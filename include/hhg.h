/* hhg.h -- C ABI of the B200 two-scale surrogate-stencil library (libhhg.so).
 *
 * Implements the hot path of Bauer, Mohr, Ruede, Weismueller, Wittmann,
 * Wohlmuth, "A two-scale approach for efficient on-the-fly operator assembly in
 * massively parallel high performance multigrid codes" (arXiv:1608.06473):
 * matrix-free application of the 15-point P1 Laplace stencil on uniformly
 * refined macro tetrahedra of a radially blended spherical shell, with every
 * volume-primitive stencil weight evaluated per fine node from a degree-q
 * surrogate polynomial of its macro element, used for the
 * operator apply, the residual and a multicolour Gauss-Seidel sweep
 * (PAPER.md:1306-1315), next to an element-wise on-the-fly FEM apply and a
 * constant-stencil (affine) apply as comparison paths.
 *
 * Conventions:
 *  - Level L: N = 2^L intervals per macro edge (the paper's l = L - 2,
 *    PAPER.md:225).  2 <= L <= 8.
 *  - Macro tet t has local vertices tets[t][0..3] = (x0,x1,x2,x3); lattice node
 *    (i,j,k), i,j,k >= 0, i+j+k <= N, sits at x0 + (i/N)(x1-x0) + (j/N)(x2-x0)
 *    + (k/N)(x3-x0) before blending (Psi_T).
 *  - Blending Phi_T(x) = x * (sum_v lambda_v r_v) / |x| (PAPER.md:249-262,
 *    reading R4); vertex_radius == NULL means Phi = Id (polyhedral domain).
 *  - Stencil direction order (test export hhg_eval_stencils):
 *      0 bc (0,0,-1)   1 be (1,0,-1)   2 bn (0,1,-1)   3 bnw (-1,1,-1)
 *      4 ms (0,-1,0)   5 mse (1,-1,0)  6 mw (-1,0,0)   7 mc (0,0,0)
 *      8 me (1,0,0)    9 mnw (-1,1,0) 10 mn (0,1,0)   11 tse (1,-1,1)
 *     12 ts (0,-1,1)  13 tw (-1,0,1)  14 tc (0,0,1)      opposite(w) = 14 - w.
 *
 * LOCAL VECTOR LAYOUT (what every vector argument points to): one block of
 * `stride` doubles per local macro, in local macro order.  Inside a block the
 * full lattice of the macro (boundary included) is stored plane by plane
 * (k = 0..N); inside plane k, by diagonal d = i + j (0..N-k), inside a
 * diagonal by j (0..d):
 *      pos(i,j,k) = planeoff(k) + d(d+1)/2 + j,
 *      planeoff(k) = sum_{k'<k} (N-k'+1)(N-k'+2)/2.
 *  Lower-primitive nodes (on macro faces/edges/vertices) are stored once per
 *  macro that contains them ("copies").  Padding slots at the end of a block
 *  are never read.
 *  Vector CONTRACT for inputs: all copies of a node hold the same value and
 *  Dirichlet slots hold 0.  Every hhg_* output satisfies it, hhg_scatter_global
 *  produces it, any linear combination of such vectors keeps it, and
 *  hhg_sync_copies restores it for arbitrary data (owner copy = copy in the
 *  lowest-numbered macro wins; Dirichlet slots zeroed).
 *
 * Vector arguments may be DEVICE pointers (the fast path: nothing is copied)
 * or HOST pointers (pageable or pinned; detected with cudaPointerGetAttributes):
 * host vectors are staged through ctx-owned device buffers with
 * cudaMemcpyAsync on the ctx stream and the call synchronises before return.
 * Inputs and outputs must not alias unless stated.
 *
 * All calls enqueue on the ctx stream (cuda_stream given at setup; NULL =
 * legacy default stream) and are asynchronous unless they return host scalars
 * (norm2, residual history) or take host vectors.  One ctx per host thread;
 * not re-entrant.  Nothing throws across the ABI; every call returns an
 * hhg_status.  CUDA failures poison the ctx (sticky HHG_ERR_CUDA); the text
 * is in hhg_last_error(ctx).
 */
#ifndef HHG_H_
#define HHG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hhg_ctx_s* hhg_ctx;

typedef enum {
  HHG_OK = 0,
  HHG_ERR_INVALID = 1,  /* bad argument: NULL pointer, L out of range, q > 4,
                           surrogate requested on L < 3 without fit, ... */
  HHG_ERR_MESH = 2,     /* degenerate tet, non-conforming / over-shared face,
                           |x_v| != r_v beyond 1e-12 relative */
  HHG_ERR_FIT = 3,      /* rank-deficient sampling matrix */
  HHG_ERR_NUMERIC = 4,  /* non-positive surrogate centre weight (the GS update
                           divides by it): raised by
                           hhg_fit_surrogates / hhg_fit_from_samples (the fit is
                           still installed: apply and residual work) and by
                           every later hhg_gs_sweep / hhg_vcycle on that level */
  HHG_ERR_DIVERGED = 5, /* V-cycle residual grew 3 cycles in a row */
  HHG_ERR_CUDA = 6,
  HHG_ERR_NCCL = 7,
  HHG_ERR_OOM = 8,
  HHG_ERR_STATE = 9     /* call order violated (e.g. apply before fit) */
} hhg_status;

typedef enum {
  HHG_OP_SURROGATE = 0,       /* L~: volume rows from the surrogate polynomials
                                 (PAPER.md:618-636), lower primitives exact FEM */
  HHG_OP_FEM_ELEMENTWISE = 1, /* exact L: element-wise on-the-fly assembly over
                                 all fine tets, blended geometry (PAPER.md:
                                 1102-1122); comparison path */
  HHG_OP_CONST_AFFINE = 2,    /* CONS: FEM of the unblended (affine) mesh, one
                                 constant stencil per macro for volume rows
                                 (PAPER.md:380-384, 886-889); comparison path */
  HHG_OP_SURROGATE_FACES = 3  /* L~ with the face-node rows from surrogates too
                                 (PAPER.md:341-345 remark): per
                                 face and neighbour entry a degree-q polynomial
                                 in the face coordinates (s, t), least squares
                                 on the face nodes of the embedded 2^(m+2)
                                 lattice; edge / vertex rows exact.  Fitted by
                                 hhg_fit_surrogates; exact at L = 2 */
} hhg_op;

typedef enum { HHG_FIT_LSQP = 0, HHG_FIT_IPOLY = 1 } hhg_fit_method;

/* Build the macro mesh, topology, per-level layouts and lower-primitive FEM
 * rows.
 *  vertices      [nv][3] host, copied.
 *  vertex_radius [nv] host or NULL (Phi = Id).
 *  tets          [nt][4] host, global vertex ids; order defines lattice axes.
 *  dirichlet_face[nt][4] host, face f = face opposite local vertex f; nonzero
 *                = homogeneous Dirichlet (u = 0).  Untagged
 *                boundary faces get natural (Neumann) boundary rows.
 *  L_max         finest level, 2..8; all levels 2..L_max are set up.
 *  macro_owner   [nt] rank of each macro, or NULL (all on rank 0).
 *  rank, nranks  this process and the job size (1 = single GPU).
 *  nccl_unique_id 128-byte ncclUniqueId from rank 0 (NULL iff nranks == 1).
 *  cuda_stream   cudaStream_t to enqueue on (NULL = default stream).
 *  out           receives the ctx (NULL on failure).
 * Errors: HHG_ERR_INVALID, HHG_ERR_MESH, HHG_ERR_OOM, HHG_ERR_CUDA, HHG_ERR_NCCL. */
hhg_status hhg_setup_macro_mesh(const double* vertices, const double* vertex_radius, int64_t nv,
                                const int64_t* tets, int64_t nt, const uint8_t* dirichlet_face,
                                int L_max, const int32_t* macro_owner, int rank, int nranks,
                                const void* nccl_unique_id, void* cuda_stream, hhg_ctx* out);

/* Fit the 15 surrogate polynomials of every local macro on every level
 * 3..L_max: exact FEM stencils at the sampling
 * set S_l = M_m(l,j), m(l,j) = min{l, max{1,j}} (LSQP) or the 10 IPOLY points
 * (q = 2 only), then a = A^+ b with A^+ from one Householder QR per level.
 * Level 2 (l = 0) uses its exact stencil.  q in 0..4 (full rank, PAPER.md:
 * 530-534).  After the fit every interior node's centre weight (and every
 * face node's, for the face surrogates) is evaluated once; a non-positive one
 * returns HHG_ERR_NUMERIC with the fit installed.  Errors: HHG_ERR_INVALID,
 * HHG_ERR_FIT, HHG_ERR_NUMERIC, HHG_ERR_CUDA. */
hhg_status hhg_fit_surrogates(hhg_ctx ctx, int q, hhg_fit_method method, int sampling_j);

/* TEST EXPORTS of the fit.
 * hhg_sample_nodes: the sampling set of level L (3 <= L <= L_max) that
 *   hhg_fit_surrogates uses for (method, sampling_j) -- LSQP: the interior
 *   nodes of the 2^(m+2) lattice, m = min(L-2, max(1, j)), at level-L indices
 *   x 2^(L-2-m); IPOLY: the 10 points of PAPER.md:490-499 --
 *   as ijk[n][3] (host, caller-owned; NULL to query n only) in fit order.
 * hhg_fit_from_samples: fit level L from the caller's samples instead of the
 *   exact FEM stencils: samples[nt_local][n][15] (host or device, fp64; sample
 *   order of hhg_sample_nodes, direction order above), a_w = A^+ b_w as in
 *   hhg_fit_surrogates.  Replaces level L's volume coefficients only (its face
 *   surrogates are dropped: HHG_OP_SURROGATE_FACES is then refused on L).
 *   Errors: HHG_ERR_INVALID, HHG_ERR_FIT, HHG_ERR_NUMERIC (see above). */
hhg_status hhg_sample_nodes(hhg_ctx ctx, int L, hhg_fit_method method, int sampling_j, int32_t* ijk, int64_t* n);
hhg_status hhg_fit_from_samples(hhg_ctx ctx, int L, int q, hhg_fit_method method, int sampling_j,
                                const double* samples);

/* Sizes at level L: doubles of a local vector (incl. copies and padding),
 * owned unknowns (each unknown counted on exactly one rank), and the length
 * of the canonical global vector (all nodes incl. Dirichlet, DESIGN.md
 * "canonical numbering").  Any output pointer may be NULL. */
hhg_status hhg_vector_layout(hhg_ctx ctx, int L, int64_t* n_local_doubles,
                             int64_t* n_owned_unknowns, int64_t* n_global_nodes);

/* y = A u over the unknowns (A = L~, L or CONS by op; PAPER.md:618-636
 * eq. ts, per-node stencils evaluated on the fly PAPER.md:654-690); y = 0 at
 * Dirichlet slots; all copies of y written.  u and y must not alias
 * (HHG_ERR_INVALID); L~ before hhg_fit_surrogates: HHG_ERR_STATE. */
hhg_status hhg_apply(hhg_ctx ctx, int L, hhg_op op, const double* u, double* y);

/* r = f - A u.  If norm2 != NULL the Euclidean norm of r
 * over the unique unknowns is returned on the host (synchronises). */
hhg_status hhg_residual(hhg_ctx ctx, int L, hhg_op op, const double* u, const double* f,
                        double* r, double* norm2);

/* n_sweeps multicolour Gauss-Seidel sweeps in place on u (eq. iteration-scheme,
 * PAPER.md:1306-1315): class steps vertices -> edge colours 0,1 -> face colours
 * 0,1,2 -> volume colours (i+2j+3k) mod 4 = 0..3; all nodes of a step update
 * simultaneously (R13, R14).  op FEM_ELEMENTWISE is not a smoother
 * (HHG_ERR_INVALID). */
hhg_status hhg_gs_sweep(hhg_ctx ctx, int L, hhg_op op, double* u, const double* f, int n_sweeps);

/* n_sweeps sweeps of the paper's own hybrid smoother with a LEXICOGRAPHIC
 * volume ordering: the lower-primitive class steps as in
 * hhg_gs_sweep (R13), then the volume nodes of every macro visited west to
 * east (i), south to north (j), bottom to top (k), each from the newest values
 * -- executed exactly as hyperplanes i + 2j + 3k in increasing order (no two
 * neighbours share one; predecessors lie on lower ones).  Same arguments and
 * errors as hhg_gs_sweep. */
hhg_status hhg_gs_sweep_lex(hhg_ctx ctx, int L, hhg_op op, double* u, const double* f, int n_sweeps);

/* n_cycles V(nu1,nu2) cycles from level L down to L_coarse:
 * GS smoothing with `op` on every level, residual, restriction R = P^T, coarse
 * grid solved by coarse_cg_iters CG iterations from zero on the exact FEM
 * operator, prolongation P (index-space linear interpolation, R18).
 * res_hist[n_cycles+1] (host, may be NULL) receives ||f - A u||_2 before the
 * first and after every cycle.  Returns HHG_ERR_DIVERGED if the residual grew
 * three cycles in a row (history still written).  Multi-rank: a collective
 * like hhg_apply; the restriction sums the partials of copies on other ranks
 * into the owner (reverse exchange) before the owners' totals are re-synced. */
hhg_status hhg_vcycle(hhg_ctx ctx, int L, int nu1, int nu2, int L_coarse, int coarse_cg_iters,
                      hhg_op op, double* u, const double* f, int n_cycles, double* res_hist);

/* Double discretisation: as hhg_vcycle, but the residuals
 * on every level -- and res_hist -- use residual_op (e.g. FEM_ELEMENTWISE, the
 * exact operator) while smoother_op (SURROGATE or CONST_AFFINE) smooths.  The
 * two operators pull towards different algebraic solutions,
 * so the history is not expected to decrease to zero and the growth check of
 * hhg_vcycle (HHG_ERR_DIVERGED) is off.  residual_op == smoother_op is
 * hhg_vcycle.  HHG_ERR_INVALID for an unknown residual_op. */
hhg_status hhg_vcycle_dd(hhg_ctx ctx, int L, int nu1, int nu2, int L_coarse, int coarse_cg_iters,
                         hhg_op smoother_op, hhg_op residual_op, double* u, const double* f, int n_cycles,
                         double* res_hist);

/* The general form of hhg_vcycle / hhg_vcycle_dd:
 * lexicographic != 0 smooths with hhg_gs_sweep_lex's ordering on every level
 * instead of the 4 colours (the paper's smoother; compare
 * convergence per cycle).  Arguments and errors as hhg_vcycle_dd. */
hhg_status hhg_vcycle_ex(hhg_ctx ctx, int L, int nu1, int nu2, int L_coarse, int coarse_cg_iters,
                         hhg_op smoother_op, hhg_op residual_op, int lexicographic, double* u, const double* f,
                         int n_cycles, double* res_hist);

/* Canonical global vector (length n_global_nodes, DESIGN.md numbering:
 * vertices, edges, faces, volumes) <-> local layout.  gather writes every
 * node (0 at Dirichlet); scatter writes every copy and zeroes Dirichlet slots.
 * Multi-rank: gather writes the entries this rank owns and 0 elsewhere (the sum
 * over ranks is the global vector); scatter takes the full global vector on
 * every rank. */
hhg_status hhg_gather_global(hhg_ctx ctx, int L, const double* local, double* global_vec);
hhg_status hhg_scatter_global(hhg_ctx ctx, int L, const double* global_vec, double* local);

/* Make a local vector satisfy the vector contract in place (owner copy wins,
 * Dirichlet slots zeroed). */
hhg_status hhg_sync_copies(hhg_ctx ctx, int L, double* local);

/* Test export: the 15 weights (direction order above) used for every interior
 * node of local macro `macro` at level L by `op`, written to out[n_int][15]
 * with nodes in (k, j, i) lexicographic order; for SURROGATE these are the
 * surrogate values P s_w(i,j,k), for FEM_ELEMENTWISE / CONST_AFFINE the exact
 * FEM stencils of the blended / affine geometry. */
hhg_status hhg_eval_stencils(hhg_ctx ctx, int L, hhg_op op, int64_t macro, double* out);

/* Writes a fresh NCCL unique id (128 bytes, caller-owned buffer) created by
 * the NCCL library this library is bound to, for rank 0 to broadcast to every
 * rank before hhg_setup_macro_mesh (so id creation and communicator setup use
 * the same NCCL build).  HHG_ERR_NCCL on failure. */
hhg_status hhg_nccl_unique_id(void* out128);

/* Multi-rank transport for contexts set up with nranks > 1 and
 * nccl_unique_id == NULL (tests; production uses NCCL).  fn moves host buffers
 * between all ranks: for every peer p, send_bytes[p] bytes (concatenated in
 * rank order in send_buf) go to p, recv_bytes[p] bytes from p land in recv_buf;
 * it returns 0 on success and must be called collectively.  Process-wide;
 * applies to the following hhg_setup_macro_mesh calls.  host_only != 0 makes
 * those setups build the partition and exchange plan on the host only (no
 * CUDA calls; compute entry points then return HHG_ERR_STATE). */
typedef int (*hhg_host_exchange_fn)(void* user, int nranks, const int64_t* send_bytes, const void* send_buf,
                                    const int64_t* recv_bytes, void* recv_buf);
hhg_status hhg_set_host_transport(hhg_host_exchange_fn fn, void* user, int host_only);

/* Partition / exchange-plan diagnostics at level L: info[5] = {owned unknowns,
 * values sent per sync, values received per sync, local macros, local + ghost
 * macro blocks}.  hhg_plan_check runs the plan once on canonical node ids
 * through the transport and returns the number of received ids that differ
 * from the expected ones (0 = consistent).  Collective. */
hhg_status hhg_plan_info(hhg_ctx ctx, int L, int64_t* info);
hhg_status hhg_plan_check(hhg_ctx ctx, int L, int64_t* mismatches);

/* Count of this library's kernel launches since setup (for the bench). */
int64_t hhg_kernel_launches(hhg_ctx ctx);

/* Per-kernel device timing for the bench: while enabled, every launch of a
 * kernel class is bracketed by CUDA events on the ctx stream.  kind: 0 =
 * volume apply/residual kernels, 1 = volume GS kernels, 2 = lower-primitive
 * row kernels, 3 = everything else.  hhg_profile_read synchronises, returns
 * the summed device time (ms) and launch count of `kind`, and clears it. */
hhg_status hhg_profile(hhg_ctx ctx, int enable);
hhg_status hhg_profile_read(hhg_ctx ctx, int kind, double* total_ms, int64_t* launches);

/* Development counters of the single-pass GS kernel: enable != 0 allocates
 * and zeroes 16 counters that later sweeps accumulate into; out16 (host,
 * may be NULL) receives them (synchronising) before they are zeroed again:
 * [0..5] cycles of the first thread of every CTA waiting for planes, in the
 * node update, waiting for halo words, checking neighbour progress, at the
 * step barrier and after it; [6] wavefront steps; [7] items; [8] failed halo
 * polls of all threads.  enable == 0 frees them. */
hhg_status hhg_gs_prof(hhg_ctx ctx, int enable, unsigned long long* out16);

/* Text of the last error of ctx (owned by ctx, valid until the next call). */
const char* hhg_last_error(hhg_ctx ctx);
/* Frees everything ctx owns (device buffers, NCCL communicator, streams,
 * cached graphs); NULL is a no-op. */
void hhg_destroy(hhg_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* HHG_H_ */
