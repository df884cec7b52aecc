// Structured lower-primitive rows of macro faces.
//
// Face nodes are the bulk of the lower-primitive unknowns (PAPER.md:300-302,
// 321-327).  Their rows are the exact FEM rows (assembled from the local
// stiffness matrices of the 24 adjacent fine tets),
// computed once at setup and stored as 15 doubles per row (structure-of-arrays,
// coalesced).  Columns are NOT stored: every face node has the same neighbour
// pattern -- centre, 6 in-face, 4 into each adjacent macro -- so the slots are
// recomputed from (face, s, t) and the face's orientation in its two macros.
#include "faces.cuh"

namespace hhg {

__global__ void k_face_values(const double* __restrict__ geo, int N, int64_t nfi, int64_t n_frows,
                              const FaceLP* __restrict__ flp, const uint32_t* __restrict__ fst, bool blended,
                              double* __restrict__ val) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_frows) return;
  const int64_t f = r / nfi;
  const FaceLP F = flp[f];
  const uint32_t st = fst[F.z * nfi + (r - f * nfi)];
  const int s = st & 0xffff, t = st >> 16;
  double acc[15];
  for (int e = 0; e < 15; ++e) acc[e] = 0.0;
  for (int side = 0; side < 2; ++side) {
    const int T = side == 0 ? F.TA : F.TB;
    if (T < 0) continue;
    const FaceNode n = face_node(side == 0 ? F.lA : F.lB, N, s, t);
    double part[15];
    fem_partial(geo + (int64_t)T * 16, N, n.i, n.j, n.k, blended, part);
    const int8_t* map = side == 0 ? F.mapA : F.mapB;
    for (int w = 0; w < 15; ++w)
      if (map[w] >= 0) acc[map[w]] += part[w];
  }
  for (int e = 0; e < 15; ++e) val[e * n_frows + r] = acc[e];
}

hhg_status build_face_values(Ctx* c, Level& lv) {
  if (lv.n_frows == 0) return HHG_OK;
  const unsigned grid = (unsigned)((lv.n_frows + 127) / 128);
  k_face_values<<<grid, 128, 0, c->stream>>>(c->d_geo, lv.N, lv.gi.nfi, lv.n_frows, lv.d_flp, lv.d_fst, true,
                                             lv.d_fval);
  HHG_LAUNCHED(c);
  k_face_values<<<grid, 128, 0, c->stream>>>(c->d_geo, lv.N, lv.gi.nfi, lv.n_frows, lv.d_flp, lv.d_fst, false,
                                             lv.d_fval_cons);
  HHG_LAUNCHED(c);
  HHG_CK(c, cudaStreamSynchronize(c->stream));
  return HHG_OK;
}

// Surrogate face weight: degree-q polynomial in index units,
// exponents (a, b) by degree, b ascending (fit.cu::fit_faces).
__device__ __forceinline__ double face_poly(const double* __restrict__ cf, int q, int s, int t) {
  const double ds = (double)s, dt = (double)t;
  if (q == 2)  // (0,0) (1,0) (0,1) (2,0) (1,1) (0,2)
    return fma(ds, fma(ds, cf[3], fma(dt, cf[4], cf[1])), fma(dt, fma(dt, cf[5], cf[2]), cf[0]));
  if (q == 1) return fma(ds, cf[1], fma(dt, cf[2], cf[0]));
  if (q == 0) return cf[0];
  double sp[5], tp[5];
  sp[0] = tp[0] = 1.0;
  for (int k = 1; k <= q; ++k) sp[k] = sp[k - 1] * s, tp[k] = tp[k - 1] * t;
  double v = 0.0;
  int x = 0;
  for (int d = 0; d <= q; ++d)
    for (int b = 0; b <= d; ++b) v = fma(cf[x++], sp[d - b] * tp[b], v);
  return v;
}

// flag |= 2 if a fitted face surrogate's centre weight (entry 0) is <= 0 (or
// NaN) at a face node (the face GS class steps divide by it).
__global__ void k_face_check_centre(int64_t nfi, int64_t n_frows, const FaceLP* __restrict__ flp,
                                    const uint32_t* __restrict__ fst, const double* __restrict__ fcoef, int fq,
                                    int* __restrict__ flag) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_frows) return;
  const int64_t fc = r / nfi;
  const uint32_t st = fst[flp[fc].z * nfi + (r - fc * nfi)];
  const int nfc = (fq + 1) * (fq + 2) / 2;
  if (!(face_poly(fcoef + fc * 15 * nfc, fq, st & 0xffff, st >> 16) > 0.0)) atomicOr(flag, 2);
}

hhg_status face_centre_check(Ctx* c, Level& lv, int* d_flag) {
  if (!lv.d_fcoef || lv.n_frows == 0) return HHG_OK;
  k_face_check_centre<<<(unsigned)((lv.n_frows + 127) / 128), 128, 0, c->stream>>>(
      lv.gi.nfi, lv.n_frows, lv.d_flp, lv.d_fst, lv.d_fcoef, lv.q, d_flag);
  HHG_LAUNCHED(c);
  return HHG_OK;
}

// Summation order of a face row: centre, in-face entries 1..6, then the 4
// into-macro entries of the macro with the LOWER global id, then the other 4
// (F.bfirst: macro B's entries 11..14 first).  Canonical, so the row's
// rounding is independent of which macro is local where (bitwise-equal
// results on any number of ranks).  acc = fma(sgn * w_e, un_e, acc) in that order.
template <class W>
__device__ __forceinline__ double face_row_chain(const FaceLP& F, double acc, double sgn, W w,
                                                 const double (&un)[14]) {
#pragma unroll
  for (int e = 0; e < 6; ++e) acc = fma(sgn * w(e + 1), un[e], acc);
  if (F.bfirst) {
#pragma unroll
    for (int e = 10; e < 14; ++e) acc = fma(sgn * w(e + 1), un[e], acc);
#pragma unroll
    for (int e = 6; e < 10; ++e) acc = fma(sgn * w(e + 1), un[e], acc);
  } else {
#pragma unroll
    for (int e = 6; e < 14; ++e) acc = fma(sgn * w(e + 1), un[e], acc);
  }
  return acc;
}

// mode: kModeApply / kModeResid (vol_kernels.cuh values 0 / 1)
__global__ void k_face_apply(int N, int64_t S, int64_t nfi, int64_t n_frows, const FaceLP* __restrict__ flp,
                             const uint32_t* __restrict__ fst, const int* __restrict__ po,
                             const double* __restrict__ val, const double* __restrict__ u,
                             const double* __restrict__ f, double* __restrict__ out, int mode,
                             const double* __restrict__ fcoef, int fq) {
  __shared__ int po_s[260];
  load_po(po_s, po, N);
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_frows) return;
  const int64_t fc = r / nfi;
  const FaceLP& F = flp[fc];
  const uint32_t st = fst[F.z * nfi + (r - fc * nfi)];
  FaceRowSlots o;
  face_row_slots(F, N, S, po_s, st & 0xffff, st >> 16, o);
  const int nfc = (fq + 1) * (fq + 2) / 2;
  auto wgt = [&](int e) -> double {  // stored exact weight, or the face surrogate
    return fcoef ? face_poly(fcoef + (fc * 15 + e) * nfc, fq, st & 0xffff, st >> 16) : val[e * n_frows + r];
  };
  double un[14];
#pragma unroll
  for (int e = 0; e < 14; ++e) un[e] = o.nb[e] >= 0 ? u[o.nb[e]] : 0.0;
  double acc;
  if (fcoef) {  // all neighbour values first (memory-level parallelism), then the weights
    acc = face_row_chain(F, wgt(0) * u[o.cA], 1.0, wgt, un);
  } else {
    // every gather and weight load first (memory-level parallelism: the face
    // rows are latency-bound, ncu r01h: long-scoreboard 74 %), then the chain
    double wv[15];
#pragma unroll
    for (int e = 0; e < 15; ++e) wv[e] = (e == 0 || o.nb[e - 1] >= 0) ? val[e * n_frows + r] : 0.0;
    acc = face_row_chain(F, wv[0] * u[o.cA], 1.0, [&](int e) { return wv[e]; }, un);
  }
  const double res = mode == 1 ? f[o.cA] - acc : acc;
  out[o.cA] = res;
  if (o.cB >= 0) out[o.cB] = res;
}

// A face node whose (s,t) is at least 2 away from the face's edges has no
// neighbour outside its own face and the two adjacent volumes, and nodes of one
// face colour are never neighbours inside a face: such nodes can be updated in
// place within a colour step without changing its simultaneous-update
// semantics (R13).  Nodes next to an edge may neighbour same-colour
// nodes of another face (through the volume), so they go through tmp.
__device__ __forceinline__ bool face_inner(int N, int s, int t) { return s >= 2 && t >= 2 && s + t <= N - 2; }

// GS colour step on face nodes of colour `colour`: inner nodes in place,
// near-edge nodes into tmp (written by k_face_write after the step).
__global__ void k_face_gs(int N, int64_t S, int64_t nfi, int64_t nfc, int q0, const FaceLP* __restrict__ flp,
                          const uint32_t* __restrict__ fst, const int* __restrict__ po, int64_t n_frows,
                          const double* __restrict__ val, double* __restrict__ u,
                          const double* __restrict__ f, double* __restrict__ tmp,
                          const double* __restrict__ fcoef, int fq) {
  __shared__ int po_s[260];
  load_po(po_s, po, N);
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per_face = nfc;
  const int64_t fc = x / per_face;
  if (x >= per_face * (n_frows / nfi)) return;
  const int64_t q = q0 + (x - fc * per_face);
  const int64_t r = fc * nfi + q;
  const FaceLP& F = flp[fc];
  const uint32_t st = fst[F.z * nfi + q];
  FaceRowSlots o;
  face_row_slots(F, N, S, po_s, st & 0xffff, st >> 16, o);
  const int ncf = (fq + 1) * (fq + 2) / 2;
  auto wgt = [&](int e) -> double {  // stored exact weight, or the face surrogate
    return fcoef ? face_poly(fcoef + (fc * 15 + e) * ncf, fq, st & 0xffff, st >> 16) : val[e * n_frows + r];
  };
  double un[14];
#pragma unroll
  for (int e = 0; e < 14; ++e) un[e] = o.nb[e] >= 0 ? u[o.nb[e]] : 0.0;
  double v;
  if (fcoef) {  // all neighbour values first (memory-level parallelism), then the weights
    v = face_row_chain(F, f[o.cA], -1.0, wgt, un) / wgt(0);
  } else {
    double wv[15];
#pragma unroll
    for (int e = 0; e < 15; ++e) wv[e] = (e == 0 || o.nb[e - 1] >= 0) ? val[e * n_frows + r] : 0.0;
    v = face_row_chain(F, f[o.cA], -1.0, [&](int e) { return wv[e]; }, un) / wv[0];
  }
  if (face_inner(N, st & 0xffff, st >> 16)) {
    u[o.cA] = v;
    if (o.cB >= 0) u[o.cB] = v;
  } else {
    tmp[r] = v;
  }
}

// near-edge rows of one colour step: tmp -> both copies (ne = the colour's
// near-edge q per mode z, `len` each)
__global__ void k_face_write(int N, int64_t S, int64_t nfi, int len, const int* __restrict__ ne,
                             const FaceLP* __restrict__ flp, const uint32_t* __restrict__ fst,
                             const int* __restrict__ po, int64_t n_faces, const double* __restrict__ tmp,
                             double* __restrict__ u) {
  __shared__ int po_s[260];
  load_po(po_s, po, N);
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t fc = x / len;
  if (fc >= n_faces) return;
  const FaceLP& F = flp[fc];
  const int64_t q = ne[F.z * len + (x - fc * len)];
  const uint32_t st = fst[F.z * nfi + q];
  const int s = st & 0xffff, t = st >> 16;
  const FaceNode a = face_node(F.lA, N, s, t);
  const double v = tmp[fc * nfi + q];
  u[fslot(F.TA, S, po_s, a.i, a.j, a.k)] = v;
  if (F.TB >= 0) {
    const FaceNode b = face_node(F.lB, N, s, t);
    u[fslot(F.TB, S, po_s, b.i, b.j, b.k)] = v;
  }
}

// dir 0: gather (local -> global), 1: scatter (global -> both copies), 2: sync (A -> B)
__global__ void k_face_gather(int N, int64_t S, int64_t nfi, int64_t n_frows, const FaceLP* __restrict__ flp,
                              const uint32_t* __restrict__ fst, const int* __restrict__ fcidx,
                              const int* __restrict__ po, int64_t base_f, double* __restrict__ local,
                              double* __restrict__ glob, int dir) {
  __shared__ int po_s[260];
  load_po(po_s, po, N);
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_frows) return;
  const int64_t fc = r / nfi;
  const int64_t q = r - fc * nfi;
  const FaceLP& F = flp[fc];
  const uint32_t st = fst[F.z * nfi + q];
  const int s = st & 0xffff, t = st >> 16;
  const FaceNode a = face_node(F.lA, N, s, t);
  const int64_t sA = fslot(F.TA, S, po_s, a.i, a.j, a.k);
  int64_t sB = -1;
  if (F.TB >= 0) {
    const FaceNode b = face_node(F.lB, N, s, t);
    sB = fslot(F.TB, S, po_s, b.i, b.j, b.k);
  }
  const int64_t g = base_f + F.fid * nfi + fcidx[F.z * nfi + q];
  if (dir == 0) {
    glob[g] = local[sA];
  } else {
    const double v = dir == 1 ? glob[g] : local[sA];
    local[sA] = v;
    if (sB >= 0) local[sB] = v;
  }
}

__global__ void k_face_dot(int N, int64_t S, int64_t nfi, int64_t n_frows, const FaceLP* __restrict__ flp,
                           const uint32_t* __restrict__ fst, const int* __restrict__ po,
                           const double* __restrict__ av, const double* __restrict__ bv, double* __restrict__ part) {
  __shared__ int po_s[260];
  __shared__ double red[32];
  load_po(po_s, po, N);
  double acc = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_frows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fc = r / nfi;
    const FaceLP& F = flp[fc];
    const uint32_t st = fst[F.z * nfi + (r - fc * nfi)];
    const FaceNode a = face_node(F.lA, N, st & 0xffff, st >> 16);
    const int64_t sl = fslot(F.TA, S, po_s, a.i, a.j, a.k);
    acc += av[sl] * bv[sl];
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
  }
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

hhg_status face_apply(Ctx* c, Level& lv, int op, int mode, const double* u, const double* f, double* out) {
  if (lv.n_frows == 0) return HHG_OK;
  const double* val = op == HHG_OP_CONST_AFFINE ? lv.d_fval_cons : lv.d_fval;
  const double* fcoef = op == HHG_OP_SURROGATE_FACES ? lv.d_fcoef : nullptr;
  ProfScope ps(c, 2);
  k_face_apply<<<nblk(lv.n_frows, 128), 128, 0, c->stream>>>(lv.N, lv.S, lv.gi.nfi, lv.n_frows, lv.d_flp,
                                                             lv.d_fst, lv.d_po, val, u, f, out, mode, fcoef, lv.q);
  HHG_LAUNCHED(c);
  return HHG_OK;
}

hhg_status face_gs_step(Ctx* c, Level& lv, int op, int colour, double* u, const double* f) {
  const int64_t nfc = lv.fcol[colour + 1] - lv.fcol[colour];
  if (lv.n_frows == 0 || nfc == 0) return HHG_OK;
  const double* val = op == HHG_OP_CONST_AFFINE ? lv.d_fval_cons : lv.d_fval;
  const double* fcoef = op == HHG_OP_SURROGATE_FACES ? lv.d_fcoef : nullptr;
  const int64_t n = nfc * lv.n_flp;
  ProfScope ps(c, 2);
  k_face_gs<<<nblk(n, 128), 128, 0, c->stream>>>(lv.N, lv.S, lv.gi.nfi, nfc, lv.fcol[colour], lv.d_flp, lv.d_fst,
                                                 lv.d_po, lv.n_frows, val, u, f, lv.d_ftmp, fcoef, lv.q);
  HHG_LAUNCHED(c);
  const int len = lv.fne_len[colour];
  if (len > 0) {
    k_face_write<<<nblk((int64_t)len * lv.n_flp, 128), 128, 0, c->stream>>>(
        lv.N, lv.S, lv.gi.nfi, len, lv.d_fne[colour], lv.d_flp, lv.d_fst, lv.d_po, lv.n_flp, lv.d_ftmp, u);
    HHG_LAUNCHED(c);
  }
  return HHG_OK;
}

hhg_status face_gather(Ctx* c, Level& lv, const double* local, double* glob, int dir) {
  if (lv.n_frows == 0) return HHG_OK;
  k_face_gather<<<nblk(lv.n_frows, 128), 128, 0, c->stream>>>(lv.N, lv.S, lv.gi.nfi, lv.n_frows, lv.d_flp,
                                                              lv.d_fst, lv.d_fcidx, lv.d_po, lv.gi.base_f,
                                                              (double*)local, glob, dir);
  HHG_LAUNCHED(c);
  return HHG_OK;
}

hhg_status face_sync(Ctx* c, Level& lv, double* u) { return face_gather(c, lv, u, nullptr, 2); }

hhg_status face_dot(Ctx* c, Level& lv, const double* a, const double* b, double* part, int nblocks) {
  if (lv.n_frows == 0) {
    HHG_CK(c, cudaMemsetAsync(part, 0, nblocks * sizeof(double), c->stream));
    return HHG_OK;
  }
  k_face_dot<<<nblocks, 256, 0, c->stream>>>(lv.N, lv.S, lv.gi.nfi, lv.n_frows, lv.d_flp, lv.d_fst, lv.d_po, a, b,
                                            part);
  HHG_LAUNCHED(c);
  return HHG_OK;
}

// v at every copy of a shared face node <- sum of its copies (restriction partials)
__global__ void k_face_sumcopies(int N, int64_t S, int64_t nfi, int64_t n_frows, const FaceLP* __restrict__ flp,
                                 const uint32_t* __restrict__ fst, const int* __restrict__ po,
                                 double* __restrict__ v) {
  __shared__ int po_s[260];
  load_po(po_s, po, N);
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_frows) return;
  const int64_t fc = r / nfi;
  const FaceLP& F = flp[fc];
  const uint32_t st = fst[F.z * nfi + (r - fc * nfi)];
  if (F.TB < 0) return;
  const int s = st & 0xffff, t = st >> 16;
  const FaceNode a = face_node(F.lA, N, s, t), b = face_node(F.lB, N, s, t);
  const int64_t sA = fslot(F.TA, S, po_s, a.i, a.j, a.k), sB = fslot(F.TB, S, po_s, b.i, b.j, b.k);
  const double x = v[sA] + v[sB];
  v[sA] = x;
  v[sB] = x;
}

hhg_status face_sum_copies(Ctx* c, Level& lv, double* v) {
  if (lv.n_frows == 0) return HHG_OK;
  k_face_sumcopies<<<nblk(lv.n_frows, 128), 128, 0, c->stream>>>(lv.N, lv.S, lv.gi.nfi, lv.n_frows, lv.d_flp,
                                                                  lv.d_fst, lv.d_po, v);
  HHG_LAUNCHED(c);
  return HHG_OK;
}

}  // namespace hhg
