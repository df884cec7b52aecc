// Surrogate fit (setup) and the stencil test export.
//
// PAPER.md:501-534 (LSQP: a = argmin |A z - b|_2, sampling sets
// S_l = M_m(l,j), m(l,j) = min{l, max{1,j}}), PAPER.md:471-499 (IPOLY, 10 P2
// points of the shrunk tet), PAPER.md:647-668 (15 polynomials per macro and
// level, computed once in a setup phase), PAPER.md:1236-1238 (DGESV/DGELS).
// The sampling matrix A depends only on the level, so A^+ = R^-1 Q^T is formed
// once per level on the host by Householder QR and applied to all macros and
// all 15 right-hand sides as one batched product on the GPU.
#include <cmath>
#include <map>

#include "fem_device.cuh"
#include "hhg_internal.h"
#include "vol_kernels.cuh"

namespace hhg {

// Householder QR of A (n x m, row-major, n >= m) -> pinv (m x n) = R^-1 Q^T.
static bool pinv_qr(std::vector<double> A, int64_t n, int m, std::vector<double>& pinv) {
  std::vector<std::vector<double>> V(m);
  std::vector<double> beta(m, 0.0);
  std::vector<double> R(m * m, 0.0);
  for (int j = 0; j < m; ++j) {
    double norm = 0.0;
    for (int64_t i = j; i < n; ++i) norm += A[i * m + j] * A[i * m + j];
    norm = std::sqrt(norm);
    double alpha = A[j * m + j] > 0 ? -norm : norm;
    std::vector<double>& v = V[j];
    v.assign(n - j, 0.0);
    for (int64_t i = j; i < n; ++i) v[i - j] = A[i * m + j];
    v[0] -= alpha;
    double vv = 0.0;
    for (double x : v) vv += x * x;
    beta[j] = vv > 0 ? 2.0 / vv : 0.0;
    for (int c = j; c < m; ++c) {
      double s = 0.0;
      for (int64_t i = j; i < n; ++i) s += v[i - j] * A[i * m + c];
      s *= beta[j];
      for (int64_t i = j; i < n; ++i) A[i * m + c] -= s * v[i - j];
    }
  }
  double rmax = 0.0;
  for (int j = 0; j < m; ++j) {
    for (int c = j; c < m; ++c) R[j * m + c] = A[j * m + c];
    rmax = std::max(rmax, std::fabs(R[j * m + j]));
  }
  for (int j = 0; j < m; ++j)
    if (!(std::fabs(R[j * m + j]) > 1e-12 * rmax)) return false;
  // Q_thin (n x m) = H_0 ... H_{m-1} [I; 0]
  std::vector<double> Q(n * m, 0.0);
  for (int j = 0; j < m; ++j) Q[j * m + j] = 1.0;
  for (int j = m - 1; j >= 0; --j) {
    const std::vector<double>& v = V[j];
    for (int c = 0; c < m; ++c) {
      double s = 0.0;
      for (int64_t i = j; i < n; ++i) s += v[i - j] * Q[i * m + c];
      s *= beta[j];
      for (int64_t i = j; i < n; ++i) Q[i * m + c] -= s * v[i - j];
    }
  }
  // pinv = R^-1 Q^T : solve R X = Q^T column by column (X m x n)
  pinv.assign(m * n, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    for (int r = m - 1; r >= 0; --r) {
      double s = Q[i * m + r];
      for (int c = r + 1; c < m; ++c) s -= R[r * m + c] * pinv[c * n + i];
      pinv[r * n + i] = s / R[r * m + r];
    }
  }
  return true;
}

// B[T][s][w] = exact stencil at sample s of macro T
__global__ void k_sample_stencils(const double* __restrict__ geo, int N, const int* __restrict__ smp,
                                  int64_t ns, bool blended, double* __restrict__ B) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t T = blockIdx.y;
  if (s >= ns) return;
  double w[15];
  fem_partial(geo + T * 16, N, smp[3 * s], smp[3 * s + 1], smp[3 * s + 2], blended, w);
  for (int q = 0; q < 15; ++q) B[(T * ns + s) * 15 + q] = w[q];
}

// coef[T][w][c] = (sum_s pinv[c][s] B[T][s][w]) * scale[c]
__global__ void k_fit_coef(const double* __restrict__ pinv, const double* __restrict__ B, int64_t ns,
                           int mq, const double* __restrict__ scale, double* __restrict__ coef) {
  int64_t T = blockIdx.x;
  int t = threadIdx.x;
  if (t >= 15 * mq) return;
  int w = t / mq, c = t % mq;
  double acc = 0.0;
  const double* b = B + T * ns * 15;
  for (int64_t s = 0; s < ns; ++s) acc += pinv[c * ns + s] * b[s * 15 + w];
  coef[(T * 15 + w) * mq + c] = acc * scale[c];
}

// Surrogate face polynomials: per face fc and entry e,
// coef = pinv * (exact weights at the face sample nodes), index units.
__global__ void k_face_fit(const double* __restrict__ pinv, int ns, int nfc, const double* __restrict__ scale,
                           const FaceLP* __restrict__ flp, const int* __restrict__ sq, int64_t nfi,
                           int64_t n_frows, const double* __restrict__ fval, double* __restrict__ fcoef) {
  const int64_t fc = blockIdx.x;
  const int t = threadIdx.x;
  if (t >= 15 * nfc) return;
  const int e = t / nfc, cc = t % nfc;
  const int* q = sq + flp[fc].z * ns;
  const double* v = fval + e * n_frows + fc * nfi;
  double acc = 0.0;
  for (int x = 0; x < ns; ++x) acc += pinv[cc * ns + x] * v[q[x]];
  fcoef[(fc * 15 + e) * nfc + cc] = acc * scale[cc];
}

static hhg_status fit_faces(Ctx* c, Level& lv, int L, int q, int sampling_j) {
  if (lv.d_fcoef) cudaFree(lv.d_fcoef);
  lv.d_fcoef = nullptr;
  if (lv.n_flp == 0 || L < 3) return HHG_OK;
  const int N = lv.N;
  const int nfc = (q + 1) * (q + 2) / 2;
  std::vector<int> ea, eb;  // face exponents (a, b): by degree, b ascending
  for (int d = 0; d <= q; ++d)
    for (int b = 0; b <= d; ++b) ea.push_back(d - b), eb.push_back(b);
  const int l = L - 2, m = std::min(l, std::max(1, sampling_j));
  const int Nm = 1 << (m + 2), sc = 1 << (l - m);
  std::vector<int> st;
  for (int t = 1; t < Nm - 1; ++t)
    for (int s = 1; s < Nm - t; ++s) st.push_back(s * sc), st.push_back(t * sc);
  const int ns = (int)st.size() / 2;
  if (ns < nfc) return set_err(c, HHG_ERR_FIT, "fewer face samples than coefficients");
  std::vector<double> A((size_t)ns * nfc);
  for (int x = 0; x < ns; ++x)
    for (int cc = 0; cc < nfc; ++cc)
      A[(size_t)x * nfc + cc] = std::pow((double)st[2 * x] / N, ea[cc]) * std::pow((double)st[2 * x + 1] / N, eb[cc]);
  std::vector<double> pinv;
  if (!pinv_qr(A, ns, nfc, pinv)) return set_err(c, HHG_ERR_FIT, "rank-deficient face sampling matrix");
  std::vector<double> scale(nfc);
  for (int cc = 0; cc < nfc; ++cc) scale[cc] = std::ldexp(1.0, -L * (ea[cc] + eb[cc]));
  // row index (within a face) of every sample node, per row mode z
  const int64_t nfi = lv.gi.nfi;
  std::vector<int> sq(3 * (size_t)ns);
  for (int z = 0; z < 3; ++z) {
    std::map<uint32_t, int> inv;
    for (int64_t x = 0; x < nfi; ++x) inv[lv.h_fst[z * nfi + x]] = (int)x;
    for (int x = 0; x < ns; ++x) sq[z * ns + x] = inv.at((uint32_t)st[2 * x] | ((uint32_t)st[2 * x + 1] << 16));
  }
  double *d_pinv, *d_scale;
  int* d_sq;
  HHG_CK(c, cudaMalloc(&d_pinv, pinv.size() * sizeof(double)));
  HHG_CK(c, cudaMalloc(&d_scale, nfc * sizeof(double)));
  HHG_CK(c, cudaMalloc(&d_sq, sq.size() * sizeof(int)));
  HHG_CK(c, cudaMalloc(&lv.d_fcoef, (size_t)lv.n_flp * 15 * nfc * sizeof(double)));
  HHG_CK(c, cudaMemcpy(d_pinv, pinv.data(), pinv.size() * sizeof(double), cudaMemcpyHostToDevice));
  HHG_CK(c, cudaMemcpy(d_scale, scale.data(), nfc * sizeof(double), cudaMemcpyHostToDevice));
  HHG_CK(c, cudaMemcpy(d_sq, sq.data(), sq.size() * sizeof(int), cudaMemcpyHostToDevice));
  k_face_fit<<<(unsigned)lv.n_flp, ((15 * nfc + 31) / 32) * 32, 0, c->stream>>>(
      d_pinv, ns, nfc, d_scale, lv.d_flp, d_sq, nfi, lv.n_frows, lv.d_fval, lv.d_fcoef);
  HHG_LAUNCHED(c);
  HHG_CK(c, cudaStreamSynchronize(c->stream));
  cudaFree(d_pinv);
  cudaFree(d_scale);
  cudaFree(d_sq);
  return HHG_OK;
}

// Level 2 (l = 0): single interior node, exact stencil as the constant term.
__global__ void k_exact_const(const double* __restrict__ geo, int N, int mq, bool blended,
                              double* __restrict__ coef) {
  int64_t T = blockIdx.x;
  if (threadIdx.x != 0) return;
  double w[15];
  fem_partial(geo + T * 16, N, 1, 1, 1, blended, w);
  for (int q = 0; q < 15; ++q) {
    coef[(T * 15 + q) * mq] = w[q];
    for (int c = 1; c < mq; ++c) coef[(T * 15 + q) * mq + c] = 0.0;
  }
}

// Sampling set of level L (lattice indices, [n][3]): LSQP S_l = M_m(l,j)
// embedded at level l (index x 2^(l-m), reading R10), or the
// 10 IPOLY points.
static std::vector<int> sample_set(int L, hhg_fit_method method, int sampling_j) {
  std::vector<int> smp;
  const int l = L - 2;
  if (method == HHG_FIT_IPOLY) {
    const int a = (1 << (l + 2)) - 3, b = (1 << (l + 1)) - 1;
    const int pts[10][3] = {{1, 1, 1}, {1, 1, a}, {1, a, 1}, {a, 1, 1}, {1, 1, b},
                            {1, b, 1}, {b, 1, 1}, {1, b, b}, {b, 1, b}, {b, b, 1}};
    for (auto& p : pts) smp.insert(smp.end(), p, p + 3);
    return smp;
  }
  const int m = std::min(l, std::max(1, sampling_j));
  const int Nm = 1 << (m + 2), sc = 1 << (l - m);
  for (int k = 1; k < Nm; ++k)
    for (int j = 1; j < Nm - k; ++j)
      for (int i = 1; i < Nm - k - j; ++i) {
        smp.push_back(i * sc);
        smp.push_back(j * sc);
        smp.push_back(k * sc);
      }
  return smp;
}

// flag |= 1 if the surrogate centre weight s_mc(i,j,k) <= 0 (or NaN) at an
// interior node: the GS update divides by it (eq. iteration-scheme,
// PAPER.md:1306-1315).  Evaluated like node_weights (vol_kernels.cuh).
__global__ void k_check_centre(int N, int64_t P, const double* __restrict__ coef, int mq, int* __restrict__ flag) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t T = blockIdx.y;
  if (p >= P) return;
  int i, j, k;
  decode_pos(N, p, i, j, k);
  if (i < 1 || j < 1 || k < 1 || i + j + k > N - 1) return;
  double s[15];
  node_weights(HHG_OP_SURROGATE, N, i, j, k, nullptr, coef + T * 15 * mq, mq, nullptr, false, s);
  if (!(s[kMC] > 0.0)) atomicOr(flag, 1);
}

static hhg_status check_centre(Ctx* c, Level& lv) {
  if (!c->d_flag) HHG_CK(c, cudaMalloc(&c->d_flag, sizeof(int)));
  HHG_CK(c, cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
  if (c->nt_local > 0) {
    dim3 g((unsigned)((lv.P + 127) / 128), (unsigned)c->nt_local);
    k_check_centre<<<g, 128, 0, c->stream>>>(lv.N, lv.P, lv.d_coef, lv.mq, c->d_flag);
    HHG_LAUNCHED(c);
  }
  hhg_status st = face_centre_check(c, lv, c->d_flag + 0);
  if (st != HHG_OK) return st;
  int h = 0;
  HHG_CK(c, cudaMemcpyAsync(&h, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  HHG_CK(c, cudaStreamSynchronize(c->stream));
  lv.centre_bad = (h & 1) != 0;
  lv.fcentre_bad = (h & 2) != 0;
  return HHG_OK;
}

// q <= 2: the march kernels read coefficients zero-padded to the q = 2 layout
// (the degree-major exponent list of q is a prefix of that of q = 2).
static hhg_status make_coef10(Ctx* c, Level& lv, int q, int mq) {
  if (lv.d_coef10) cudaFree(lv.d_coef10);
  lv.d_coef10 = nullptr;
  if (lv.d_cC) cudaFree(lv.d_cC);  // derived from d_coef10 on first use (ops.cu)
  lv.d_cC = nullptr;
  if (q > 2) return HHG_OK;
  HHG_CK(c, cudaMalloc(&lv.d_coef10, c->nt_local * 150 * sizeof(double)));
  HHG_CK(c, cudaMemsetAsync(lv.d_coef10, 0, c->nt_local * 150 * sizeof(double), c->stream));
  HHG_CK(c, cudaMemcpy2DAsync(lv.d_coef10, 10 * sizeof(double), lv.d_coef, mq * sizeof(double),
                              mq * sizeof(double), c->nt_local * 15, cudaMemcpyDeviceToDevice, c->stream));
  return HHG_OK;
}

// Fit one level L >= 3: coefficients = A^+ B with B the exact FEM stencils at
// the sampling set (d_samples = nullptr) or the caller's planted samples
// (d_samples [nt_local][n][15], hhg_fit_from_samples).
static hhg_status fit_level(Ctx* c, Level& lv, int L, int q, hhg_fit_method method, int sampling_j,
                            const double* d_samples) {
  const int N = lv.N;
  const int mq = n_coeffs(q);
  std::vector<int> el, em, en;
  exponents(q, el, em, en);
  const std::vector<int> smp = sample_set(L, method, sampling_j);
  const int64_t ns = (int64_t)smp.size() / 3;
  if (ns < mq) return set_err(c, HHG_ERR_FIT, "fewer sampling points than coefficients");
  std::vector<double> A(ns * mq);
  for (int64_t s = 0; s < ns; ++s)
    for (int cc = 0; cc < mq; ++cc)
      A[s * mq + cc] = std::pow((double)smp[3 * s] / N, el[cc]) * std::pow((double)smp[3 * s + 1] / N, em[cc]) *
                       std::pow((double)smp[3 * s + 2] / N, en[cc]);
  std::vector<double> pinv;
  if (!pinv_qr(A, ns, mq, pinv))
    return set_err(c, HHG_ERR_FIT, "rank-deficient sampling matrix at level " + std::to_string(L));
  // index-unit scaling: x = i/N => a_lmn / N^(l+m+n) (exact powers of two)
  std::vector<double> scale(mq);
  for (int cc = 0; cc < mq; ++cc) scale[cc] = std::ldexp(1.0, -L * (el[cc] + em[cc] + en[cc]));
  if (lv.d_coef) cudaFree(lv.d_coef);
  lv.d_coef = nullptr;
  HHG_CK(c, cudaMalloc(&lv.d_coef, c->nt_local * 15 * mq * sizeof(double)));
  lv.q = q;
  lv.mq = mq;
  int* d_smp;
  double *d_pinv, *d_B = nullptr, *d_scale;
  HHG_CK(c, cudaMalloc(&d_smp, smp.size() * sizeof(int)));
  HHG_CK(c, cudaMalloc(&d_pinv, pinv.size() * sizeof(double)));
  HHG_CK(c, cudaMalloc(&d_scale, mq * sizeof(double)));
  HHG_CK(c, cudaMemcpyAsync(d_smp, smp.data(), smp.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  HHG_CK(c, cudaMemcpyAsync(d_pinv, pinv.data(), pinv.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  HHG_CK(c, cudaMemcpyAsync(d_scale, scale.data(), mq * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  if (!d_samples) {
    HHG_CK(c, cudaMalloc(&d_B, c->nt_local * ns * 15 * sizeof(double)));
    dim3 g1((unsigned)((ns + 127) / 128), (unsigned)c->nt_local);
    k_sample_stencils<<<g1, 128, 0, c->stream>>>(c->d_geo, N, d_smp, ns, c->blended, d_B);
    HHG_LAUNCHED(c);
  }
  k_fit_coef<<<(unsigned)c->nt_local, ((15 * mq + 31) / 32) * 32, 0, c->stream>>>(
      d_pinv, d_samples ? d_samples : d_B, ns, mq, d_scale, lv.d_coef);
  HHG_LAUNCHED(c);
  HHG_CK(c, cudaStreamSynchronize(c->stream));
  cudaFree(d_smp);
  cudaFree(d_pinv);
  if (d_B) cudaFree(d_B);
  cudaFree(d_scale);
  return make_coef10(c, lv, q, mq);
}

static hhg_status fit_args(Ctx* c, int q, hhg_fit_method method) {
  if (!c) return HHG_ERR_INVALID;
  if (c->poisoned) return HHG_ERR_CUDA;
  if (c->host_only) return set_err(c, HHG_ERR_STATE, "plan-only context");
  if (q < 0 || q > 4) return set_err(c, HHG_ERR_INVALID, "q must be in 0..4 (PAPER.md:530-534)");
  if (method != HHG_FIT_LSQP && method != HHG_FIT_IPOLY) return set_err(c, HHG_ERR_INVALID, "method");
  if (method == HHG_FIT_IPOLY && q != 2)
    return set_err(c, HHG_ERR_INVALID, "IPOLY points are defined for q = 2 (PAPER.md:490-499)");
  if (c->vc_graph) {  // a cached V-cycle graph holds the old coefficient buffers
    cudaStreamSynchronize(c->stream);
    cudaGraphExecDestroy(c->vc_graph);
    c->vc_graph = nullptr;
  }
  return HHG_OK;
}

}  // namespace hhg

using namespace hhg;

extern "C" hhg_status hhg_fit_surrogates(hhg_ctx ctx, int q, hhg_fit_method method, int sampling_j) {
  Ctx* c = (Ctx*)ctx;
  hhg_status st = fit_args(c, q, method);
  if (st != HHG_OK) return st;
  const int mq = n_coeffs(q);
  bool bad = false;
  for (int L = 2; L <= c->L_max; ++L) {
    Level& lv = c->levels[L];
    if (L == 2) {  // l = 0: the exact stencil of the single interior node
      if (lv.d_coef) cudaFree(lv.d_coef);
      HHG_CK(c, cudaMalloc(&lv.d_coef, c->nt_local * 15 * mq * sizeof(double)));
      lv.q = q;
      lv.mq = mq;
      k_exact_const<<<(unsigned)c->nt_local, 32, 0, c->stream>>>(c->d_geo, lv.N, mq, c->blended, lv.d_coef);
      HHG_LAUNCHED(c);
      if ((st = make_coef10(c, lv, q, mq)) != HHG_OK) return st;
    } else {
      if ((st = fit_level(c, lv, L, q, method, sampling_j, nullptr)) != HHG_OK) return st;
      if ((st = fit_faces(c, lv, L, q, sampling_j)) != HHG_OK) return st;
    }
    if ((st = check_centre(c, lv)) != HHG_OK) return st;
    bad = bad || lv.centre_bad || lv.fcentre_bad;
    lv.fitted = true;
  }
  HHG_CK(c, cudaStreamSynchronize(c->stream));
  if (bad)
    return set_err(c, HHG_ERR_NUMERIC,
                   "non-positive surrogate centre weight: the fit is installed (apply/residual work), "
                   "the GS smoother and V-cycle refuse it");
  return HHG_OK;
}

extern "C" hhg_status hhg_sample_nodes(hhg_ctx ctx, int L, hhg_fit_method method, int sampling_j, int32_t* ijk,
                                       int64_t* n) {
  Ctx* c = (Ctx*)ctx;
  if (!c || !n || L < 3 || L > c->L_max) return c ? set_err(c, HHG_ERR_INVALID, "L must be in 3..L_max") : HHG_ERR_INVALID;
  if (method != HHG_FIT_LSQP && method != HHG_FIT_IPOLY) return set_err(c, HHG_ERR_INVALID, "method");
  const std::vector<int> smp = sample_set(L, method, sampling_j);
  *n = (int64_t)smp.size() / 3;
  if (ijk) std::copy(smp.begin(), smp.end(), ijk);
  return HHG_OK;
}

extern "C" hhg_status hhg_fit_from_samples(hhg_ctx ctx, int L, int q, hhg_fit_method method, int sampling_j,
                                           const double* samples) {
  Ctx* c = (Ctx*)ctx;
  hhg_status st = fit_args(c, q, method);
  if (st != HHG_OK) return st;
  if (L < 3 || L > c->L_max || !samples) return set_err(c, HHG_ERR_INVALID, "L must be in 3..L_max, samples non-NULL");
  const int64_t ns = (int64_t)sample_set(L, method, sampling_j).size() / 3;
  const size_t bytes = (size_t)c->nt_local * ns * 15 * sizeof(double);
  cudaPointerAttributes pa;
  const bool dev = cudaPointerGetAttributes(&pa, samples) == cudaSuccess &&
                   (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged);
  cudaGetLastError();
  double* d_s = nullptr;
  if (!dev) {
    HHG_CK(c, cudaMalloc(&d_s, std::max<size_t>(bytes, 8)));
    HHG_CK(c, cudaMemcpyAsync(d_s, samples, bytes, cudaMemcpyHostToDevice, c->stream));
  }
  Level& lv = c->levels[L];
  st = fit_level(c, lv, L, q, method, sampling_j, dev ? samples : d_s);
  if (d_s) cudaFree(d_s);
  if (st != HHG_OK) return st;
  // planted samples define no face polynomials: SURROGATE_FACES is unavailable on this level
  if (lv.d_fcoef) cudaFree(lv.d_fcoef);
  lv.d_fcoef = nullptr;
  if ((st = check_centre(c, lv)) != HHG_OK) return st;
  lv.fitted = true;
  if (lv.centre_bad) return set_err(c, HHG_ERR_NUMERIC, "non-positive surrogate centre weight (installed; GS refuses it)");
  return HHG_OK;
}
