// Node-wise exact FEM stencils on the blended (or affine) fine mesh.
//
// the stencil of node I is the sum of the local stiffness
// matrices K_T[a][b] = |T| grad(lambda_a).grad(lambda_b) of the fine tets
// adjacent to I; the fine tets of a macro are its Bey refinement, i.e. the
// Kuhn simplices of x=i+j+k, y=j+k, z=k restricted to N >= x >= y >= z >= 0
// (reading R4).  Fine vertices are Phi_T(Psi_T(i,j,k)).
// For a node on a macro face/edge/vertex only the fine tets inside the given
// macro contribute ("partial stencil"); summing partials over all macros that
// contain the node gives the global FEM row (used for lower primitives,
// PAPER.md:321-327).  Used at setup (sampling for the fit, lower-primitive
// rows) and by the node-wise FEM comparison operator.
#include "fem_device.cuh"
#include "hhg_internal.h"

namespace hhg {

__global__ void k_fem_partial_slots(const double* __restrict__ geo, int N, int64_t S,
                                    const uint32_t* __restrict__ slots, int64_t n, bool blended,
                                    double* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint32_t s = slots[t];
  int64_t T = s / S;
  int i, j, k;
  decode_pos(N, s - T * S, i, j, k);
  double w[15];
  fem_partial(geo + T * 16, N, i, j, k, blended, w);
  for (int q = 0; q < 15; ++q) out[t * 15 + q] = w[q];
}

hhg_status launch_fem_partial(Ctx* c, int L, const uint32_t* d_slots, int64_t n, bool blended,
                              double* d_out15) {
  if (n == 0) return HHG_OK;
  const Level& lv = c->levels[L];
  k_fem_partial_slots<<<(unsigned)((n + 127) / 128), 128, 0, c->stream>>>(
      c->d_geo, lv.N, lv.S, d_slots, n, blended, d_out15);
  HHG_LAUNCHED(c);
  return HHG_OK;
}

// One thread per lower-primitive row: sum the partial stencils of all copies
// (ascending macro order => deterministic) into the row's CSR entries.
__global__ void k_lp_values(const double* __restrict__ geo, int N, int64_t S, int64_t n_rows,
                            const uint64_t* __restrict__ row_ptr,
                            const uint64_t* __restrict__ copy_ptr,
                            const uint32_t* __restrict__ copy, const uint32_t* __restrict__ cord,
                            const uint8_t* __restrict__ cmap, bool blended, double* __restrict__ val) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  uint64_t e0 = row_ptr[r], e1 = row_ptr[r + 1];
  for (uint64_t e = e0; e < e1; ++e) val[e] = 0.0;
  // copies in canonical order (cord: global macro id), so the sums are partition-independent
  for (uint64_t x = copy_ptr[r]; x < copy_ptr[r + 1]; ++x) {
    const uint64_t cc = cord[x];
    uint32_t s = copy[cc];
    int64_t T = s / S;
    int i, j, k;
    decode_pos(N, s - T * S, i, j, k);
    double w[15];
    fem_partial(geo + T * 16, N, i, j, k, blended, w);
    for (int q = 0; q < 15; ++q) {
      uint8_t m = cmap[cc * 16 + q];
      if (m != 255) val[e0 + m] += w[q];
    }
  }
}

hhg_status build_lp_values(Ctx* c, Level& lv, const std::vector<uint8_t>& cmap, const std::vector<uint32_t>& cord) {
  if (lv.n_rows == 0) return HHG_OK;
  uint8_t* d_cmap = nullptr;
  uint32_t* d_cord = nullptr;
  HHG_CK(c, cudaMalloc(&d_cmap, cmap.size()));
  HHG_CK(c, cudaMemcpyAsync(d_cmap, cmap.data(), cmap.size(), cudaMemcpyHostToDevice, c->stream));
  HHG_CK(c, cudaMalloc(&d_cord, cord.size() * sizeof(uint32_t)));
  HHG_CK(c, cudaMemcpyAsync(d_cord, cord.data(), cord.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
  unsigned grid = (unsigned)((lv.n_rows + 127) / 128);
  k_lp_values<<<grid, 128, 0, c->stream>>>(c->d_geo, lv.N, lv.S, lv.n_rows, lv.d_row_ptr,
                                          lv.d_copy_ptr, lv.d_copy, d_cord, d_cmap, true, lv.d_val);
  HHG_LAUNCHED(c);
  k_lp_values<<<grid, 128, 0, c->stream>>>(c->d_geo, lv.N, lv.S, lv.n_rows, lv.d_row_ptr,
                                          lv.d_copy_ptr, lv.d_copy, d_cord, d_cmap, false, lv.d_val_cons);
  HHG_LAUNCHED(c);
  HHG_CK(c, cudaStreamSynchronize(c->stream));
  HHG_CK(c, cudaFree(d_cmap));
  HHG_CK(c, cudaFree(d_cord));
  return HHG_OK;
}

}  // namespace hhg
