// Face-row helpers shared by faces.cu and coarse.cu: the lattice node of
// face point (s,t) in one of the face's macros and the slots of a face row.
#pragma once
#include "fem_device.cuh"
#include "hhg_internal.h"

namespace hhg {

struct FaceNode {
  int i, j, k;
};

__device__ __forceinline__ FaceNode face_node(const int8_t* l, int N, int s, int t) {
  int w[4] = {0, 0, 0, 0};
  w[l[0]] = N - s - t;
  w[l[1]] = s;
  w[l[2]] = t;
  return FaceNode{w[1], w[2], w[3]};
}

__device__ __forceinline__ int64_t fslot(int64_t T, int64_t S, const int* po, int i, int j, int k) {
  return T * S + po[k] + col_idx(i, j);
}

// Slots of one face row: centre in A (and B), 14 neighbours.
struct FaceRowSlots {
  int64_t cA, cB;      // centre copies (cB = -1 if none)
  int64_t nb[14];      // neighbours for entries 1..14 (-1 if absent)
};

__device__ __forceinline__ void face_row_slots(const FaceLP& F, int N, int64_t S, const int* po, int s, int t,
                                               FaceRowSlots& o) {
  const FaceNode a = face_node(F.lA, N, s, t);
  o.cA = fslot(F.TA, S, po, a.i, a.j, a.k);
#pragma unroll
  for (int e = 0; e < 10; ++e)
    o.nb[e] = fslot(F.TA, S, po, a.i + F.off[e][0], a.j + F.off[e][1], a.k + F.off[e][2]);
  if (F.TB >= 0) {
    const FaceNode b = face_node(F.lB, N, s, t);
    o.cB = fslot(F.TB, S, po, b.i, b.j, b.k);
#pragma unroll
    for (int e = 10; e < 14; ++e)
      o.nb[e] = fslot(F.TB, S, po, b.i + F.off[e][0], b.j + F.off[e][1], b.k + F.off[e][2]);
  } else {
    o.cB = -1;
#pragma unroll
    for (int e = 10; e < 14; ++e) o.nb[e] = -1;
  }
}

__device__ __forceinline__ void load_po(int* po_s, const int* po, int N) {
  for (int p = threadIdx.x; p <= N + 1; p += blockDim.x) po_s[p] = po[p];
  __syncthreads();
}

}  // namespace hhg
