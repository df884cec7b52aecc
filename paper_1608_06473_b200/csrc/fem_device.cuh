// Device helpers: lattice decode, blended coordinates, node-wise FEM stencil.
#pragma once
#include "hhg_internal.h"

namespace hhg {

__device__ __constant__ static const int kDir[15][3] = HHG_DIRS_INIT;

// Decode a macro-local lattice position -> (i,j,k) (layout in include/hhg.h).
__host__ __device__ inline void decode_pos(int N, int64_t p, int& i, int& j, int& k) {
  int lo = 0, hi = N;  // largest k with plane_off(k) <= p
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (plane_off(N, mid) <= p) lo = mid; else hi = mid - 1;
  }
  k = lo;
  int64_t c = p - plane_off(N, k);
  int64_t d = (int64_t)((sqrt(8.0 * (double)c + 1.0) - 1.0) * 0.5);
  while ((d + 1) * (d + 2) / 2 <= c) ++d;
  while (d * (d + 1) / 2 > c) --d;
  j = (int)(c - d * (d + 1) / 2);
  i = (int)d - j;
}

// Phi_T(Psi_T(i,j,k)): geo = [4][4] (x,y,z,r) of the local vertices.
__host__ __device__ inline void node_xyz(const double* geo, int N, int i, int j, int k, bool blended,
                                         double x[3]) {
  const double invN = 1.0 / (double)N;
  const double l[4] = {(double)(N - i - j - k) * invN, (double)i * invN, (double)j * invN,
                       (double)k * invN};
  double X[3] = {0.0, 0.0, 0.0};
  double r = 0.0;
  for (int v = 0; v < 4; ++v) {
    X[0] += l[v] * geo[4 * v + 0];
    X[1] += l[v] * geo[4 * v + 1];
    X[2] += l[v] * geo[4 * v + 2];
    r += l[v] * geo[4 * v + 3];
  }
  if (blended) {
    double s = r / sqrt(X[0] * X[0] + X[1] * X[1] + X[2] * X[2]);
    X[0] *= s; X[1] *= s; X[2] *= s;
  }
  x[0] = X[0]; x[1] = X[1]; x[2] = X[2];
}

__device__ inline int dir_of(int di, int dj, int dk) {
  for (int w = 0; w < 15; ++w)
    if (kDir[w][0] == di && kDir[w][1] == dj && kDir[w][2] == dk) return w;
  return -1;
}

// Partial node stencil of lattice node (i,j,k) from the fine tets of this
// macro containing it (all 24 for an interior node).  out[15] in direction order.
__device__ inline void fem_partial(const double* geo, int N, int i, int j, int k, bool blended,
                                   double out[15]) {
  double P[15][3];
  for (int w = 0; w < 15; ++w) {
    out[w] = 0.0;
    int a = i + kDir[w][0], b = j + kDir[w][1], c = k + kDir[w][2];
    if (a >= 0 && b >= 0 && c >= 0 && a + b + c <= N) node_xyz(geo, N, a, b, c, blended, P[w]);
  }
  const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  const int X = i + j + k, Y = j + k, Z = k;
  for (int s = 0; s < 6; ++s) {
    int path[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {1, 1, 1}};
    path[1][perms[s][0]] = 1;
    path[2][perms[s][0]] = 1;
    path[2][perms[s][1]] = 1;
    for (int m = 0; m < 4; ++m) {
      int bx = X - path[m][0], by = Y - path[m][1], bz = Z - path[m][2];
      int wv[4];
      bool ok = true;
      for (int a = 0; a < 4; ++a) {
        int vx = bx + path[a][0], vy = by + path[a][1], vz = bz + path[a][2];
        if (!(vx <= N && vx >= vy && vy >= vz && vz >= 0)) { ok = false; break; }
        wv[a] = dir_of(vx - vy - i, vy - vz - j, vz - k);
      }
      if (!ok) continue;
      const double* p0 = P[wv[0]];
      double e1[3], e2[3], e3[3];
      for (int d = 0; d < 3; ++d) {
        e1[d] = P[wv[1]][d] - p0[d];
        e2[d] = P[wv[2]][d] - p0[d];
        e3[d] = P[wv[3]][d] - p0[d];
      }
      double c23[3] = {e2[1] * e3[2] - e2[2] * e3[1], e2[2] * e3[0] - e2[0] * e3[2],
                       e2[0] * e3[1] - e2[1] * e3[0]};
      double c31[3] = {e3[1] * e1[2] - e3[2] * e1[1], e3[2] * e1[0] - e3[0] * e1[2],
                       e3[0] * e1[1] - e3[1] * e1[0]};
      double c12[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                       e1[0] * e2[1] - e1[1] * e2[0]};
      double det = e1[0] * c23[0] + e1[1] * c23[1] + e1[2] * c23[2];
      double g[4][3];
      for (int d = 0; d < 3; ++d) {
        g[1][d] = c23[d] / det;
        g[2][d] = c31[d] / det;
        g[3][d] = c12[d] / det;
        g[0][d] = -(g[1][d] + g[2][d] + g[3][d]);
      }
      double vol = fabs(det) / 6.0;
      for (int b = 0; b < 4; ++b)
        out[wv[b]] += vol * (g[m][0] * g[b][0] + g[m][1] * g[b][1] + g[m][2] * g[b][2]);
    }
  }
}

}  // namespace hhg
