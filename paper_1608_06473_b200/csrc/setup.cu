// Host setup: mesh ingest/validation, topology, canonical numbering, per-level
// layouts, lower-primitive rows, gather/scatter, errors (include/hhg.h).
//
// PAPER.md:202-207 (unstructured macro mesh T_-2), 295-338 (HHG primitives:
// vertex/edge/face/volume; ghost copies of lower primitives), 321-327 (lower
// primitive stencils assembled from local stiffness matrices), 372-379
// (index set).  Canonical numbering: DESIGN.md.
#include <omp.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <numeric>

#include "fem_device.cuh"
#include "hhg_internal.h"

namespace hhg {

const int kDirHost[15][3] = HHG_DIRS_INIT;

hhg_status set_err(Ctx* c, hhg_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

hhg_status check_cuda(Ctx* c, cudaError_t e, const char* what) {
  std::string m = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  if (c) {
    c->err = m;
    c->poisoned = true;
  }
  if (e == cudaErrorMemoryAllocation) return HHG_ERR_OOM;
  return HHG_ERR_CUDA;
}

int n_coeffs(int q) { return (q + 3) * (q + 2) * (q + 1) / 6; }

void exponents(int q, std::vector<int>& l, std::vector<int>& m, std::vector<int>& n) {
  l.clear(); m.clear(); n.clear();
  for (int d = 0; d <= q; ++d)
    for (int a = d; a >= 0; --a)
      for (int b = d - a; b >= 0; --b) {
        l.push_back(a); m.push_back(b); n.push_back(d - a - b);
      }
}

namespace {

struct RowDesc {
  int8_t type;  // 0 vertex 1 edge 2 face
  int32_t a, b; // edge: m ; face: s, t
  int64_t id;   // vertex / edge / face id
};

struct Topology {
  std::vector<int64_t> ekey, fkey;               // sorted unique keys
  std::vector<std::vector<int32_t>> vinc, einc, finc;  // incident blocks (ascending global id)
  std::vector<uint8_t> vdir, edir, fdir;
  std::vector<int32_t> vown, eown, fown;         // owner rank of each primitive
};

inline void corner(int lv, int N, int w[4]) {
  w[0] = w[1] = w[2] = w[3] = 0;
  w[lv] = N;
}

}  // namespace

static int local_of(const int64_t* tv, int64_t g) {
  for (int v = 0; v < 4; ++v)
    if (tv[v] == g) return v;
  return -1;
}

// Structured rows of the non-Dirichlet faces (FaceLP, hhg_internal.h).
static hhg_status build_face_rows(Ctx* c, Topology& tp, Level& lv) {
  const int N = lv.N;
  const int64_t nfi = lv.gi.nfi;
  // In-face node orders, one per "row mode" z in {0,1,2}: colour-major
  // ((s+2t) mod 3, the face colouring of the GS class steps), then rows of
  // constant weight w_z on the face's z-th sorted vertex, inner index moving
  // weight between the two other vertices.  A face uses the mode whose inner
  // direction stays inside one lattice plane of its primary macro (contiguous
  // along a diagonal when the face contains local vertices 1 and 2), so
  // consecutive threads touch neighbouring addresses.
  std::vector<uint32_t> fst;
  std::vector<int> fcidx;
  for (int z = 0; z < 3; ++z) {
    const int x = z == 0 ? 1 : 0, y = z == 2 ? 1 : 2;
    for (int col = 0; col < 3; ++col) {
      if (z == 0) lv.fcol[col] = (int)(fst.size());
      for (int wz = 1; wz <= N - 2; ++wz)
        for (int wy = 1; wy <= N - 1 - wz; ++wy) {
          int w[3];
          w[z] = wz;
          w[y] = wy;
          w[x] = N - wz - wy;
          const int s = w[1], t = w[2];
          if ((s + 2 * t) % 3 != col) continue;
          fst.push_back((uint32_t)s | ((uint32_t)t << 16));
          fcidx.push_back((t - 1) * (N - 1) - (t - 1) * t / 2 + (s - 1));
        }
    }
    if (z == 0) lv.fcol[3] = (int)fst.size();
  }
  const int D[6][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}, {-1, 1}, {1, -1}};
  std::vector<FaceLP> flp;
  for (int64_t f = 0; f < c->n_f; ++f) {
    if (tp.fdir[f] || tp.finc[f].empty() || tp.fown[f] != c->rank) continue;
    const int64_t key = tp.fkey[f];
    const int64_t vc = key % c->nv, ab = key / c->nv;
    const int64_t va = ab / c->nv, vb = ab % c->nv;
    FaceLP F{};
    F.fid = f;
    F.TA = tp.finc[f][0];
    F.TB = tp.finc[f].size() > 1 ? tp.finc[f][1] : -1;
    {
      // primary frame: prefer the macro in which the face contains local vertices 1 and 2
      // (contiguous rows); only swap between two local macros (the exchange plan serves A)
      auto opp = [&](int T) {
        const int64_t* gv = c->topo[T].gv;
        return 6 - local_of(gv, va) - local_of(gv, vb) - local_of(gv, vc);
      };
      if (F.TB >= 0 && F.TA < c->nt_local && F.TB < c->nt_local) {
        const int la = opp(F.TA), lb = opp(F.TB);
        if ((la == 1 || la == 2) && (lb == 0 || lb == 3)) std::swap(F.TA, F.TB);
      }
    }
    F.bfirst = (int8_t)(F.TB >= 0 && c->topo[F.TB].gT < c->topo[F.TA].gT);
    for (int side = 0; side < 2; ++side) {
      const int T = side == 0 ? F.TA : F.TB;
      int8_t* l = side == 0 ? F.lA : F.lB;
      int8_t* map = side == 0 ? F.mapA : F.mapB;
      for (int w = 0; w < 15; ++w) map[w] = -1;
      if (T < 0) continue;
      const int64_t* gv = c->topo[T].gv;
      l[0] = (int8_t)local_of(gv, va);
      l[1] = (int8_t)local_of(gv, vb);
      l[2] = (int8_t)local_of(gv, vc);
      const int lf = 6 - l[0] - l[1] - l[2];
      int n_into = 0;
      for (int w = 0; w < 15; ++w) {
        const int* dv = kDirHost[w];
        const int dw[4] = {-dv[0] - dv[1] - dv[2], dv[0], dv[1], dv[2]};
        if (w == kMC) { map[w] = 0; continue; }
        if (dw[lf] == 0) {  // in-face: (ds, dt) = (dw[lb], dw[lc])
          for (int e = 0; e < 6; ++e)
            if (D[e][0] == dw[l[1]] && D[e][1] == dw[l[2]]) {
              map[w] = (int8_t)(1 + e);
              if (side == 0) for (int x = 0; x < 3; ++x) F.off[e][x] = (int8_t)dv[x];
            }
        } else if (dw[lf] == 1) {
          map[w] = (int8_t)((side == 0 ? 7 : 11) + n_into);
          for (int x = 0; x < 3; ++x) F.off[(side == 0 ? 6 : 10) + n_into][x] = (int8_t)dv[x];
          ++n_into;
        }
      }
      if (n_into != 4) return set_err(c, HHG_ERR_MESH, "face with != 4 into-macro directions");
    }
    {
      const int lf = 6 - F.lA[0] - F.lA[1] - F.lA[2];
      const int want = lf == 3 ? 0 : 3;  // hold the weight of local vertex 0 (k=0 face) or 3 (keep k)
      F.z = 0;
      for (int p = 0; p < 3; ++p)
        if (F.lA[p] == want) F.z = (int8_t)p;
    }
    flp.push_back(F);
  }
  lv.n_flp = (int64_t)flp.size();
  lv.n_frows = lv.n_flp * nfi;
  lv.h_flp = flp;
  lv.h_fst = fst;
  lv.h_fcidx = fcidx;
  if (c->host_only) return HHG_OK;
  std::vector<int> po(N + 2);
  for (int p = 0; p <= N + 1; ++p) po[p] = (int)plane_off(N, p);
  auto up = [&](auto*& dptr, const auto& vec) -> hhg_status {
    using TT = typename std::remove_reference<decltype(vec)>::type::value_type;
    size_t bytes = std::max<size_t>(vec.size(), 1) * sizeof(TT);
    HHG_CK(c, cudaMalloc((void**)&dptr, bytes));
    if (!vec.empty())
      HHG_CK(c, cudaMemcpy(dptr, vec.data(), vec.size() * sizeof(TT), cudaMemcpyHostToDevice));
    return HHG_OK;
  };
  hhg_status st;
  if ((st = up(lv.d_flp, flp)) != HHG_OK) return st;
  if ((st = up(lv.d_fst, fst)) != HHG_OK) return st;
  if ((st = up(lv.d_fcidx, fcidx)) != HHG_OK) return st;
  if ((st = up(lv.d_po, po)) != HHG_OK) return st;
  // near-edge rows (k_face_gs writes them through tmp; k_face_write visits only these)
  for (int col = 0; col < 3; ++col) {
    std::vector<int> ne[3];
    for (int z = 0; z < 3; ++z)
      for (int q = lv.fcol[col]; q < lv.fcol[col + 1]; ++q) {
        const int s = fst[z * nfi + q] & 0xffff, t = fst[z * nfi + q] >> 16;
        if (!(s >= 2 && t >= 2 && s + t <= N - 2)) ne[z].push_back(q);
      }
    if (ne[0].size() != ne[1].size() || ne[0].size() != ne[2].size())
      return set_err(c, HHG_ERR_STATE, "near-edge face rows differ between modes");
    std::vector<int> all;
    for (int z = 0; z < 3; ++z) all.insert(all.end(), ne[z].begin(), ne[z].end());
    lv.fne_len[col] = (int)ne[0].size();
    if ((st = up(lv.d_fne[col], all)) != HHG_OK) return st;
  }
  const size_t nv = (size_t)std::max<int64_t>(lv.n_frows, 1);
  HHG_CK(c, cudaMalloc(&lv.d_fval, 15 * nv * sizeof(double)));
  HHG_CK(c, cudaMalloc(&lv.d_fval_cons, 15 * nv * sizeof(double)));
  HHG_CK(c, cudaMalloc(&lv.d_ftmp, nv * sizeof(double)));
  return build_face_values(c, lv);
}

// Build lower-primitive rows of one level.
static hhg_status build_level(Ctx* c, Topology& tp, int L) {
  Level& lv = c->levels[L];
  const int N = 1 << L;
  lv.L = L;
  lv.N = N;
  lv.P = n_lattice(N);
  lv.S = (lv.P + 2 + 31) / 32 * 32;  // >= P+2: 16-byte-rounded bulk copies stay inside the block
  // column-march bands: consecutive diagonals with <= W interior columns
  auto make_bands = [&](int W, std::vector<Band>& out, int& slot_len) -> bool {
    out.clear();
    slot_len = 0;
    for (int d = 2; d <= N - 2;) {
      Band b{};
      b.d0 = d;
      int cnt = 0;
      while (d <= N - 2 && cnt + (d - 1) <= W) cnt += d - 1, ++d;
      if (cnt == 0) return false;
      b.d1 = d;
      b.ncolumns = cnt;
      b.c_lo = (int)col_idx(b.d0 - 1, 0);
      b.ncols = (int)col_idx(0, b.d1) + 1 - b.c_lo;  // through the end of diagonal d1
      b.kmax = N - 1 - b.d0;
      out.push_back(b);
      slot_len = std::max(slot_len, (b.ncols + 2 + 3) / 4 * 4);
    }
    return true;
  };
  if (!make_bands(kMarchThreads, lv.bands, lv.slot_len))
    return set_err(c, HHG_ERR_INVALID, "diagonal longer than a CTA");
  // wide bands (<= 2 kMarchThreads columns) of the single-pass GS (gsfront.cuh)
  if (!make_bands(2 * kMarchThreads, lv.bands_w, lv.slot_len_w))
    return set_err(c, HHG_ERR_INVALID, "diagonal longer than a CTA");
  // producer-warp GS bands (7 / 15 compute warps); empty if a diagonal does not fit
  for (int x = 0; x < 2; ++x)
    if (!make_bands(x ? 480 : 224, lv.bands_p[x], lv.slot_len_p[x])) lv.bands_p[x].clear();
  // element-wise FEM bands: <= kMarchThreads ANCHOR columns (every column of a
  // diagonal, d+1; the first band also anchors diagonal 1's 2 columns)
  lv.bands_fem.clear();
  for (int d = 2; d <= N - 2;) {
    Band b{};
    b.d0 = d;
    int cnt = d == 2 ? 2 : 0, ni = 0;
    while (d <= N - 2 && cnt + (d + 1) <= kMarchThreads) cnt += d + 1, ni += d - 1, ++d;
    if (d == b.d0) return set_err(c, HHG_ERR_INVALID, "diagonal longer than a CTA (fem bands)");
    b.d1 = d;
    b.ncolumns = ni;
    b.c_lo = (int)col_idx(b.d0 - 1, 0);
    b.ncols = (int)col_idx(0, b.d1) + 1 - b.c_lo;
    b.kmax = N - 1 - b.d0;
    lv.bands_fem.push_back(b);
  }
  lv.n_local = lv.S * c->nt_blocks;
  GidInfo& g = lv.gi;
  g.N = N;
  g.nv = c->nv;
  g.n_e = c->n_e;
  g.n_f = c->n_f;
  g.nfi = (int64_t)(N - 1) * (N - 2) / 2;
  g.nvi = n_interior(N);
  g.base_e = c->nv;
  g.base_f = g.base_e + c->n_e * (N - 1);
  g.base_v = g.base_f + c->n_f * g.nfi;
  g.n_total = g.base_v + c->nt * g.nvi;

  // ---- enumerate rows (owned unknown lower-primitive nodes) in GS step order
  std::vector<RowDesc> rows;
  std::vector<RowDesc> drows;  // Dirichlet lower nodes (all copies zeroed)
  int64_t steps[kNumLpSteps + 1];
  steps[0] = 0;
  // rows: owned by this rank (owner of the lowest-id macro containing the node);
  // Dirichlet nodes: every copy on this rank is zeroed
  for (int64_t v = 0; v < c->nv; ++v) {
    if (tp.vinc[v].empty()) continue;
    if (tp.vdir[v]) drows.push_back(RowDesc{0, 0, 0, v});
    else if (tp.vown[v] == c->rank) rows.push_back(RowDesc{0, 0, 0, v});
  }
  steps[1] = (int64_t)rows.size();
  for (int col = 0; col < 2; ++col) {
    for (int64_t e = 0; e < c->n_e; ++e) {
      if (tp.einc[e].empty()) continue;
      for (int m = 1; m <= N - 1; ++m) {
        if ((m % 2) != col) continue;
        if (tp.edir[e]) drows.push_back(RowDesc{1, m, 0, e});
        else if (tp.eown[e] == c->rank) rows.push_back(RowDesc{1, m, 0, e});
      }
    }
    steps[2 + col] = (int64_t)rows.size();
  }
  for (int col = 0; col < 3; ++col) {
    for (int64_t f = 0; f < c->n_f; ++f)
      if (!tp.finc[f].empty())
      for (int t = 1; t <= N - 2; ++t)
        for (int s = 1; s <= N - 1 - t; ++s) {
          if ((s + 2 * t) % 3 != col) continue;
          // non-Dirichlet face nodes are handled by the structured face rows below
          if (tp.fdir[f]) drows.push_back(RowDesc{2, s, t, f});
        }
    steps[4 + col] = (int64_t)rows.size();
  }
  for (int s = 0; s <= kNumLpSteps; ++s) lv.step_start[s] = steps[s];
  lv.n_rows = (int64_t)rows.size();
  {
    hhg_status stf = build_face_rows(c, tp, lv);
    if (stf != HHG_OK) return stf;
  }
  lv.n_owned = lv.n_rows + lv.n_frows + c->nt_local * g.nvi;

  const int64_t S = lv.S;
  auto is_dir = [&](int64_t gid) -> bool {
    if (gid < g.base_e) return tp.vdir[gid] != 0;
    if (gid < g.base_f) return tp.edir[(gid - g.base_e) / (N - 1)] != 0;
    if (gid < g.base_v) return tp.fdir[(gid - g.base_f) / g.nfi] != 0;
    return false;
  };
  // copies of a row: (local macro, ijk)
  auto copies_of = [&](const RowDesc& r, std::vector<std::array<int, 4>>& out) {
    out.clear();
    if (r.type == 0) {
      for (int32_t T : tp.vinc[r.id]) {
        int lvx = local_of(c->topo[T].gv, r.id);
        int w[4];
        corner(lvx, N, w);
        out.push_back(std::array<int, 4>{{(int)T, w[1], w[2], w[3]}});
      }
    } else if (r.type == 1) {
      int64_t a = tp.ekey[r.id] / c->nv, b = tp.ekey[r.id] % c->nv;
      for (int32_t T : tp.einc[r.id]) {
        int la = local_of(c->topo[T].gv, a), lb = local_of(c->topo[T].gv, b);
        int w[4] = {0, 0, 0, 0};
        w[la] = N - r.a;
        w[lb] = r.a;
        out.push_back(std::array<int, 4>{{(int)T, w[1], w[2], w[3]}});
      }
    } else {
      int64_t key = tp.fkey[r.id];
      int64_t cc = key % c->nv, ab = key / c->nv;
      int64_t a = ab / c->nv, b = ab % c->nv;
      for (int32_t T : tp.finc[r.id]) {
        int la = local_of(c->topo[T].gv, a), lb = local_of(c->topo[T].gv, b),
            lc = local_of(c->topo[T].gv, cc);
        int w[4] = {0, 0, 0, 0};
        w[la] = N - r.a - r.b;
        w[lb] = r.a;
        w[lc] = r.b;
        out.push_back(std::array<int, 4>{{(int)T, w[1], w[2], w[3]}});
      }
    }
    std::sort(out.begin(), out.end());
  };
  auto slot_of = [&](int T, int i, int j, int k) -> int64_t { return T * S + lattice_pos(N, i, j, k); };
  auto row_gid = [&](const RowDesc& r) -> int64_t {
    if (r.type == 0) return r.id;
    if (r.type == 1) return g.base_e + r.id * (N - 1) + (r.a - 1);
    int64_t s = r.a, t = r.b;
    return g.base_f + r.id * g.nfi + (t - 1) * (N - 1) - (t - 1) * t / 2 + (s - 1);
  };
  if ((uint64_t)lv.n_local >= (1ull << 32))
    return set_err(c, HHG_ERR_INVALID, "local vector exceeds 2^32 doubles at level " + std::to_string(L));

  // ---- pass 1: counts
  const int64_t nr = lv.n_rows;
  std::vector<uint64_t> rp(nr + 1, 0), cp(nr + 1, 0);
#pragma omp parallel
  {
    std::vector<std::array<int, 4>> cps;
    std::vector<int64_t> cols;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t r = 0; r < nr; ++r) {
      copies_of(rows[r], cps);
      cols.clear();
      cols.push_back(row_gid(rows[r]));
      for (auto& cpy : cps) {
        for (int w = 0; w < 15; ++w) {
          if (w == kMC) continue;
          int i = cpy[1] + kDirHost[w][0], j = cpy[2] + kDirHost[w][1], k = cpy[3] + kDirHost[w][2];
          if (i < 0 || j < 0 || k < 0 || i + j + k > N) continue;
          int64_t gj = node_gid(g, c->topo[cpy[0]], i, j, k);
          if (is_dir(gj)) continue;
          if (std::find(cols.begin(), cols.end(), gj) == cols.end()) cols.push_back(gj);
        }
      }
      rp[r + 1] = cols.size();
      cp[r + 1] = cps.size();
    }
  }
  for (int64_t r = 0; r < nr; ++r) {
    rp[r + 1] += rp[r];
    cp[r + 1] += cp[r];
  }
  lv.nnz = (int64_t)rp[nr];
  lv.n_copies = (int64_t)cp[nr];
  std::vector<uint32_t> col(lv.nnz), copy(lv.n_copies), cord(lv.n_copies);
  std::vector<int64_t> rgid(nr);
  std::vector<uint8_t> cmap(lv.n_copies * 16, 255);
  bool overflow = false;
  // The copies of a row are stored in local block order (the first is read as
  // the row's own value), but the row's columns are discovered -- and its
  // partial stencils summed (cord, k_lp_values) -- in the CANONICAL order of
  // the copies (global macro id, then i, j, k): the row's entries and their
  // rounding are then the same on every partition (bitwise-equal results on
  // any number of ranks).
#pragma omp parallel
  {
    std::vector<std::array<int, 4>> cps;
    std::vector<int64_t> cols;
    std::vector<int> perm;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t r = 0; r < nr; ++r) {
      copies_of(rows[r], cps);
      perm.resize(cps.size());
      for (size_t q = 0; q < cps.size(); ++q) perm[q] = (int)q;
      std::sort(perm.begin(), perm.end(), [&](int a, int b) {
        const int64_t ga = c->topo[cps[a][0]].gT, gb = c->topo[cps[b][0]].gT;
        if (ga != gb) return ga < gb;
        return cps[a] < cps[b];
      });
      cols.clear();
      rgid[r] = row_gid(rows[r]);
      cols.push_back(rgid[r]);
      uint64_t e0 = rp[r];
      col[e0] = (uint32_t)slot_of(cps[0][0], cps[0][1], cps[0][2], cps[0][3]);
      for (size_t q = 0; q < cps.size(); ++q) {
        auto& cpy = cps[q];
        copy[cp[r] + q] = (uint32_t)slot_of(cpy[0], cpy[1], cpy[2], cpy[3]);
        cord[cp[r] + q] = (uint32_t)(cp[r] + perm[q]);
      }
      for (size_t qq = 0; qq < cps.size(); ++qq) {
        const size_t q = (size_t)perm[qq];
        auto& cpy = cps[q];
        uint64_t ci = cp[r] + q;
        cmap[ci * 16 + kMC] = 0;
        for (int w = 0; w < 15; ++w) {
          if (w == kMC) continue;
          int i = cpy[1] + kDirHost[w][0], j = cpy[2] + kDirHost[w][1], k = cpy[3] + kDirHost[w][2];
          if (i < 0 || j < 0 || k < 0 || i + j + k > N) continue;
          int64_t gj = node_gid(g, c->topo[cpy[0]], i, j, k);
          if (is_dir(gj)) continue;
          auto it = std::find(cols.begin(), cols.end(), gj);
          size_t pos = it - cols.begin();
          if (it == cols.end()) {
            cols.push_back(gj);
            col[e0 + pos] = (uint32_t)slot_of(cpy[0], i, j, k);
          }
          if (pos > 250) overflow = true;
          cmap[ci * 16 + w] = (uint8_t)pos;
        }
      }
    }
  }
  if (overflow) return set_err(c, HHG_ERR_MESH, "lower-primitive row with more than 250 neighbours");

  // ---- Dirichlet slots
  std::vector<uint32_t> dslot;
  std::vector<int64_t> dgid;
  {
    std::vector<std::array<int, 4>> cps;
    for (auto& r : drows) {
      copies_of(r, cps);
      int64_t gg = row_gid(r);
      for (auto& cpy : cps) {
        dslot.push_back((uint32_t)slot_of(cpy[0], cpy[1], cpy[2], cpy[3]));
        dgid.push_back(gg);
      }
    }
  }
  lv.n_dir = (int64_t)dslot.size();

  // ---- exchange plan (multi-rank): which slots of this rank mirror values
  // owned elsewhere ((a) ghost-block slots read by the owned rows, (b) the
  // local copies of lower-primitive nodes owned by another rank), and which
  // owned values this rank serves.
  if (c->nranks > 1) {
    auto value_rank = [&](int64_t T, int i, int j, int k, int64_t& gid) -> int {
      gid = node_gid(g, c->topo[T], i, j, k);
      if (gid >= g.base_v) return c->owner[c->topo[T].gT];
      if (gid < g.base_e) return tp.vown[gid];
      if (gid < g.base_f) return tp.eown[(gid - g.base_e) / (N - 1)];
      return tp.fown[(gid - g.base_f) / g.nfi];
    };
    std::vector<std::pair<uint32_t, int64_t>> cand;  // (slot, gid)
    std::vector<int32_t> cand_rank;
    auto consider = [&](int64_t T, int i, int j, int k) {
      int64_t gid;
      const int r = value_rank(T, i, j, k, gid);
      if (r == c->rank || is_dir(gid)) return;
      cand.push_back({(uint32_t)slot_of((int)T, i, j, k), gid});
      cand_rank.push_back(r);
    };
    // (a) CSR columns in ghost blocks
    for (int64_t e = 0; e < lv.nnz; ++e) {
      const int64_t T = col[e] / S;
      if (T < c->nt_local) continue;
      int i, j, k;
      decode_pos(N, col[e] - T * S, i, j, k);
      consider(T, i, j, k);
    }
    // (a) face rows: the 4 into-B neighbours when B is a ghost
    for (const FaceLP& F : lv.h_flp) {
      if (F.TB < c->nt_local) continue;
      for (int64_t q = 0; q < g.nfi; ++q) {
        const int s = lv.h_fst[F.z * g.nfi + q] & 0xffff, t = lv.h_fst[F.z * g.nfi + q] >> 16;
        int w[4] = {0, 0, 0, 0};
        w[F.lB[0]] = N - s - t;
        w[F.lB[1]] = s;
        w[F.lB[2]] = t;
        for (int e = 10; e < 14; ++e) consider(F.TB, w[1] + F.off[e][0], w[2] + F.off[e][1], w[3] + F.off[e][2]);
      }
    }
    // (b) local copies of lower-primitive nodes owned elsewhere
    {
      std::vector<std::array<int, 4>> cps;
      auto add_local = [&](const RowDesc& r) {
        copies_of(r, cps);
        for (auto& cpy : cps)
          if (cpy[0] < c->nt_local) consider(cpy[0], cpy[1], cpy[2], cpy[3]);
      };
      for (int64_t v = 0; v < c->nv; ++v)
        if (!tp.vinc[v].empty() && !tp.vdir[v] && tp.vown[v] != c->rank) add_local(RowDesc{0, 0, 0, v});
      for (int64_t e = 0; e < c->n_e; ++e)
        if (!tp.einc[e].empty() && !tp.edir[e] && tp.eown[e] != c->rank)
          for (int m = 1; m <= N - 1; ++m) add_local(RowDesc{1, m, 0, e});
      for (int64_t f = 0; f < c->n_f; ++f)
        if (!tp.finc[f].empty() && !tp.fdir[f] && tp.fown[f] != c->rank)
          for (int t = 1; t <= N - 2; ++t)
            for (int s = 1; s <= N - 1 - t; ++s) add_local(RowDesc{2, s, t, f});
    }
    // dedupe by slot
    std::vector<size_t> ord(cand.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return cand[a].first < cand[b].first; });
    std::vector<uint32_t> r_slot;
    std::vector<int64_t> r_gid;
    std::vector<int32_t> r_rank;
    for (size_t x = 0; x < ord.size(); ++x) {
      if (x > 0 && cand[ord[x]].first == cand[ord[x - 1]].first) continue;
      r_slot.push_back(cand[ord[x]].first);
      r_gid.push_back(cand[ord[x]].second);
      r_rank.push_back(cand_rank[ord[x]]);
    }
    // values served by this rank: owned LP rows (first copy = owner macro, local)
    std::vector<std::pair<int64_t, uint32_t>> serve;
    for (int64_t r = 0; r < nr; ++r) serve.push_back({rgid[r], copy[cp[r]]});
    for (size_t fi = 0; fi < lv.h_flp.size(); ++fi) {
      const FaceLP& F = lv.h_flp[fi];
      for (int64_t q = 0; q < g.nfi; ++q) {
        const int s = lv.h_fst[F.z * g.nfi + q] & 0xffff, t = lv.h_fst[F.z * g.nfi + q] >> 16;
        int w[4] = {0, 0, 0, 0};
        w[F.lA[0]] = N - s - t;
        w[F.lA[1]] = s;
        w[F.lA[2]] = t;
        serve.push_back({g.base_f + F.fid * g.nfi + lv.h_fcidx[F.z * g.nfi + q],
                         (uint32_t)slot_of(F.TA, w[1], w[2], w[3])});
      }
    }
    std::sort(serve.begin(), serve.end());
    hhg_status sp = dist_build_plan(c, lv, r_slot, r_gid, r_rank, serve);
    if (sp != HHG_OK) return sp;
  }
  if (c->host_only) return HHG_OK;

  // ---- upload
  auto up = [&](auto*& dptr, const auto& vec) -> hhg_status {
    using T = typename std::remove_reference<decltype(vec)>::type::value_type;
    size_t bytes = std::max<size_t>(vec.size(), 1) * sizeof(T);
    HHG_CK(c, cudaMalloc((void**)&dptr, bytes));
    if (!vec.empty())
      HHG_CK(c, cudaMemcpy(dptr, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice));
    return HHG_OK;
  };
  hhg_status st;
  if ((st = up(lv.d_row_ptr, rp)) != HHG_OK) return st;
  if ((st = up(lv.d_col, col)) != HHG_OK) return st;
  if ((st = up(lv.d_copy_ptr, cp)) != HHG_OK) return st;
  if ((st = up(lv.d_copy, copy)) != HHG_OK) return st;
  if ((st = up(lv.d_row_gid, rgid)) != HHG_OK) return st;
  if ((st = up(lv.d_dir_slot, dslot)) != HHG_OK) return st;
  if ((st = up(lv.d_dir_gid, dgid)) != HHG_OK) return st;
  if ((st = up(lv.d_bands, lv.bands)) != HHG_OK) return st;
  if ((st = up(lv.d_bands_w, lv.bands_w)) != HHG_OK) return st;
  for (int x = 0; x < 2; ++x)
    if (!lv.bands_p[x].empty() && (st = up(lv.d_bands_p[x], lv.bands_p[x])) != HHG_OK) return st;
  if ((st = up(lv.d_bands_fem, lv.bands_fem)) != HHG_OK) return st;
  {
    const size_t nfl = (size_t)c->nt_local * std::max<size_t>(lv.bands.size(), 1) * 4;
    HHG_CK(c, cudaMalloc(&lv.d_gs_flags, nfl * sizeof(int)));
    HHG_CK(c, cudaMemset(lv.d_gs_flags, 0, nfl * sizeof(int)));
    HHG_CK(c, cudaMalloc(&lv.d_gs_counter, sizeof(int)));
  }
  HHG_CK(c, cudaMalloc(&lv.d_val, std::max<int64_t>(lv.nnz, 1) * sizeof(double)));
  HHG_CK(c, cudaMalloc(&lv.d_val_cons, std::max<int64_t>(lv.nnz, 1) * sizeof(double)));
  HHG_CK(c, cudaMalloc(&lv.d_tmp, std::max<int64_t>(nr, 1) * sizeof(double)));
  HHG_CK(c, cudaMalloc(&lv.d_cons, c->nt_local * 15 * sizeof(double)));
  if ((st = build_lp_values(c, lv, cmap, cord)) != HHG_OK) return st;
  // constant (affine) stencil per macro: interior node (1,1,1)
  {
    std::vector<uint32_t> sl(c->nt_local);
    for (int64_t T = 0; T < c->nt_local; ++T) sl[T] = (uint32_t)slot_of((int)T, 1, 1, 1);
    uint32_t* d_sl = nullptr;
    if ((st = up(d_sl, sl)) != HHG_OK) return st;
    if ((st = launch_fem_partial(c, L, d_sl, c->nt_local, false, lv.d_cons)) != HHG_OK) return st;
    HHG_CK(c, cudaStreamSynchronize(c->stream));
    cudaFree(d_sl);
  }
  return HHG_OK;
}

static void free_level(Level& lv) {
  void* ps[] = {lv.d_row_ptr, lv.d_col, lv.d_val, lv.d_val_cons, lv.d_copy_ptr, lv.d_copy,
                lv.d_row_gid, lv.d_dir_slot, lv.d_dir_gid, lv.d_tmp, lv.d_coef, lv.d_cons,
                lv.d_coef10, lv.d_bands, lv.d_gs_flags, lv.d_gs_counter,
                lv.d_flp, lv.d_fst, lv.d_fcidx, lv.d_fval, lv.d_fval_cons, lv.d_ftmp, lv.d_po,
                lv.d_send_slot, lv.d_recv_slot, lv.d_sendbuf, lv.d_recvbuf, lv.d_cC, lv.d_rsum_ptr, lv.d_rsum_slot, lv.d_rsum_idx, lv.d_ew_lo, lv.d_ew_hi, lv.d_bands_fem, lv.d_fcoef, lv.d_cg_rp, lv.d_cg_col, lv.d_cg_val, lv.d_cg_vec, lv.d_cg_part, lv.d_cg_red, lv.d_fne[0], lv.d_fne[1], lv.d_fne[2], lv.d_gs_ex, lv.d_gs_prog, lv.d_gs_epoch, lv.d_bands_w, lv.d_bands_p[0], lv.d_bands_p[1]};
  for (void* p : ps)
    if (p) cudaFree(p);
  lv = Level();
}

}  // namespace hhg

using namespace hhg;

extern "C" hhg_status hhg_setup_macro_mesh(const double* vertices, const double* vertex_radius,
                                           int64_t nv, const int64_t* tets, int64_t nt,
                                           const uint8_t* dirichlet_face, int L_max,
                                           const int32_t* macro_owner, int rank, int nranks,
                                           const void* nccl_unique_id, void* cuda_stream,
                                           hhg_ctx* out) {
  if (!out) return HHG_ERR_INVALID;
  *out = nullptr;
  if (!vertices || !tets || !dirichlet_face || nv < 4 || nt < 1 || L_max < 2 || L_max > 8)
    return HHG_ERR_INVALID;
  if (nranks < 1 || rank < 0 || rank >= nranks) return HHG_ERR_INVALID;
  if (macro_owner)
    for (int64_t t = 0; t < nt; ++t)
      if (macro_owner[t] < 0 || macro_owner[t] >= nranks) return HHG_ERR_INVALID;
  Ctx* c = new Ctx();
  c->stream = (cudaStream_t)cuda_stream;
  c->rank = rank;
  c->nranks = nranks;
  c->owner.resize(nt);
  for (int64_t t = 0; t < nt; ++t)
    c->owner[t] = macro_owner ? macro_owner[t] : (int32_t)((t * nranks) / nt);
  if (nranks > 1) {
    hhg_status ts = dist_init_transport(c, nccl_unique_id);
    if (ts != HHG_OK) {
      fprintf(stderr, "hhg_setup_macro_mesh: transport: %s\n", c->err.c_str());
      delete c;
      return ts;
    }
  }
  c->L_max = L_max;
  c->nv = nv;
  c->nt = nt;
  c->blended = vertex_radius != nullptr;
  c->vertices.assign(vertices, vertices + 3 * nv);
  if (vertex_radius) c->radius.assign(vertex_radius, vertex_radius + nv);
  c->tets.assign(tets, tets + 4 * nt);
  c->dirichlet.assign(dirichlet_face, dirichlet_face + 4 * nt);
  auto fail = [&](hhg_status s, const std::string& m) {
    // keep the ctx so hhg_last_error works? ABI: out = NULL on failure.
    fprintf(stderr, "hhg_setup_macro_mesh: %s\n", m.c_str());
    delete c;
    return s;
  };
  // ---- validation
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t* tv = &tets[4 * t];
    for (int a = 0; a < 4; ++a) {
      if (tv[a] < 0 || tv[a] >= nv) return fail(HHG_ERR_MESH, "vertex id out of range");
      for (int b = a + 1; b < 4; ++b)
        if (tv[a] == tv[b]) return fail(HHG_ERR_MESH, "repeated vertex in tet");
    }
    double e[3][3], scale = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int d = 0; d < 3; ++d) {
        e[a][d] = vertices[3 * tv[a + 1] + d] - vertices[3 * tv[0] + d];
        scale = std::max(scale, std::fabs(e[a][d]));
      }
    double det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                 e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                 e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
    if (!(std::fabs(det) > 1e-12 * scale * scale * scale))
      return fail(HHG_ERR_MESH, "degenerate tet " + std::to_string(t));
  }
  if (vertex_radius) {
    for (int64_t v = 0; v < nv; ++v) {
      double n = std::sqrt(vertices[3 * v] * vertices[3 * v] + vertices[3 * v + 1] * vertices[3 * v + 1] +
                           vertices[3 * v + 2] * vertices[3 * v + 2]);
      if (!(vertex_radius[v] > 0) || std::fabs(n - vertex_radius[v]) > 1e-12 * vertex_radius[v])
        return fail(HHG_ERR_MESH, "|x_v| != r_v at vertex " + std::to_string(v));
    }
  }
  // ---- topology
  Topology tp;
  std::vector<int64_t> ek, fk;
  ek.reserve(6 * nt);
  fk.reserve(4 * nt);
  for (int64_t t = 0; t < nt; ++t) {
    int64_t s[4];
    for (int a = 0; a < 4; ++a) s[a] = tets[4 * t + a];
    std::sort(s, s + 4);
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) ek.push_back(s[a] * nv + s[b]);
    for (int f = 0; f < 4; ++f) {
      int64_t q[3];
      int n = 0;
      for (int a = 0; a < 4; ++a)
        if (a != f) q[n++] = s[a];
      fk.push_back((q[0] * nv + q[1]) * nv + q[2]);
    }
  }
  std::sort(ek.begin(), ek.end());
  ek.erase(std::unique(ek.begin(), ek.end()), ek.end());
  std::sort(fk.begin(), fk.end());
  fk.erase(std::unique(fk.begin(), fk.end()), fk.end());
  tp.ekey = ek;
  tp.fkey = fk;
  c->n_e = (int64_t)ek.size();
  c->n_f = (int64_t)fk.size();
  // topology of every global macro
  std::vector<MacroTopo> gtopo(nt);
  std::vector<int> fcount(c->n_f, 0);
  for (int64_t t = 0; t < nt; ++t) {
    MacroTopo& m = gtopo[t];
    m.gT = t;
    for (int a = 0; a < 4; ++a) m.gv[a] = tets[4 * t + a];
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) {
        int64_t x = std::min(m.gv[a], m.gv[b]), y = std::max(m.gv[a], m.gv[b]);
        m.e[local_edge(a, b)] = std::lower_bound(ek.begin(), ek.end(), x * nv + y) - ek.begin();
      }
    for (int f = 0; f < 4; ++f) {
      int64_t q[3];
      int n = 0;
      for (int a = 0; a < 4; ++a)
        if (a != f) q[n++] = m.gv[a];
      std::sort(q, q + 3);
      m.f[f] = std::lower_bound(fk.begin(), fk.end(), (q[0] * nv + q[1]) * nv + q[2]) - fk.begin();
      fcount[m.f[f]]++;
    }
  }
  for (int64_t f = 0; f < c->n_f; ++f)
    if (fcount[f] > 2) return fail(HHG_ERR_MESH, "face shared by more than two tets");
  // owner rank of every primitive = rank of the lowest-id macro containing it
  tp.vown.assign(nv, -1);
  tp.eown.assign(c->n_e, -1);
  tp.fown.assign(c->n_f, -1);
  for (int64_t t = nt - 1; t >= 0; --t) {
    const MacroTopo& m = gtopo[t];
    for (int a = 0; a < 4; ++a) tp.vown[m.gv[a]] = c->owner[t];
    for (int e = 0; e < 6; ++e) tp.eown[m.e[e]] = c->owner[t];
    for (int f = 0; f < 4; ++f) tp.fown[m.f[f]] = c->owner[t];
  }
  // blocks: local macros, then ghosts (other ranks' macros sharing a vertex with a local one)
  std::vector<char> vlocal(nv, 0), isblk(nt, 0);
  for (int64_t t = 0; t < nt; ++t)
    if (c->owner[t] == rank)
      for (int a = 0; a < 4; ++a) vlocal[gtopo[t].gv[a]] = 1;
  // local macros: BOUNDARY ones first (a vertex shared with another rank's
  // macro: their values are exchanged), then the interior ones, each in
  // ascending global id -- the exchange can then overlap the interior range
  // (dist_sync_overlapped)
  std::vector<char> vforeign(nv, 0);
  for (int64_t t = 0; t < nt; ++t)
    if (c->owner[t] != rank)
      for (int a = 0; a < 4; ++a) vforeign[gtopo[t].gv[a]] = 1;
  c->local_macros.clear();
  for (int pass = 0; pass < 2; ++pass)
    for (int64_t t = 0; t < nt; ++t) {
      if (c->owner[t] != rank) continue;
      bool b = false;
      for (int a = 0; a < 4; ++a) b = b || vforeign[gtopo[t].gv[a]];
      if (b == (pass == 0)) c->local_macros.push_back(t);
      if (pass == 0 && b) ++c->nt_bnd;
    }
  c->nt_local = (int64_t)c->local_macros.size();
  for (int64_t t = 0; t < nt; ++t) {
    if (c->owner[t] == rank) continue;
    bool g = false;
    for (int a = 0; a < 4; ++a) g = g || vlocal[gtopo[t].gv[a]];
    if (g) c->local_macros.push_back(t);
  }
  c->nt_blocks = (int64_t)c->local_macros.size();
  if (c->nt_local == 0) return fail(HHG_ERR_INVALID, "rank owns no macro");
  c->g2b.assign(nt, -1);
  for (int64_t T = 0; T < c->nt_blocks; ++T) c->g2b[c->local_macros[T]] = T;
  c->topo.resize(c->nt_blocks);
  for (int64_t T = 0; T < c->nt_blocks; ++T) c->topo[T] = gtopo[c->local_macros[T]];
  // block incidence, ascending GLOBAL macro id (canonical summation order)
  tp.vinc.assign(nv, {});
  tp.einc.assign(c->n_e, {});
  tp.finc.assign(c->n_f, {});
  tp.vdir.assign(nv, 0);
  tp.edir.assign(c->n_e, 0);
  tp.fdir.assign(c->n_f, 0);
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t T = c->g2b[t];
    if (T < 0) continue;
    const MacroTopo& m = c->topo[T];
    for (int a = 0; a < 4; ++a) tp.vinc[m.gv[a]].push_back((int32_t)T);
    for (int e = 0; e < 6; ++e) tp.einc[m.e[e]].push_back((int32_t)T);
    for (int f = 0; f < 4; ++f) tp.finc[m.f[f]].push_back((int32_t)T);
  }
  // primitive ownership (lowest local macro id) for the restriction R = P^T
  c->own.assign(c->nt_local, 0);
  for (int64_t T = 0; T < c->nt_local; ++T) {
    const MacroTopo& m = c->topo[T];
    uint16_t o = 0;
    for (int f = 0; f < 4; ++f)
      if (tp.finc[m.f[f]][0] == T) o |= (uint16_t)(1u << f);
    for (int e = 0; e < 6; ++e)
      if (tp.einc[m.e[e]][0] == T) o |= (uint16_t)(1u << (4 + e));
    for (int v = 0; v < 4; ++v)
      if (tp.vinc[m.gv[v]][0] == T) o |= (uint16_t)(1u << (10 + v));
    c->own[T] = o;
  }
  // Dirichlet closure (tags of every global macro)
  for (int64_t t = 0; t < nt; ++t) {
    const MacroTopo& m = gtopo[t];
    for (int f = 0; f < 4; ++f) {
      if (!dirichlet_face[4 * m.gT + f]) continue;
      tp.fdir[m.f[f]] = 1;
      for (int a = 0; a < 4; ++a) {
        if (a == f) continue;
        tp.vdir[m.gv[a]] = 1;
        for (int b = a + 1; b < 4; ++b)
          if (b != f) tp.edir[m.e[local_edge(a, b)]] = 1;
      }
    }
  }
  // ---- device geometry (every block: ghost geometry feeds the face rows)
  std::vector<double> geo(c->nt_blocks * 16);
  for (int64_t T = 0; T < c->nt_blocks; ++T)
    for (int a = 0; a < 4; ++a) {
      int64_t v = c->topo[T].gv[a];
      for (int d = 0; d < 3; ++d) geo[T * 16 + 4 * a + d] = vertices[3 * v + d];
      geo[T * 16 + 4 * a + 3] = vertex_radius ? vertex_radius[v] : 0.0;
    }
  if (!c->host_only) {
    cudaError_t e1 = cudaMalloc(&c->d_geo, geo.size() * sizeof(double));
    if (e1 != cudaSuccess) return fail(HHG_ERR_CUDA, cudaGetErrorString(e1));
    cudaMemcpy(c->d_geo, geo.data(), geo.size() * sizeof(double), cudaMemcpyHostToDevice);
    cudaMalloc(&c->d_topo, c->topo.size() * sizeof(MacroTopo));
    cudaMemcpy(c->d_topo, c->topo.data(), c->topo.size() * sizeof(MacroTopo), cudaMemcpyHostToDevice);
  }
  c->levels.resize(L_max + 1);
  for (int L = 2; L <= L_max; ++L) {
    hhg_status st = build_level(c, tp, L);
    if (st != HHG_OK) {
      std::string m = c->err;
      hhg_destroy((hhg_ctx)c);
      fprintf(stderr, "hhg_setup_macro_mesh: level %d: %s\n", L, m.c_str());
      return st;
    }
  }
  *out = (hhg_ctx)c;
  return HHG_OK;
}

extern "C" hhg_status hhg_vector_layout(hhg_ctx ctx, int L, int64_t* n_local, int64_t* n_owned,
                                        int64_t* n_global) {
  Ctx* c = (Ctx*)ctx;
  if (!c || L < 2 || L > c->L_max) return HHG_ERR_INVALID;
  const Level& lv = c->levels[L];
  if (n_local) *n_local = lv.n_local;
  if (n_owned) *n_owned = lv.n_owned;
  if (n_global) *n_global = lv.gi.n_total;
  return HHG_OK;
}

extern "C" const char* hhg_last_error(hhg_ctx ctx) {
  Ctx* c = (Ctx*)ctx;
  return c ? c->err.c_str() : "null ctx";
}

extern "C" int64_t hhg_kernel_launches(hhg_ctx ctx) {
  Ctx* c = (Ctx*)ctx;
  return c ? c->launches : -1;
}

extern "C" void hhg_destroy(hhg_ctx ctx) {
  Ctx* c = (Ctx*)ctx;
  if (!c) return;
  if (c->host_only) {
    delete c;
    return;
  }
  cudaStreamSynchronize(c->stream);
  dist_destroy(c);
  for (auto& lv : c->levels) free_level(lv);
  if (c->d_geo) cudaFree(c->d_geo);
  if (c->d_topo) cudaFree(c->d_topo);
  for (auto* p : c->d_stage)
    if (p) cudaFree(p);
  if (c->d_red) cudaFree(c->d_red);
  if (c->h_red) cudaFreeHost(c->h_red);
  for (auto* v : {&c->vc_u, &c->vc_f, &c->vc_r})
    for (double* p : *v)
      if (p) cudaFree(p);
  if (c->d_cg) cudaFree(c->d_cg);
  if (c->d_scal) cudaFree(c->d_scal);
  if (c->d_flag) cudaFree(c->d_flag);
  if (c->d_own) cudaFree(c->d_own);
  if (c->vc_graph) cudaGraphExecDestroy(c->vc_graph);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (auto& v : c->ev_rec)
    for (auto& p : v) {
      cudaEventDestroy(p.first);
      cudaEventDestroy(p.second);
    }
  delete c;
}
