"""Oracle geometry: macro lattice, blending, fine tetrahedra, canonical numbering.

Follows PAPER.md:195-262 (Psi_T, Phi_T, mesh families T and T~),
PAPER.md:295-338 (HHG primitives, Bey refinement, n_l)
(15-point stencil, index set I_l).

Level convention (R5): BASELINE level L has N = 2**L intervals per
macro edge; the paper's level is l = L - 2 (h_l = 2^-(l+2) H).
"""
from __future__ import annotations

import itertools

import numpy as np

# ---------------------------------------------------------------------------
# 15 stencil directions (offsets = DESIGN.md reading R7).
# Order: opposite of index x is index 14 - x; mc is index 7.
# b/m/t = k-1/k/k+1; in-plane compass with i = west->east, j = south->north.
# ---------------------------------------------------------------------------
DIR_NAMES = ["bc", "be", "bn", "bnw", "ms", "mse", "mw", "mc",
             "me", "mnw", "mn", "tse", "ts", "tw", "tc"]
DIRS = np.array([
    (0, 0, -1), (1, 0, -1), (0, 1, -1), (-1, 1, -1),
    (0, -1, 0), (1, -1, 0), (-1, 0, 0), (0, 0, 0),
    (1, 0, 0), (-1, 1, 0), (0, 1, 0),
    (1, -1, 1), (0, -1, 1), (-1, 0, 1), (0, 0, 1),
], dtype=np.int64)
MC = 7


def opposite(w: int) -> int:
    return 14 - w


def n_interior(N: int) -> int:
    """Number of volume-primitive (interior) nodes, eq. numInteriorPoints
     with N = 2^(l+2): (N-3)(N-2)(N-1)/6."""
    return (N - 3) * (N - 2) * (N - 1) // 6


def n_lattice(N: int) -> int:
    return (N + 1) * (N + 2) * (N + 3) // 6


def lattice_ijk(N: int) -> np.ndarray:
    """All lattice nodes (i,j,k), 0<=i,j,k, i+j+k<=N, order k, j, i (i fastest)."""
    out = []
    for k in range(N + 1):
        for j in range(N + 1 - k):
            for i in range(N + 1 - k - j):
                out.append((i, j, k))
    return np.array(out, dtype=np.int64)


def interior_ijk(N: int) -> np.ndarray:
    """Index set I_l (R6): i,j,k >= 1, i+j+k <= N-1,
    lexicographic order k outer, j, i inner (the smoother traversal,
    PAPER.md:1317-1321)."""
    out = []
    for k in range(1, N):
        for j in range(1, N - k):
            for i in range(1, N - k - j):
                out.append((i, j, k))
    return np.array(out, dtype=np.int64).reshape(-1, 3)


# ---------------------------------------------------------------------------
# Fine tetrahedra of the uniformly refined macro (Bey refinement, PAPER.md:
# 205-207, 297-301).  In coordinates x=i+j+k, y=j+k, z=k the refinement is the
# Kuhn/Freudenthal triangulation restricted to N >= x >= y >= z >= 0
# (R4; pinned against a literal recursive Bey refinement in
# tests/test_oracle_geometry.py).
# ---------------------------------------------------------------------------
_E = np.eye(3, dtype=np.int64)
PERMS = list(itertools.permutations(range(3)))


def _to_ijk(xyz):
    x, y, z = xyz[..., 0], xyz[..., 1], xyz[..., 2]
    return np.stack([x - y, y - z, z], axis=-1)


def _in_region(xyz, N):
    x, y, z = xyz[..., 0], xyz[..., 1], xyz[..., 2]
    return (x <= N) & (x >= y) & (y >= z) & (z >= 0)


def kuhn_tets(N: int) -> np.ndarray:
    """All N^3 fine tets of the macro lattice as [N^3, 4, 3] (i,j,k) triples."""
    pts = []
    for x in range(N):
        for y in range(x + 1):
            for z in range(y + 1):
                pts.append((x, y, z))
    p = np.array(pts, dtype=np.int64)
    out = []
    for s in PERMS:
        v0 = p
        v1 = v0 + _E[s[0]]
        v2 = v1 + _E[s[1]]
        v3 = v0 + 1
        tet = np.stack([v0, v1, v2, v3], axis=1)
        ok = np.all(_in_region(tet, N), axis=1)
        out.append(tet[ok])
    tets = np.concatenate(out, axis=0)
    return _to_ijk(tets)


def incident_kuhn_tets(ijk: np.ndarray, N: int, inside_only=True):
    """The Kuhn tets containing node `ijk` [3] -> list of [4,3] arrays
    (24 for an interior node)."""
    i, j, k = (int(v) for v in ijk)
    node = np.array([i + j + k, j + k, k], dtype=np.int64)
    out = []
    for s in PERMS:
        path = [np.zeros(3, np.int64), _E[s[0]], _E[s[0]] + _E[s[1]], np.ones(3, np.int64)]
        for m in range(4):
            p = node - path[m]
            tet = np.stack([p + q for q in path])
            if inside_only and not np.all(_in_region(tet, N)):
                continue
            out.append(_to_ijk(tet))
    return out


# ---------------------------------------------------------------------------
# Coordinates: affine map Psi_T and radial blending Phi_T (
# DESIGN.md R4: x -> x * (sum_v lambda_v r_v) / |x|).
# ---------------------------------------------------------------------------
def barycentric(ijk: np.ndarray, N: int) -> np.ndarray:
    ijk = np.asarray(ijk, dtype=np.float64)
    i, j, k = ijk[..., 0], ijk[..., 1], ijk[..., 2]
    return np.stack([(N - i - j - k) / N, i / N, j / N, k / N], axis=-1)


def node_coords(mesh, T: int, ijk: np.ndarray, N: int, blended: bool = True) -> np.ndarray:
    """Physical coordinates of lattice nodes of macro T.  Affine:
    X = sum_v lambda_v X_v (Psi_T).  Blended: Phi_T(X) = X * r(X) / |X| with
    r = sum_v lambda_v r_v (spherical layers)."""
    lam = barycentric(ijk, N)
    Xv = mesh.vertices[mesh.tets[T]]           # [4,3]
    X = lam @ Xv
    if not blended or mesh.radius is None:
        return X
    r = lam @ mesh.radius[mesh.tets[T]]
    return X * (r / np.linalg.norm(X, axis=-1))[..., None]


# ---------------------------------------------------------------------------
# Canonical numbering: the convention
# shared (by documentation, not code) with the C-ABI's gather/scatter.
#   [vertices nv][edges n_e*(N-1)][faces n_f*(N-1)(N-2)/2][volumes nt*n_int]
# ---------------------------------------------------------------------------
class Numbering:
    """Global node ids, classes, Dirichlet mask and GS colours at level N."""

    VERTEX, EDGE, FACE, VOLUME = 0, 1, 2, 3

    def __init__(self, mesh, N: int):
        self.mesh = mesh
        self.N = N
        tets = mesh.tets
        nv, nt = mesh.nv, mesh.nt
        edges = set()
        faces = set()
        for t in tets:
            for a, b in itertools.combinations(sorted(int(x) for x in t), 2):
                edges.add((a, b))
            for f in itertools.combinations(sorted(int(x) for x in t), 3):
                faces.add(f)
        self.edges = np.array(sorted(edges), dtype=np.int64).reshape(-1, 2)
        self.faces = np.array(sorted(faces), dtype=np.int64).reshape(-1, 3)
        self._ekey = self.edges[:, 0] * nv + self.edges[:, 1]
        self._fkey = (self.faces[:, 0] * nv + self.faces[:, 1]) * nv + self.faces[:, 2]
        self.n_e = len(self.edges)
        self.n_f = len(self.faces)
        self.nfi = (N - 1) * (N - 2) // 2
        self.nvi = n_interior(N)
        self.base_e = nv
        self.base_f = nv + self.n_e * (N - 1)
        self.base_v = self.base_f + self.n_f * self.nfi
        self.n_total = self.base_v + nt * self.nvi
        # interior index lookup (k outer, j, i inner)
        inter = interior_ijk(N)
        self._vidx = -np.ones((N + 1, N + 1, N + 1), dtype=np.int64)
        self._vidx[inter[:, 0], inter[:, 1], inter[:, 2]] = np.arange(len(inter))
        # Dirichlet: closure of tagged faces
        dface = set()
        for T in range(nt):
            for f in range(4):
                if mesh.dirichlet[T, f]:
                    dface.add(tuple(sorted(int(tets[T, v]) for v in range(4) if v != f)))
        self.dirichlet_faces = dface
        dverts = set(v for f in dface for v in f)
        dedges = set(e for f in dface for e in itertools.combinations(f, 2))
        self.dirichlet_mask = np.zeros(self.n_total, dtype=bool)
        for v in dverts:
            self.dirichlet_mask[v] = True
        for e in dedges:
            eid = self.edge_id(*e)
            self.dirichlet_mask[self.base_e + eid * (N - 1): self.base_e + (eid + 1) * (N - 1)] = True
        for f in dface:
            fid = self.face_id(*f)
            self.dirichlet_mask[self.base_f + fid * self.nfi: self.base_f + (fid + 1) * self.nfi] = True
        self.unknown_mask = ~self.dirichlet_mask

    def edge_id(self, a, b):
        a, b = min(a, b), max(a, b)
        i = np.searchsorted(self._ekey, a * self.mesh.nv + b)
        assert self._ekey[i] == a * self.mesh.nv + b
        return int(i)

    def face_id(self, a, b, c):
        a, b, c = sorted((a, b, c))
        key = (a * self.mesh.nv + b) * self.mesh.nv + c
        i = np.searchsorted(self._fkey, key)
        assert self._fkey[i] == key
        return int(i)

    def gids(self, T: int, ijk: np.ndarray) -> np.ndarray:
        """Canonical global id of lattice nodes `ijk` [n,3] of macro T."""
        N = self.N
        nv = self.mesh.nv
        ijk = np.asarray(ijk, dtype=np.int64).reshape(-1, 3)
        w = np.stack([N - ijk.sum(1), ijk[:, 0], ijk[:, 1], ijk[:, 2]], axis=1)  # [n,4]
        gv = self.mesh.tets[T]
        pos = w > 0
        cnt = pos.sum(1)
        out = np.empty(len(ijk), dtype=np.int64)
        # vertices
        m1 = cnt == 1
        out[m1] = gv[np.argmax(w[m1], axis=1)]
        # edges / faces: sort support by global vertex id
        gvb = np.where(pos, gv[None, :], np.iinfo(np.int64).max)
        order = np.argsort(gvb, axis=1, kind="stable")
        gs = np.take_along_axis(gvb, order, axis=1)
        ws = np.take_along_axis(w, order, axis=1)
        m2 = cnt == 2
        if m2.any():
            a, b, mb = gs[m2, 0], gs[m2, 1], ws[m2, 1]
            eid = np.searchsorted(self._ekey, a * nv + b)
            out[m2] = self.base_e + eid * (N - 1) + (mb - 1)
        m3 = cnt == 3
        if m3.any():
            a, b, c = gs[m3, 0], gs[m3, 1], gs[m3, 2]
            s, t = ws[m3, 1], ws[m3, 2]
            fid = np.searchsorted(self._fkey, (a * nv + b) * nv + c)
            idx = (t - 1) * (N - 1) - (t - 1) * t // 2 + (s - 1)
            out[m3] = self.base_f + fid * self.nfi + idx
        m4 = cnt == 4
        if m4.any():
            v = self._vidx[ijk[m4, 0], ijk[m4, 1], ijk[m4, 2]]
            out[m4] = self.base_v + T * self.nvi + v
        return out

    def _face_st(self, idx):
        """(s, t) of in-face index idx = (t-1)(N-1) - (t-1)t/2 + (s-1)."""
        N = self.N
        t = 1
        while idx >= N - 1 - t:
            idx -= N - 1 - t
            t += 1
        return idx + 1, t

    def locate(self, gid: int):
        """Every (macro T, lattice ijk) holding node `gid`, ascending T: the
        inverse of `gids` (vertex: gid; edge (a<b): node a + (m/N)(b-a); face
        (a<b<c): a + (s/N)(b-a) + (t/N)(c-a); volume: (T, k, j, i) order)."""
        N = self.N
        gid = int(gid)
        if gid >= self.base_v:
            T, v = divmod(gid - self.base_v, self.nvi)
            if not hasattr(self, "_inter"):
                self._inter = interior_ijk(N)
            return [(int(T), self._inter[v].copy())]
        if gid >= self.base_f:
            fid, idx = divmod(gid - self.base_f, self.nfi)
            a, b, c = (int(x) for x in self.faces[fid])
            s, t = self._face_st(idx)
            wts = {a: N - s - t, b: s, c: t}
        elif gid >= self.base_e:
            eid, m1 = divmod(gid - self.base_e, N - 1)
            a, b = (int(x) for x in self.edges[eid])
            wts = {a: N - (m1 + 1), b: m1 + 1}
        else:
            wts = {gid: N}
        if not hasattr(self, "_vmacros"):
            self._vmacros = [[] for _ in range(self.mesh.nv)]
            for T, tv in enumerate(self.mesh.tets):
                for v in tv:
                    self._vmacros[int(v)].append(T)
        out = []
        for T in self._vmacros[next(iter(wts))]:
            tv = [int(v) for v in self.mesh.tets[T]]
            if all(v in tv for v in wts):
                w = [wts.get(v, 0) for v in tv]
                out.append((T, np.array(w[1:4], dtype=np.int64)))
        return out

    def step_of(self, gid: int) -> int:
        """Index of the GS class step (in `gs_steps` order) that updates node
        `gid`: 0 vertices, 1-2 edge colours, 3-5 face colours, 6-9 volume
        colours; -1 for Dirichlet nodes (never updated)."""
        gid = int(gid)
        if self.dirichlet_mask[gid]:
            return -1
        N = self.N
        if gid < self.base_e:
            return 0
        if gid < self.base_f:
            m = (gid - self.base_e) % (N - 1) + 1
            return 1 + m % 2
        if gid < self.base_v:
            s, t = self._face_st((gid - self.base_f) % self.nfi)
            return 3 + (s + 2 * t) % 3
        i, j, k = self.locate(gid)[0][1]
        return 6 + int(i + 2 * j + 3 * k) % 4

    def node_class(self, gid):
        gid = np.asarray(gid)
        return np.where(gid < self.base_e, 0, np.where(gid < self.base_f, 1,
                        np.where(gid < self.base_v, 2, 3)))

    def gs_steps(self):
        """Ordered GS class steps (R13/R14): vertices;
        edge colours m%2 = 0,1; face colours (s+2t)%3 = 0,1,2; volume colours
        (i+2j+3k)%4 = 0..3.  Returns list of gid arrays (unknowns only)."""
        N = self.N
        unk = self.unknown_mask
        steps = []
        g = np.arange(self.mesh.nv)
        steps.append(g[unk[g]])
        ge = np.arange(self.base_e, self.base_f)
        m = (ge - self.base_e) % (N - 1) + 1
        for c in range(2):
            s = ge[(m % 2) == c]
            steps.append(s[unk[s]])
        gf = np.arange(self.base_f, self.base_v)
        idx = (gf - self.base_f) % self.nfi
        st = []
        for t in range(1, N - 1):
            for s in range(1, N - t):
                st.append((s, t))
        st = np.array(st, dtype=np.int64).reshape(-1, 2)
        col = (st[idx, 0] + 2 * st[idx, 1]) % 3 if len(st) else np.zeros(0, np.int64)
        for c in range(3):
            s = gf[col == c]
            steps.append(s[unk[s]])
        inter = interior_ijk(N)
        vcol = (inter[:, 0] + 2 * inter[:, 1] + 3 * inter[:, 2]) % 4
        for c in range(4):
            loc = np.nonzero(vcol == c)[0]
            s = (self.base_v + np.arange(self.mesh.nt)[:, None] * self.nvi + loc[None, :]).ravel()
            steps.append(np.sort(s))
        return steps

    def coords(self, blended=True) -> np.ndarray:
        """Coordinates of every global node (from the lowest-id macro containing it)."""
        X = np.full((self.n_total, 3), np.nan)
        lat = lattice_ijk(self.N)
        for T in range(self.mesh.nt - 1, -1, -1):
            g = self.gids(T, lat)
            X[g] = node_coords(self.mesh, T, lat, self.N, blended)
        return X
