"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the paper's method (no blending, no
stiffness, no stencils, no fit).  It only produces *inputs*:

* macro meshes of a spherical shell (the paper's T_{-2}, PAPER.md:202-207;
  construction unstated by the paper -- DESIGN.md reading R2: icosahedron x
  radial layers, prisms split into 3 tets by global vertex id), and the single
  curved macro tetrahedron of BASELINE configs 1/2;
* the canonical node numbering's *sizes* are NOT here (each side derives its
  own numbering independently);
* the counter-based random generator used for u, f (reading R21):
  value(gid) = 2 * (splitmix64(seed ^ gid) >> 11) * 2^-53 - 1.

Both the oracle (oracle/) and the CUDA path's tests call this module; neither
imports the other.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "splitmix64",
    "uniform_pm1",
    "shell_mesh",
    "single_tet",
    "MacroMesh",
]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    """SplitMix64 finaliser applied to uint64 array `x` (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uniform_pm1(seed: int, gids) -> np.ndarray:
    """U[-1,1) value per global node id: 2*(splitmix64(seed^gid)>>11)*2^-53 - 1."""
    g = np.asarray(gids, dtype=np.uint64)
    z = splitmix64(np.uint64(seed) ^ g)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


class MacroMesh:
    """Plain container: vertices [nv,3] f64, radius [nv] f64 (or None = Phi=Id),
    tets [nt,4] int64 (local vertex order = lattice axes x0,x1,x2,x3),
    dirichlet [nt,4] uint8 (face f = face opposite local vertex f)."""

    def __init__(self, vertices, radius, tets, dirichlet, name=""):
        self.vertices = np.ascontiguousarray(vertices, dtype=np.float64)
        self.radius = None if radius is None else np.ascontiguousarray(radius, dtype=np.float64)
        self.tets = np.ascontiguousarray(tets, dtype=np.int64)
        self.dirichlet = np.ascontiguousarray(dirichlet, dtype=np.uint8)
        self.name = name

    @property
    def nv(self):
        return self.vertices.shape[0]

    @property
    def nt(self):
        return self.tets.shape[0]


_PHI = (1.0 + 5.0 ** 0.5) / 2.0


def _icosahedron():
    p = _PHI
    v = []
    for a in (-1.0, 1.0):
        for b in (-p, p):
            v.append((0.0, a, b))
            v.append((a, b, 0.0))
            v.append((b, 0.0, a))
    v = np.array(v, dtype=np.float64)
    # faces: triples of mutually adjacent vertices (edge length 2 in these coords)
    d = np.linalg.norm(v[:, None, :] - v[None, :, :], axis=2)
    adj = np.abs(d - 2.0) < 1e-9
    faces = []
    n = len(v)
    for a in range(n):
        for b in range(a + 1, n):
            if not adj[a, b]:
                continue
            for c in range(b + 1, n):
                if adj[a, c] and adj[b, c]:
                    faces.append((a, b, c))
    assert len(faces) == 20
    v = v / np.linalg.norm(v, axis=1, keepdims=True)
    return v, np.array(faces, dtype=np.int64)


def _subdivide(v, faces):
    verts = [tuple(x) for x in v]
    cache = {}

    def mid(a, b):
        key = (min(a, b), max(a, b))
        if key not in cache:
            m = (np.asarray(verts[a]) + np.asarray(verts[b])) * 0.5
            m = m / np.linalg.norm(m)
            cache[key] = len(verts)
            verts.append(tuple(m))
        return cache[key]

    out = []
    for a, b, c in faces:
        ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
        out += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
    return np.array(verts, dtype=np.float64), np.array(out, dtype=np.int64)


def shell_mesh(r1: float = 0.55, r2: float = 1.0, t: int = 0, n_r: int = 1) -> MacroMesh:
    """Icosahedral shell macro mesh with 60 * 4**t * n_r tetrahedra.

    Surface: icosahedron, t midpoint subdivisions re-projected to the unit
    sphere.  Layers m = 0..n_r at r_m = r1 + m (r2 - r1) / n_r (uniform in r,
    DESIGN.md reading R3).  Vertex id = m * n_surface + s.  Each prism with
    bottom (a<b<c) and top (A,B,C) becomes (a,b,c,C), (a,b,B,C), (a,A,B,C):
    every quad is split along (lower-id bottom vertex, higher-id top vertex),
    which is conforming between neighbouring prisms.  Faces on r1 or r2 are
    tagged Dirichlet (the model problem's u = 0 on the boundary,
    PAPER.md:171-179).
    """
    if not (0.0 < r1 < r2) or t < 0 or n_r < 1:
        raise ValueError("need 0 < r1 < r2, t >= 0, n_r >= 1")
    sv, sf = _icosahedron()
    for _ in range(t):
        sv, sf = _subdivide(sv, sf)
    ns = sv.shape[0]
    radii = [r1 + m * (r2 - r1) / n_r for m in range(n_r + 1)]
    radii[-1] = r2
    verts = np.concatenate([sv * r for r in radii], axis=0)
    vrad = np.concatenate([np.full(ns, r) for r in radii])
    tets = []
    for m in range(n_r):
        for tri in sf:
            a, b, c = sorted(int(x) for x in tri)
            a0, b0, c0 = m * ns + a, m * ns + b, m * ns + c
            A, B, C = a0 + ns, b0 + ns, c0 + ns
            tets += [(a0, b0, c0, C), (a0, b0, B, C), (a0, A, B, C)]
    tets = np.array(tets, dtype=np.int64)
    layer = np.arange(verts.shape[0]) // ns
    dirichlet = np.zeros(tets.shape, dtype=np.uint8)
    for f in range(4):
        others = [v for v in range(4) if v != f]
        lay = layer[tets[:, others]]
        on_in = np.all(lay == 0, axis=1)
        on_out = np.all(lay == n_r, axis=1)
        dirichlet[:, f] = (on_in | on_out).astype(np.uint8)
    return MacroMesh(verts, vrad, tets, dirichlet, name=f"shell(t={t},n_r={n_r})")


def single_tet(r1: float = 0.55, r2: float = 1.0) -> MacroMesh:
    """BASELINE config 1/2 macro: (r1*v0, v0, v1, v2) of the normalised
    icosahedral face ((0,1,phi), (0,-1,phi), (phi,0,1)); all faces Dirichlet."""
    p = _PHI
    f = np.array([(0.0, 1.0, p), (0.0, -1.0, p), (p, 0.0, 1.0)])
    f = f / np.linalg.norm(f, axis=1, keepdims=True)
    verts = np.stack([r1 * f[0], r2 * f[0], r2 * f[1], r2 * f[2]])
    rad = np.array([r1, r2, r2, r2])
    tets = np.array([[0, 1, 2, 3]], dtype=np.int64)
    dirichlet = np.ones((1, 4), dtype=np.uint8)
    return MacroMesh(verts, rad, tets, dirichlet, name="single_tet")


def tet_batch(n: int, r1: float = 0.55, r2: float = 1.0) -> MacroMesh:
    """n disjoint copies of `single_tet` (BASELINE config 2 as a batch: the
    same curved macro n times, every face Dirichlet, no shared primitives)."""
    one = single_tet(r1, r2)
    verts = np.tile(one.vertices, (n, 1))
    rad = np.tile(one.radius, n)
    tets = (np.arange(n, dtype=np.int64)[:, None] * 4 + np.arange(4, dtype=np.int64)[None, :])
    dirichlet = np.ones((n, 4), dtype=np.uint8)
    return MacroMesh(verts, rad, tets, dirichlet, name=f"tet_batch{n}")

