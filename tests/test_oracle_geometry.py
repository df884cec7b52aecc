"""Pins for oracle/geometry.py against what the paper and mathematics fix."""
import itertools
import os

import numpy as np
import pytest
import scipy.sparse as sp

import synth
from oracle import geometry as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    out = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            out.append(line.split())
    return out


def test_interior_counts_match_paper():
    for key, a, b, *_ in _golden("paper_counts.txt"):
        if key == "n_l":
            l, n = int(a), int(b)
            assert G.n_interior(2 ** (l + 2)) == n
            if l <= 3:
                assert len(G.interior_ijk(2 ** (l + 2))) == n


def test_index_set_bounds_redundant_but_consistent():
    # PAPER.md:374-376 prints 0 < i,j,k < 2^(l+2)-2 and i+j+k < 2^(l+2);
    # DESIGN.md R6 reads the interior as i,j,k>=1, i+j+k<=N-1.  The extra
    # per-coordinate bound is implied (i <= N-1-j-k <= N-3).
    for N in (4, 8, 16):
        I = G.interior_ijk(N)
        assert np.all(I < N - 2)
        brute = [(i, j, k) for i in range(1, N) for j in range(1, N) for k in range(1, N)
                 if i + j + k <= N - 1]
        assert len(brute) == len(I)


def _bey(tet, depth):
    """Literal recursive Bey refinement (8 children) on integer vertices."""
    if depth == 0:
        return [tet]
    x0, x1, x2, x3 = [np.array(v) for v in tet]
    m = lambda a, b: tuple((a + b) // 2)
    x01, x02, x03 = m(x0, x1), m(x0, x2), m(x0, x3)
    x12, x13, x23 = m(x1, x2), m(x1, x3), m(x2, x3)
    x0, x1, x2, x3 = tuple(x0), tuple(x1), tuple(x2), tuple(x3)
    kids = [(x0, x01, x02, x03), (x01, x1, x12, x13), (x02, x12, x2, x23), (x03, x13, x23, x3),
            (x01, x02, x03, x13), (x01, x02, x12, x13), (x02, x03, x13, x23), (x02, x12, x13, x23)]
    out = []
    for k in kids:
        out += _bey(k, depth - 1)
    return out


@pytest.mark.parametrize("N", [2, 4, 8])
def test_kuhn_equals_bey_refinement(N):
    d = int(np.log2(N))
    ref = ((0, 0, 0), (N, 0, 0), (0, N, 0), (0, 0, N))
    bey = {frozenset(t) for t in _bey(ref, d)}
    kuhn = {frozenset(tuple(v) for v in t) for t in G.kuhn_tets(N)}
    assert len(bey) == N ** 3
    assert bey == kuhn


def test_stencil_shape_24_tets_14_neighbours_valences():
    gold = {k: int(v) for k, v, *_ in (r for r in _golden("paper_counts.txt") if len(r) >= 2)
            if k in ("valence4", "valence6", "incident")}
    N = 8
    inc = G.incident_kuhn_tets(np.array([2, 2, 2]), N)
    assert len(inc) == gold["incident"]
    val = {}
    for t in inc:
        for v in t:
            d = tuple(v - np.array([2, 2, 2]))
            if d != (0, 0, 0):
                val[d] = val.get(d, 0) + 1
    assert set(val) == {tuple(d) for d in G.DIRS if tuple(d) != (0, 0, 0)}
    counts = np.array(list(val.values()))
    assert (counts == 4).sum() == gold["valence4"]
    assert (counts == 6).sum() == gold["valence6"]
    four = {G.DIR_NAMES[[tuple(x) for x in G.DIRS].index(d)] for d, c in val.items() if c == 4}
    assert four == {"mn", "ms", "tw", "be", "tse", "bnw"}


def test_lexicographic_predecessors_and_opposites():
    rows = {r[0]: r[1:] for r in _golden("lexicographic.txt")}
    name = dict(zip(G.DIR_NAMES, map(tuple, G.DIRS)))
    for w in rows["updated"]:
        di, dj, dk = name[w]
        assert (dk, dj, di) < (0, 0, 0)      # earlier in (k, j, i) lexicographic order
    for w in rows["pending"]:
        di, dj, dk = name[w]
        assert (dk, dj, di) > (0, 0, 0)
    a, b = rows["opposite"]
    assert G.opposite(G.DIR_NAMES.index(a)) == G.DIR_NAMES.index(b)
    for w in range(15):
        assert np.all(G.DIRS[G.opposite(w)] == -G.DIRS[w])


def test_volume_colouring_is_proper():
    # (i + 2j + 3k) mod 4 never equal for neighbours (R14)
    for d in G.DIRS:
        if np.any(d):
            assert (d[0] + 2 * d[1] + 3 * d[2]) % 4 != 0
    # red-black (i+j+k)%2 is NOT proper on this lattice
    assert any((d.sum() % 2) == 0 for d in G.DIRS if np.any(d))


@pytest.mark.parametrize("t,n_r", [(0, 1), (0, 2), (1, 1)])
def test_shell_mesh_counts_and_tags(t, n_r):
    m = synth.shell_mesh(0.55, 1.0, t, n_r)
    assert m.nt == 60 * 4 ** t * n_r
    # conforming: every face shared by <= 2 tets; boundary faces exactly the r1/r2 ones
    faces = {}
    for T in range(m.nt):
        for f in range(4):
            key = tuple(sorted(int(m.tets[T, v]) for v in range(4) if v != f))
            faces.setdefault(key, []).append((T, f))
    for key, owners in faces.items():
        assert len(owners) <= 2
        r = m.radius[list(key)]
        on_bnd = np.allclose(r, 0.55) or np.allclose(r, 1.0)
        if len(owners) == 1:
            assert on_bnd
        for T, f in owners:
            assert m.dirichlet[T, f] == (len(owners) == 1)
    E = m.vertices[m.tets]
    det = np.linalg.det(np.stack([E[:, 1] - E[:, 0], E[:, 2] - E[:, 0], E[:, 3] - E[:, 0]], -1))
    assert np.all(np.abs(det) > 1e-6)
    assert np.allclose(np.linalg.norm(m.vertices, axis=1), m.radius, rtol=1e-13)


def test_numbering_bijective_and_consistent():
    m = synth.shell_mesh(0.55, 1.0, 0, 2)
    N = 8
    num = G.Numbering(m, N)
    lat = G.lattice_ijk(N)
    seen = np.zeros(num.n_total, dtype=int)
    X = {}
    for T in range(m.nt):
        g = num.gids(T, lat)
        assert len(np.unique(g)) == len(g)
        seen[g] += 1
        c = G.node_coords(m, T, lat, N)
        for gg, cc in zip(g[:: 7], c[:: 7]):
            if gg in X:
                assert np.allclose(X[gg], cc, atol=1e-14)
            X[gg] = cc
    assert np.all(seen >= 1)
    # volume nodes appear once; shared primitives more often
    assert np.all(seen[num.base_v:] == 1)
    # closed-form unknown counts: faces in the interior only (boundary faces Dirichlet)
    n_int_faces = num.n_f - len(num.dirichlet_faces)
    assert num.unknown_mask[num.base_f:num.base_v].sum() == n_int_faces * num.nfi
    assert num.unknown_mask[num.base_v:].sum() == m.nt * G.n_interior(N)


def test_blending_properties():
    m = synth.single_tet()
    N = 16
    lat = G.lattice_ijk(N)
    x = G.node_coords(m, 0, lat, N)
    lam = G.barycentric(lat, N)
    r = lam @ m.radius
    assert np.allclose(np.linalg.norm(x, axis=1), r, rtol=1e-14)
    # macro vertices map to themselves
    for v, ijk in enumerate([(0, 0, 0), (N, 0, 0), (0, N, 0), (0, 0, N)]):
        xi = G.node_coords(m, 0, np.array([ijk]), N)[0]
        assert np.allclose(xi, m.vertices[v], atol=1e-15)
    # Phi = Id when radii are absent
    m2 = synth.MacroMesh(m.vertices, None, m.tets, m.dirichlet)
    X = G.node_coords(m2, 0, lat, N)
    assert np.allclose(X, lam @ m.vertices, atol=1e-15)


def test_gs_steps_partition_unknowns():
    m = synth.shell_mesh(0.55, 1.0, 0, 2)
    num = G.Numbering(m, 8)
    steps = num.gs_steps()
    allg = np.concatenate(steps)
    assert len(allg) == len(np.unique(allg)) == num.unknown_mask.sum()


def test_locate_inverts_gids_and_finds_every_copy():
    """Numbering.locate(g) lists exactly the (macro, ijk) with gids(T, ijk) == g
    (brute force over every lattice node of every macro)."""
    mesh = synth.shell_mesh(0.55, 1.0, 0, 1)
    N = 4
    num = G.Numbering(mesh, N)
    lat = G.lattice_ijk(N)
    where = {}
    for T in range(mesh.nt):
        for x, g in enumerate(num.gids(T, lat)):
            where.setdefault(int(g), []).append((T, tuple(int(v) for v in lat[x])))
    for g in range(num.n_total):
        got = [(T, tuple(int(v) for v in ijk)) for T, ijk in num.locate(g)]
        assert got == where[g], g


def test_step_of_matches_gs_steps():
    mesh = synth.shell_mesh(0.55, 1.0, 0, 1)
    num = G.Numbering(mesh, 8)
    step = -np.ones(num.n_total, dtype=int)
    for s, ids in enumerate(num.gs_steps()):
        step[ids] = s
    for g in range(0, num.n_total, 7):
        assert num.step_of(g) == step[g], g


def test_class_colours_are_independent_inside_each_primitive():
    """Face colours (s+2t) mod 3 are independent sets inside every face, edge
    parity classes inside every edge, and vertices are never neighbours (the
    simultaneous update of one class step is then a true GS step inside each
    primitive; across primitives it is the Jacobi-like coupling of the hybrid
    smoother)."""
    from oracle import fem
    mesh = synth.shell_mesh(0.55, 1.0, 0, 1)
    N = 8
    num = G.Numbering(mesh, N)
    A = fem.assemble(mesh, N, num, blended=True).tocsr()
    steps = num.gs_steps()
    for s in range(6):
        ids = steps[s]
        if s == 0:
            groups = [ids]
        elif s < 3:
            groups = [ids[(ids - num.base_e) // (N - 1) == e] for e in np.unique((ids - num.base_e) // (N - 1))]
        else:
            groups = [ids[(ids - num.base_f) // num.nfi == f] for f in np.unique((ids - num.base_f) // num.nfi)]
        for grp in groups:
            sub = A[grp][:, grp]
            sub = sub - sp.diags(sub.diagonal())
            assert abs(sub).max() == 0.0 if sub.nnz else True, (s, grp[:4])
    # and the classes are not globally independent across faces (the hybrid
    # smoother's Jacobi-like interface couplings exist on this mesh)
    coupled = 0
    for s in range(3, 6):
        sub = A[steps[s]][:, steps[s]]
        coupled += (sub - sp.diags(sub.diagonal())).nnz
    assert coupled > 0


def test_ipoly_points_are_the_papers():
    """IPOLY points equal the golden list written out from
    the paper's formula, are interior, and are the P2 nodes (vertices + edge
    midpoints) of the shrunk tet with vertices (1,1,1), (a,1,1), (1,a,1),
    (1,1,a)."""
    from oracle import surrogate as S
    rows = _golden("ipoly_points.txt")
    for L in (3, 4, 5):
        gold = {tuple(int(x) for x in r[1:]) for r in rows if int(r[0]) == L}
        pts = {tuple(int(v) for v in p) for p in S.ipoly_samples(L)}
        assert pts == gold and len(gold) == 10
        N = 2 ** L
        for i, j, k in pts:
            assert i >= 1 and j >= 1 and k >= 1 and i + j + k <= N - 1
        a = N - 3
        V = [np.array(v) for v in ((1, 1, 1), (a, 1, 1), (1, a, 1), (1, 1, a))]
        p2 = {tuple(int(x) for x in v) for v in V}
        p2 |= {tuple(int(x) for x in (V[p] + V[q]) // 2) for p, q in itertools.combinations(range(4), 2)}
        assert pts == p2
