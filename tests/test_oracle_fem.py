"""Pins for oracle/fem.py: closed forms, invariants, special cases, brute force."""
import numpy as np
import pytest

import synth
from oracle import fem, geometry as G


def two_macro_mesh():
    """Two tets of the shell sharing one face; all other faces Dirichlet."""
    sh = synth.shell_mesh(0.55, 1.0, 0, 1)
    tets = sh.tets[:2]
    vids = np.unique(tets)
    remap = {int(v): i for i, v in enumerate(vids)}
    t2 = np.vectorize(remap.get)(tets)
    d = np.ones((2, 4), dtype=np.uint8)
    shared = set(t2[0]) & set(t2[1])
    for T in range(2):
        for f in range(4):
            if set(int(t2[T, v]) for v in range(4) if v != f) == shared:
                d[T, f] = 0
    return synth.MacroMesh(sh.vertices[vids], sh.radius[vids], t2, d)


def test_reference_stiffness_closed_form():
    P = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float)
    K = fem.local_stiffness(P)
    ref = np.array([[3, -1, -1, -1], [-1, 1, 0, 0], [-1, 0, 1, 0], [-1, 0, 0, 1]]) / 6.0
    assert np.allclose(K, ref, atol=1e-15)


def test_stiffness_invariances():
    rng = np.random.default_rng(1)
    P = rng.normal(size=(4, 3))
    K = fem.local_stiffness(P)
    assert np.allclose(K.sum(1), 0, atol=1e-13)
    assert np.allclose(K, K.T)
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    assert np.allclose(fem.local_stiffness(P @ Q.T + 3.0), K, atol=1e-12)
    assert np.allclose(fem.local_stiffness(2.0 * P), 2.0 * K, atol=1e-12)   # |T| h^3 * h^-2
    # vertex permutation permutes the matrix
    p = [2, 0, 3, 1]
    assert np.allclose(fem.local_stiffness(P[p]), K[np.ix_(p, p)], atol=1e-12)


def _brute_assemble(mesh, N):
    """Independent assembly: python dict over every fine tet of every macro."""
    num = G.Numbering(mesh, N)
    A = {}
    for T in range(mesh.nt):
        for tet in G.kuhn_tets(N):
            P = G.node_coords(mesh, T, tet, N)
            K = fem.local_stiffness(P)
            g = num.gids(T, tet)
            for a in range(4):
                for b in range(4):
                    A[(g[a], g[b])] = A.get((g[a], g[b]), 0.0) + K[a, b]
    return num, A


def test_csr_equals_brute_force_two_macros():
    m = two_macro_mesh()
    N = 4
    num, A = _brute_assemble(m, N)
    C = fem.assemble(m, N, num).tocoo()
    got = {(int(r), int(c)): v for r, c, v in zip(C.row, C.col, C.data)}
    assert set(got) == set(A)
    for k in A:
        assert abs(got[k] - A[k]) < 1e-14


def test_nodewise_rows_equal_csr_rows_for_lower_primitives():
    m = synth.shell_mesh(0.55, 1.0, 0, 1)
    N = 4
    num = G.Numbering(m, N)
    C = fem.assemble(m, N, num).tocsr()
    rng = np.random.default_rng(0)
    for gid in list(rng.choice(num.base_v, 12, replace=False)) + [0, num.base_e, num.base_f]:
        row = fem.fem_row(m, num, int(gid))
        r = C[int(gid)]
        csr = dict(zip(r.indices.tolist(), r.data.tolist()))
        assert set(csr) == set(row)
        for k in row:
            assert abs(csr[k] - row[k]) < 1e-14


def test_exact_stencil_invariants_blended():
    m = synth.single_tet()
    N = 16
    I = G.interior_ijk(N)
    s = fem.volume_stencils(m, 0, I, N)
    # zero row sums (Galerkin, constants in the kernel)
    assert np.abs(s.sum(1)).max() < 1e-14 * np.abs(s).max() * 15
    # P1 annihilates linear functions on a straight-sided fine mesh
    for c in range(3):
        acc = np.zeros(len(I))
        for w, d in enumerate(G.DIRS):
            acc += s[:, w] * G.node_coords(m, 0, I + d, N)[:, c]
        assert np.abs(acc).max() < 1e-14
    # exact symmetry s_w(I) = s_{w°}(I + w) for interior neighbour pairs
    lut = {tuple(v): n for n, v in enumerate(I)}
    nchk = 0
    for n, v in enumerate(I):
        for w, d in enumerate(G.DIRS):
            J = tuple(v + d)
            if J in lut:
                assert abs(s[n, w] - s[lut[J], G.opposite(w)]) < 1e-15
                nchk += 1
    assert nchk > 1000
    assert np.all(s[:, G.MC] > 0)
    # the blended stencil is genuinely non-constant (curved macro)
    assert np.ptp(s[:, G.MC]) > 1e-3 * s[:, G.MC].mean()


def test_affine_macro_constant_stencil_and_level_scaling():
    m = synth.single_tet()
    flat = synth.MacroMesh(m.vertices, None, m.tets, m.dirichlet)
    prev = None
    for L in (2, 3, 4, 5):
        N = 2 ** L
        I = G.interior_ijk(N)
        s = fem.volume_stencils(flat, 0, I, N)
        assert np.abs(s - s[0]).max() < 1e-14
        if prev is not None:
            # s^I = 2^-l s_hat
            assert np.allclose(s[0], prev / 2.0, rtol=1e-13, atol=1e-16)
        prev = s[0]
    # the affine stencil is symmetric in opposite directions
    assert np.allclose(prev, prev[::-1], atol=1e-15)


def test_global_matrix_symmetric_and_annihilates_constants():
    m = synth.shell_mesh(0.55, 1.0, 0, 1)
    num = G.Numbering(m, 4)
    A = fem.assemble(m, 4, num)
    assert abs(A - A.T).max() < 1e-15
    assert np.abs(A @ np.ones(num.n_total)).max() < 1e-14
    B = fem.apply_dirichlet(A, num)
    # SPD on unknowns
    u = num.unknown_mask.astype(float) * np.random.default_rng(0).normal(size=num.n_total)
    assert u @ (B @ u) > 0


def test_lumped_rhs_total_volume():
    # sum_I f_I with f == 1 and no Dirichlet masking equals the mesh volume
    m = synth.single_tet()
    N = 8
    num = G.Numbering(m, N)
    one = lambda x, y, z: np.ones_like(x)
    num.dirichlet_mask[:] = False
    f = fem.rhs_lumped(m, num, one)
    vol = 0.0
    for tet in G.kuhn_tets(N):
        P = G.node_coords(m, 0, tet, N)
        vol += abs(np.linalg.det(np.stack([P[1] - P[0], P[2] - P[0], P[3] - P[0]]))) / 6
    assert abs(f.sum() - vol) < 1e-14
