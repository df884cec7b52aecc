"""Pins for oracle/solvers.py: invariants, fixed points, textbook special cases."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import synth
from oracle import fem, geometry as G, solvers, surrogate as S


@pytest.fixture(scope="module")
def shell3():
    m = synth.shell_mesh(0.55, 1.0, 0, 1)
    L = 3
    num = G.Numbering(m, 2 ** L)
    Lt, Lx, _ = S.surrogate_operator(m, L, 2, num=num)
    return m, num, Lt, Lx


def test_apply_annihilates_constants_away_from_boundary(shell3):
    m, num, Lt, Lx = shell3
    y = Lt @ np.ones(num.n_total)
    vol = np.arange(num.base_v, num.n_total)
    assert np.abs(y[vol]).max() < 1e-13
    # with Dirichlet masking only rows with a Dirichlet neighbour change
    Lm = Lt.tocsr()
    u = num.unknown_mask.astype(float)
    y2 = solvers.apply(Lt, num, u)
    for g in vol[::37]:
        cols = Lm[g].indices
        if num.unknown_mask[cols].all():
            assert abs(y2[g]) < 1e-13


def test_residual_of_zero_is_rhs(shell3):
    m, num, Lt, Lx = shell3
    f = synth.uniform_pm1(3, np.arange(num.n_total))
    f[num.dirichlet_mask] = 0
    r = solvers.residual(Lt, num, np.zeros(num.n_total), f)
    assert np.array_equal(r, f)


def test_affine_surrogate_apply_equals_fem_apply():
    m = synth.single_tet()
    flat = synth.MacroMesh(m.vertices, None, m.tets, m.dirichlet)
    L = 4
    num = G.Numbering(flat, 2 ** L)
    A = fem.assemble(flat, 2 ** L, num, blended=False)
    cf = np.stack([S.fit_macro(flat, 0, L, 2, blended=False)])
    Lt, _, _ = S.surrogate_operator(flat, L, 2, num=num, A_exact=A, coeffs=cf)
    u = synth.uniform_pm1(0, np.arange(num.n_total))
    assert np.abs(solvers.apply(Lt, num, u) - solvers.apply(A, num, u)).max() < 1e-13


def test_gs_fixed_point_and_independent_volume_colours(shell3):
    m, num, Lt, Lx = shell3
    gs = solvers.GS(Lt, num)
    unk = np.nonzero(num.unknown_mask)[0]
    f = synth.uniform_pm1(1, np.arange(num.n_total))
    f[num.dirichlet_mask] = 0
    Lu = Lt.tocsr()[unk][:, unk]
    ustar = np.zeros(num.n_total)
    ustar[unk] = spla.spsolve(Lu.tocsc(), f[unk])
    u1 = gs.sweep(ustar.copy(), f)
    assert np.abs(u1 - ustar).max() < 1e-12 * np.abs(ustar).max()
    for s in gs.steps[-4:]:                              # volume colours
        sub = Lt.tocsr()[s][:, s]
        sub = sub - sp.diags(sub.diagonal())
        assert abs(sub).max() == 0.0


def test_gs_matches_dense_colour_gs(shell3):
    m, num, Lt, Lx = shell3
    gs = solvers.GS(Lt, num)
    D = Lt.toarray()
    msk = num.unknown_mask
    u0 = synth.uniform_pm1(5, np.arange(num.n_total)) * msk
    f = synth.uniform_pm1(6, np.arange(num.n_total)) * msk
    u = u0.copy()
    for s in gs.steps:                                   # dense, literal eq. iteration-scheme
        old = u.copy()
        for I in s:
            acc = f[I]
            for J in np.nonzero(D[I])[0]:
                if J != I and msk[J]:
                    acc -= D[I, J] * old[J]
            u[I] = acc / D[I, I]
    assert np.abs(gs.sweep(u0.copy(), f) - u).max() < 1e-13


def test_gs_reduces_energy_error_for_symmetric_fem(shell3):
    m, num, Lt, Lx = shell3
    gs = solvers.GS(Lx, num)
    Lm = fem.apply_dirichlet(Lx, num)
    e = synth.uniform_pm1(2, np.arange(num.n_total)) * num.unknown_mask
    f = np.zeros(num.n_total)
    en = [e @ (Lm @ e)]
    for _ in range(3):
        e = gs.sweep(e, f)
        en.append(e @ (Lm @ e))
    assert all(b < a for a, b in zip(en, en[1:]))


def test_parity_rule_unique_coarse_edge_brute_force():
    N = 8
    lat = G.lattice_ijk(N)
    coarse = lat[np.all(lat % 2 == 0, axis=1)]
    cset = {tuple(c) for c in coarse}
    for F in lat:
        if np.all(F % 2 == 0):
            continue
        # exactly one coarse edge (pair of coarse nodes 2d apart along a lattice
        # direction) has F as its midpoint, and it is the parity-class direction
        pairs = {frozenset({tuple(F - d), tuple(F + d)}) for d in G.DIRS if np.any(d)
                 and tuple(F - d) in cset and tuple(F + d) in cset}
        assert len(pairs) == 1
        d = solvers._PARITY_DIR[tuple(F % 2)]
        assert pairs == {frozenset({tuple(F - np.array(d)), tuple(F + np.array(d))})}


def test_prolongation_reproduces_affine_functions_and_R_is_transpose():
    m = synth.shell_mesh(0.55, 1.0, 0, 1)
    flat = synth.MacroMesh(m.vertices, None, m.tets, m.dirichlet)
    nc, nf = G.Numbering(flat, 4), G.Numbering(flat, 8)
    P = solvers.prolongation(flat, nc, nf, masked=False)
    Xc, Xf = nc.coords(False), nf.coords(False)
    assert np.abs(P @ Xc - Xf).max() < 1e-14
    assert np.allclose(P @ np.ones(nc.n_total), 1.0)
    Pm = solvers.prolongation(flat, nc, nf)
    assert abs(Pm.T - Pm.T.tocsr()).max() == 0


def test_cg_matches_scipy_and_vcycle_contracts():
    m = synth.shell_mesh(0.55, 1.0, 0, 1)
    H = solvers.Hierarchy(m, 4, 2, 2)
    A = H.A_coarse
    num = H.num[2]
    b = synth.uniform_pm1(9, np.arange(num.n_total)) * num.unknown_mask
    x = solvers.cg(A, b, 50)
    unk = num.unknown_mask
    ref, _ = spla.cg(A[unk][:, unk], b[unk], rtol=1e-14, atol=0, maxiter=500)
    assert np.abs(x[unk] - ref).max() < 1e-8 * np.abs(ref).max()
    # zero rhs + zero guess stays zero
    z = np.zeros(H.num[4].n_total)
    u, hist = H.solve(z.copy(), z, 1)
    assert np.all(u == 0) and np.all(hist == 0)
    num4 = H.num[4]
    f = synth.uniform_pm1(4, np.arange(num4.n_total)) * num4.unknown_mask
    u0 = synth.uniform_pm1(7, np.arange(num4.n_total)) * num4.unknown_mask
    u, hist = H.solve(u0, f, 6)
    rates = hist[1:] / hist[:-1]
    assert np.all(rates[2:] < 0.5), rates


def test_double_discretisation_special_cases():
    """Double discretisation (surrogate smoother, exact
    residual).  Pins: on an affine macro mesh the surrogate IS the exact
    operator, so the DD cycle equals the plain cycle; zero
    data stays zero; on the curved shell the DD history is the exact-operator
    residual of the DD iterate."""
    m = synth.shell_mesh(0.55, 1.0, 0, 1)
    flat = synth.MacroMesh(m.vertices, None, m.tets, m.dirichlet)
    H = solvers.Hierarchy(flat, 4, 2, 2)
    num = H.num[4]
    g = np.arange(num.n_total)
    f = synth.uniform_pm1(4, g) * num.unknown_mask
    u0 = synth.uniform_pm1(7, g) * num.unknown_mask
    u1, h1 = H.solve(u0.copy(), f, 3)
    u2, h2 = H.solve(u0.copy(), f, 3, dd=True)
    assert np.abs(h1 - h2).max() <= 1e-11 * h1[0]
    assert np.linalg.norm(u1 - u2) <= 1e-11 * np.linalg.norm(u1)
    z = np.zeros(num.n_total)
    uz, hz = H.solve(z.copy(), z, 1, dd=True)
    assert np.all(uz == 0) and np.all(hz == 0)
    Hc = solvers.Hierarchy(m, 4, 2, 2)
    numc = Hc.num[4]
    A = fem.assemble(m, 16, numc, blended=True)
    fc = synth.uniform_pm1(4, np.arange(numc.n_total)) * numc.unknown_mask
    uc0 = synth.uniform_pm1(7, np.arange(numc.n_total)) * numc.unknown_mask
    uc, hc = Hc.solve(uc0.copy(), fc, 2, dd=True)
    mk = numc.unknown_mask
    assert abs(hc[-1] - np.linalg.norm(mk * (fc - A @ (mk * uc)))) <= 1e-12 * hc[0]
    assert hc[-1] < 0.5 * hc[0]


def test_lexicographic_gs_is_forward_substitution(shell3):
    """Lexicographic hybrid GS: after the lower-primitive
    class steps, the volume update equals the textbook forward substitution
    (D + L)^-1 (f - U u - A_vb u_b) with L / U the strictly lower / upper
    parts of the volume block in lexicographic order (scipy's triangular
    solve); the exact solution is a fixed point."""
    m, num, Lt, Lx = shell3
    gs = solvers.GS(Lt, num)
    g = np.arange(num.n_total)
    u = synth.uniform_pm1(3, g) * num.unknown_mask
    f = synth.uniform_pm1(4, g) * num.unknown_mask
    ul = gs.sweep_lex(u.copy(), f, 1)
    # reference: class steps of the colour sweep, then a triangular solve
    ub = u * num.unknown_mask
    for s, O in zip(gs.steps, gs.offrows):
        if s[0] < num.base_v:
            ub[s] = (f[s] - O @ ub) / gs.diag[s]
    vol = np.arange(num.base_v, num.n_total)
    mk = sp.diags(num.unknown_mask.astype(float))
    A = (mk @ Lt @ mk).tocsr()
    Avv = A[vol][:, vol]
    rhs = f[vol] - A[vol] @ np.where(np.arange(num.n_total) >= num.base_v, 0.0, ub) - sp.triu(Avv, 1) @ ub[vol]
    uv = spla.spsolve_triangular(sp.tril(Avv, 0).tocsr(), rhs, lower=True)
    assert np.abs(ul[vol] - uv).max() <= 1e-12 * np.abs(uv).max()
    assert np.abs(ul[:num.base_v] - ub[:num.base_v]).max() == 0
    # fixed point: the exact discrete solution is unchanged
    unk = num.unknown_mask
    x = np.zeros(num.n_total)
    x[unk] = spla.spsolve(A[unk][:, unk].tocsc(), f[unk])
    assert np.abs(gs.sweep_lex(x.copy(), f, 1) - x).max() <= 1e-10 * np.abs(x).max()


@pytest.mark.parametrize("L", [1, 2, 3])
def test_class_step_schedule_vertex_exchange_can_ride_with_edge_colour_0(L):
    """The lattice fact behind the library's 6-exchange GS sweep
    (ops.cu::gs_sweep_dev skips the exchange after the vertex step): in the
    assembled FEM matrix no edge row of colour 0 (even positions m >= 2) has a
    vertex column, and an edge row of colour 1 reads edge-colour-0 nodes of
    its OWN edge only -- so the vertex values may travel with the edge-colour-0
    exchange, while edge colour 1 still needs it."""
    mesh = synth.shell_mesh(0.55, 1.0, 0, 2)
    N = 2 ** L
    num = G.Numbering(mesh, N)
    A = fem.assemble(mesh, N, num).tocsr()
    saw_vertex_in_colour1 = False
    for g in range(num.base_e, num.base_f):
        if num.dirichlet_mask[g]:
            continue
        eid, m0 = divmod(g - num.base_e, N - 1)
        cols = A.indices[A.indptr[g]:A.indptr[g + 1]]
        if (m0 + 1) % 2 == 0:
            assert not np.any(cols < num.base_e), (g, cols[cols < num.base_e])
        else:
            saw_vertex_in_colour1 |= bool(np.any(cols < num.base_e))
            ec = cols[(cols >= num.base_e) & (cols < num.base_f)]
            other = ec[(ec - num.base_e) // (N - 1) != eid]
            assert all(num.step_of(int(x)) != 1 for x in other), (g, other)  # step 1 = edge colour 0
    assert saw_vertex_in_colour1 == (N >= 2)
