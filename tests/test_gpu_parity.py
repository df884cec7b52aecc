"""Parity of the CUDA path (through the C-ABI) against the CPU oracle.

Tolerance (BASELINE north_star): relative 1e-12 in the 2-norm per vector.
Inputs: synth.uniform_pm1 on canonical global ids, zero on Dirichlet nodes.
"""
import functools

import numpy as np
import pytest

import synth
from oracle import fem, geometry as G, solvers, surrogate as S

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def elem_rel(a, b, scale):
    """Element-wise max relative error: max_i |a_i - b_i| / scale_i, with scale_i
    the magnitude of the terms summed into entry i (|L||u| + |f| for apply /
    residual: the natural per-row scale of a rounding error)."""
    a, b, scale = (np.asarray(x, dtype=np.float64) for x in (a, b, scale))
    m = scale > 0
    assert np.all(a[~m] == b[~m])
    return float(np.max(np.abs(a[m] - b[m]) / scale[m])) if m.any() else 0.0


MESHES = {
    "tet": lambda: synth.single_tet(),
    "shell60": lambda: synth.shell_mesh(0.55, 1.0, 0, 1),
    "shell120": lambda: synth.shell_mesh(0.55, 1.0, 0, 2),
    "shell480": lambda: synth.shell_mesh(0.55, 1.0, 1, 2),
    "flat_tet": lambda: (lambda m: synth.MacroMesh(m.vertices, None, m.tets, m.dirichlet))(synth.single_tet()),
}


@functools.lru_cache(maxsize=None)
def oracle_case(mesh_name, L, q=2, method="lsqp", j=2):
    mesh = MESHES[mesh_name]()
    num = G.Numbering(mesh, 2 ** L)
    A = fem.assemble(mesh, 2 ** L, num, blended=mesh.radius is not None)
    if L >= 3:
        cf = np.stack([S.fit_macro(mesh, T, L, q, method, j, blended=mesh.radius is not None)
                       for T in range(mesh.nt)])
    else:
        cf = None
    Lt, _, _ = S.surrogate_operator(mesh, L, q, method, j, num=num, A_exact=A, coeffs=cf)
    return mesh, num, Lt, A, cf


@functools.lru_cache(maxsize=None)
def gpu_ctx(mesh_name, L, q=2, method="lsqp", j=2):
    import paper_1608_06473_b200 as hhg
    mesh = MESHES[mesh_name]()
    ctx = hhg.Ctx.from_mesh(mesh, L)
    ctx.fit(q, method, j)
    return ctx


def vecs(num, seeds=(0, 1)):
    g = np.arange(num.n_total)
    return [synth.uniform_pm1(s, g) * num.unknown_mask for s in seeds]


def to_local(ctx, L, x):
    import torch
    loc = ctx.zeros(L)
    ctx.scatter_global(L, torch.from_numpy(x).cuda(), loc)
    return loc


# ("tet", 7) is BASELINE config 2 at full size (129 nodes per edge, 36 bands of
# the march kernels); the 480-macro configs at L = 6, 7 are checked on sampled
# outputs in test_gpu_fullsize.py
# ("shell480", 5): the 480-macro shell of the bench workload at L = 5 (2.66 M
# nodes, 2 march bands per macro, curved non-Dirichlet faces) full-vector
CASES = [("tet", 2), ("tet", 3), ("tet", 4), ("tet", 5), ("tet", 6), ("tet", 7), ("shell60", 3), ("shell60", 4),
         ("shell120", 3), ("shell480", 3), ("shell480", 5)]


@pytest.mark.parametrize("mesh_name,L", CASES)
def test_layout_and_roundtrip(mesh_name, L):
    mesh, num, *_ = oracle_case(mesh_name, L)
    ctx = gpu_ctx(mesh_name, L)
    n_local, n_owned, n_global = ctx.layout(L)
    assert n_global == num.n_total
    assert n_owned == int(num.unknown_mask.sum())
    u, _ = vecs(num)
    loc = to_local(ctx, L, u)
    back = ctx.gather_global(L, loc)
    assert np.array_equal(back, u)


@pytest.mark.parametrize("mesh_name,L", CASES)
def test_surrogate_weights_match_oracle(mesh_name, L):
    mesh, num, Lt, A, cf = oracle_case(mesh_name, L)
    ctx = gpu_ctx(mesh_name, L)
    N = 2 ** L
    I = G.interior_ijk(N)
    for T in sorted({0, mesh.nt - 1}):
        got = ctx.eval_stencils(L, T, "surrogate")
        if L >= 3:
            ref = S.eval_weights(cf[T], I, N, 2)
        else:
            ref = fem.volume_stencils(mesh, T, I, N)
        assert np.abs(got - ref).max() <= TOL * np.abs(ref).max()
        fem_got = ctx.eval_stencils(L, T, "fem")
        fem_ref = fem.volume_stencils(mesh, T, I, N)
        assert np.abs(fem_got - fem_ref).max() <= TOL * np.abs(fem_ref).max()


@pytest.mark.parametrize("mesh_name,L", CASES)
def test_apply_residual_gs_match_oracle(mesh_name, L):
    import torch
    mesh, num, Lt, A, cf = oracle_case(mesh_name, L)
    ctx = gpu_ctx(mesh_name, L)
    u, f = vecs(num)
    du, df, dy, dr = to_local(ctx, L, u), to_local(ctx, L, f), ctx.zeros(L), ctx.zeros(L)
    ctx.apply(L, du, dy)
    y_ref = solvers.apply(Lt, num, u)
    y = ctx.gather_global(L, dy)
    assert rel(y, y_ref) < TOL
    m = solvers.mask(num)
    absLu = m * (abs(Lt) @ np.abs(m * u))
    assert elem_rel(y, y_ref, absLu) < TOL
    nrm = ctx.residual(L, du, df, dr, norm=True)
    r_ref = solvers.residual(Lt, num, u, f)
    r = ctx.gather_global(L, dr)
    assert rel(r, r_ref) < TOL
    assert elem_rel(r, r_ref, absLu + m * np.abs(f)) < TOL
    assert abs(nrm - np.linalg.norm(r_ref)) <= TOL * np.linalg.norm(r_ref)
    # copies of lower primitives are all written consistently
    y2 = ctx.zeros(L)
    y2.copy_(dy)
    ctx.sync_copies(L, y2)
    assert torch.equal(y2, dy)
    gs = solvers.GS(Lt, num)
    ug = du.clone()
    ctx.gs_sweep(L, ug, df, 2)
    u_ref = gs.sweep(u.copy(), f, 2)
    u2 = ctx.gather_global(L, ug)
    assert rel(u2, u_ref) < TOL
    # per node: (|f| + sum_{w != mc} |s_w u_w|) / |s_mc| at the final iterate
    # (the scale of the last update's rounding; the first sweep's errors are
    # damped by the second)
    d = np.where(m > 0, np.abs(gs.diag), 1.0)
    sc = m * (np.abs(f) + abs(gs.off) @ np.abs(u_ref)) / d
    assert elem_rel(u2, u_ref, sc) < 10 * TOL


@pytest.mark.parametrize("mesh_name,L", [("tet", 4), ("tet", 6), ("tet", 7), ("shell60", 3), ("flat_tet", 4)])
def test_fem_and_const_operators(mesh_name, L):
    mesh, num, Lt, A, cf = oracle_case(mesh_name, L)
    ctx = gpu_ctx(mesh_name, L)
    u, f = vecs(num)
    du, dy = to_local(ctx, L, u), ctx.zeros(L)
    ctx.apply(L, du, dy, op="fem")
    assert rel(ctx.gather_global(L, dy), solvers.apply(A, num, u)) < TOL
    flat = synth.MacroMesh(mesh.vertices, None, mesh.tets, mesh.dirichlet)
    Aff = fem.assemble(flat, 2 ** L, G.Numbering(flat, 2 ** L), blended=False)
    ctx.apply(L, du, dy, op="const")
    assert rel(ctx.gather_global(L, dy), solvers.apply(Aff, num, u)) < TOL


def test_host_pointer_inputs_match_device():
    mesh, num, Lt, A, cf = oracle_case("shell60", 3)
    ctx = gpu_ctx("shell60", 3)
    u, f = vecs(num)
    du, dy = to_local(ctx, 3, u), ctx.zeros(3)
    ctx.apply(3, du, dy)
    hu = du.cpu().numpy().copy()
    hy = np.zeros_like(hu)
    ctx.apply(3, hu, hy)
    # compare node values (padding slots of a layout block are undefined)
    assert np.array_equal(ctx.gather_global(3, hy), ctx.gather_global(3, dy))


def test_ipoly_and_other_degrees():
    for q, method in ((1, "lsqp"), (3, "lsqp"), (4, "lsqp"), (2, "ipoly")):
        mesh, num, Lt, A, cf = oracle_case("tet", 5, q, method)
        ctx = gpu_ctx("tet", 5, q, method)
        got = ctx.eval_stencils(5, 0)
        ref = S.eval_weights(cf[0], G.interior_ijk(32), 32, q)
        assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max(), (q, method)
        u, _ = vecs(num)
        du, dy = to_local(ctx, 5, u), ctx.zeros(5)
        ctx.apply(5, du, dy)
        assert rel(ctx.gather_global(5, dy), solvers.apply(Lt, num, u)) < TOL


def test_errors_are_reported():
    import paper_1608_06473_b200 as hhg
    m = synth.single_tet()
    ctx = hhg.Ctx.from_mesh(m, 3)
    u, y = ctx.zeros(3), ctx.zeros(3)
    with pytest.raises(hhg.HHGError) as e:
        ctx.apply(3, u, y)
    assert e.value.status == 9                    # STATE: fit first
    with pytest.raises(hhg.HHGError) as e:
        ctx.fit(5)
    assert e.value.status == 1                    # q > 4
    bad = synth.MacroMesh(np.zeros((4, 3)), None, m.tets, m.dirichlet)
    with pytest.raises(hhg.HHGError) as e:
        hhg.Ctx.from_mesh(bad, 3)
    assert e.value.status == 2                    # degenerate
    wrong_r = synth.MacroMesh(m.vertices, m.radius * 1.01, m.tets, m.dirichlet)
    with pytest.raises(hhg.HHGError) as e:
        hhg.Ctx.from_mesh(wrong_r, 3)
    assert e.value.status == 2
    ctx.fit(2)
    f = ctx.zeros(3)
    with pytest.raises(hhg.HHGError) as e:          # FEM is not a smoother
        ctx.vcycle(3, u, f, op="fem")
    assert e.value.status == 1
    with pytest.raises(hhg.HHGError) as e:          # unknown residual operator
        ctx._check(ctx._lib.hhg_vcycle_dd(ctx.h, 3, 3, 3, 2, 50, 0, 7, u.data_ptr(), f.data_ptr(), 1, None))
    assert e.value.status == 1
    with pytest.raises(hhg.HHGError) as e:          # u and f alias
        ctx.vcycle(3, u, u)
    assert e.value.status == 1


@functools.lru_cache(maxsize=None)
def oracle_hierarchy(mesh_name, L):
    return solvers.Hierarchy(MESHES[mesh_name](), L, 2, 2)


@pytest.mark.parametrize("mesh_name,L,cycles", [("tet", 4, 3), ("shell60", 4, 3), ("shell120", 3, 2),
                                               ("shell480", 5, 2)])
def test_vcycle_history_matches_oracle(mesh_name, L, cycles):
    """V(3,3), coarse 50 CG at L=2, 4-colour GS on every level: residual
    histories agree to 1e-10 relative (north_star), iterates to 1e-10."""
    H = oracle_hierarchy(mesh_name, L)
    num = H.num[L]
    u0, f = vecs(num, (7, 8))
    u_ref, hist_ref = H.solve(u0.copy(), f, cycles)
    ctx = gpu_ctx(mesh_name, L)
    du, df = to_local(ctx, L, u0), to_local(ctx, L, f)
    hist = ctx.vcycle(L, du, df, n_cycles=cycles)
    assert np.all(np.abs(hist - hist_ref) <= 1e-10 * hist_ref), (hist, hist_ref)
    assert rel(ctx.gather_global(L, du), u_ref) < 1e-10
    assert hist[-1] < 0.1 * hist[0]


@functools.lru_cache(maxsize=None)
def oracle_hierarchy_c(mesh_name, L, Lc):
    return solvers.Hierarchy(MESHES[mesh_name](), L, Lc, 2)


@pytest.mark.parametrize("mesh_name,L,Lc,cycles", [("tet", 3, 3, 1), ("shell60", 3, 3, 1), ("shell60", 4, 3, 2),
                                                   ("shell120", 4, 3, 1)])
def test_coarse_solve_level3_matches_oracle(mesh_name, L, Lc, cycles):
    """The replicated coarse solve (coarse.cu: exact FEM CSR over the canonical
    ids, all 50 CG iterations in one cooperative kernel) on a level with volume,
    face, edge and vertex rows: L = Lc is a pure CG solve from zero, L > Lc a
    V(3,3) cycle on top of it; histories and iterates agree with the oracle's
    cg on its assembled coarse matrix to 1e-10."""
    H = oracle_hierarchy_c(mesh_name, L, Lc)
    num = H.num[L]
    u0, f = vecs(num, (7, 8))
    u_ref, hist_ref = H.solve(u0.copy(), f, cycles)
    ctx = gpu_ctx(mesh_name, L)
    du, df = to_local(ctx, L, u0), to_local(ctx, L, f)
    hist = ctx.vcycle(L, du, df, n_cycles=cycles, L_coarse=Lc)
    assert np.all(np.abs(hist - hist_ref) <= 1e-10 * hist_ref), (hist, hist_ref)
    assert rel(ctx.gather_global(L, du), u_ref) < 1e-10


@pytest.mark.parametrize("mesh_name,L,cycles", [("tet", 4, 3), ("shell60", 4, 3)])
def test_vcycle_double_discretisation_matches_oracle(mesh_name, L, cycles):
    """Double discretisation: surrogate GS smoother, exact
    FEM residual (the element-wise on-the-fly kernel) on every level; history
    = exact-operator residual norm.  Agrees with the oracle to 1e-10."""
    H = oracle_hierarchy(mesh_name, L)
    num = H.num[L]
    u0, f = vecs(num, (7, 8))
    u_ref, hist_ref = H.solve(u0.copy(), f, cycles, dd=True)
    ctx = gpu_ctx(mesh_name, L)
    du, df = to_local(ctx, L, u0), to_local(ctx, L, f)
    hist = ctx.vcycle(L, du, df, n_cycles=cycles, residual_op="fem")
    assert np.all(np.abs(hist - hist_ref) <= 1e-10 * hist_ref), (hist, hist_ref)
    assert rel(ctx.gather_global(L, du), u_ref) < 1e-10


@pytest.mark.parametrize("mesh_name,L", [("tet", 3), ("tet", 5), ("shell60", 3), ("shell60", 4), ("shell120", 3)])
def test_lexicographic_gs_matches_oracle(mesh_name, L):
    """The paper's lexicographic hybrid smoother run as
    hyperplane wavefronts on the GPU equals the oracle's node-by-node
    lexicographic sweep (2 sweeps) to 1e-12."""
    mesh, num, Lt, A, cf = oracle_case(mesh_name, L)
    ctx = gpu_ctx(mesh_name, L)
    u, f = vecs(num)
    du, df = to_local(ctx, L, u), to_local(ctx, L, f)
    ctx.gs_sweep(L, du, df, 2, lexicographic=True)
    u_ref = solvers.GS(Lt, num).sweep_lex(u.copy(), f, 2)
    assert rel(ctx.gather_global(L, du), u_ref) < TOL


@pytest.mark.parametrize("mesh_name,L,cycles", [("tet", 4, 3), ("shell60", 4, 3)])
def test_vcycle_lexicographic_matches_oracle(mesh_name, L, cycles):
    """V(3,3) with the lexicographic smoother: residual history and iterate
    agree with the oracle to 1e-10."""
    H = oracle_hierarchy(mesh_name, L)
    num = H.num[L]
    u0, f = vecs(num, (7, 8))
    u_ref, hist_ref = H.solve(u0.copy(), f, cycles, lex=True)
    ctx = gpu_ctx(mesh_name, L)
    du, df = to_local(ctx, L, u0), to_local(ctx, L, f)
    hist = ctx.vcycle(L, du, df, n_cycles=cycles, lexicographic=True)
    assert np.all(np.abs(hist - hist_ref) <= 1e-10 * hist_ref), (hist, hist_ref)
    assert rel(ctx.gather_global(L, du), u_ref) < 1e-10


@functools.lru_cache(maxsize=None)
def oracle_faces_case(mesh_name, L):
    mesh, num, Lt, A, cf = oracle_case(mesh_name, L)
    Lf, _, _ = S.surrogate_operator_faces(mesh, L, 2, num=num, A_exact=A, coeffs=cf)
    return mesh, num, Lf


@pytest.mark.parametrize("mesh_name,L", [("shell60", 3), ("shell60", 4), ("shell120", 3), ("shell120", 4)])
def test_surrogate_faces_operator_matches_oracle(mesh_name, L):
    """Surrogate face rows: apply, residual and a GS sweep with
    op = surrogate_faces equal the oracle's operator with fitted face rows
    (oracle.surrogate.surrogate_operator_faces) to 1e-12."""
    mesh, num, Lf = oracle_faces_case(mesh_name, L)
    ctx = gpu_ctx(mesh_name, L)
    u, f = vecs(num)
    du, df, dy, dr = to_local(ctx, L, u), to_local(ctx, L, f), ctx.zeros(L), ctx.zeros(L)
    ctx.apply(L, du, dy, op="surrogate_faces")
    assert rel(ctx.gather_global(L, dy), solvers.apply(Lf, num, u)) < TOL
    ctx.residual(L, du, df, dr, op="surrogate_faces")
    assert rel(ctx.gather_global(L, dr), solvers.residual(Lf, num, u, f)) < TOL
    ug = du.clone()
    ctx.gs_sweep(L, ug, df, 1, op="surrogate_faces")
    assert rel(ctx.gather_global(L, ug), solvers.GS(Lf, num).sweep(u.copy(), f, 1)) < TOL


@pytest.mark.parametrize("mesh_name,L", [("shell60", 4)])
def test_vcycle_graph_replay_matches_eager(mesh_name, L, monkeypatch):
    """HHG_VCYCLE_GRAPH=1 (cycles after the first replay one captured CUDA
    graph, the cooperative coarse-CG kernel included) gives bit-identical
    residual histories and iterates to the eager launches."""
    H = oracle_hierarchy(mesh_name, L)
    u0, f = vecs(H.num[L], (7, 8))
    ctx = gpu_ctx(mesh_name, L)
    du, df = to_local(ctx, L, u0), to_local(ctx, L, f)
    hist_e = ctx.vcycle(L, du, df, n_cycles=3)
    ue = ctx.gather_global(L, du)
    monkeypatch.setenv("HHG_VCYCLE_GRAPH", "1")
    du2 = to_local(ctx, L, u0)
    hist_g = ctx.vcycle(L, du2, df, n_cycles=3)
    assert np.array_equal(hist_g, hist_e), (hist_g, hist_e)
    assert np.array_equal(ctx.gather_global(L, du2), ue)


def _planted(rng, q, N):
    """15 random polynomials of degree <= q in index units (monomials
    i^l j^m k^n, l+m+n <= q) with a dominant positive centre weight."""
    ex = [(l, m, n) for d in range(q + 1) for l in range(d, -1, -1) for m in range(d - l, -1, -1)
          for n in [d - l - m]]
    c = rng.uniform(-1, 1, (15, len(ex))) / np.array([float(N) ** sum(e) for e in ex])
    c[7, 0] = 50.0

    def ev(ijk):
        ijk = np.asarray(ijk, dtype=np.float64)
        mono = np.stack([ijk[:, 0] ** l * ijk[:, 1] ** m * ijk[:, 2] ** n for l, m, n in ex], axis=1)
        return mono @ c.T  # [n, 15]
    return ev


@pytest.mark.parametrize("mesh_name,L,q_plant,q_fit,method", [("tet", 5, 2, 2, "lsqp"), ("shell60", 4, 1, 2, "lsqp"),
                                                              ("shell60", 5, 2, 2, "ipoly"), ("tet", 4, 3, 3, "lsqp")])
def test_fit_reproduces_planted_polynomials(mesh_name, L, q_plant, q_fit, method):
    """hhg_fit_from_samples (test export): a planted weight field that is a
    polynomial of degree <= q is reproduced exactly at every interior node
    (the least-squares fit of an exactly representable field is the field,
    PAPER.md:501-534) -- pins the library's sampling set, basis, QR
    pseudo-inverse and index-unit scaling independently of the FEM sampler."""
    import paper_1608_06473_b200 as hhg
    mesh = MESHES[mesh_name]()
    N = 2 ** L
    ctx = hhg.Ctx.from_mesh(mesh, L)
    rng = np.random.default_rng(10 * L + q_plant)
    smp = ctx.sample_nodes(L, method, 2)
    ref_smp = S.ipoly_samples(L) if method == "ipoly" else S.lsqp_samples(L, 2)
    assert {tuple(x) for x in smp} == {tuple(x) for x in ref_smp}
    fields = [_planted(rng, q_plant, N) for _ in range(mesh.nt)]
    ctx.fit_from_samples(L, np.stack([fld(smp) for fld in fields]), q=q_fit, method=method)
    I = G.interior_ijk(N)
    for T in sorted({0, mesh.nt - 1}):
        got = ctx.eval_stencils(L, T)
        ref = fields[T](I)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), T
    ctx.close()


def test_fit_affine_macro_gives_the_fem_constant_stencil():
    """On an unblended (affine) macro every exact stencil is the same
    (PAPER.md:380-384), so the fitted surrogate equals the FEM stencil at every
    node and the surrogate apply equals the CONS apply."""
    mesh, num, Lt, A, cf = oracle_case("flat_tet", 5)
    ctx = gpu_ctx("flat_tet", 5)
    sur = ctx.eval_stencils(5, 0, "surrogate")
    fem_w = ctx.eval_stencils(5, 0, "fem")
    assert np.abs(sur - fem_w).max() <= 1e-12 * np.abs(fem_w).max()
    assert np.abs(fem_w - fem_w[0]).max() <= 1e-12 * np.abs(fem_w).max()
    u, _ = vecs(num)
    du, dy, dc = to_local(ctx, 5, u), ctx.zeros(5), ctx.zeros(5)
    ctx.apply(5, du, dy)
    ctx.apply(5, du, dc, op="const")
    assert rel(ctx.gather_global(5, dy), ctx.gather_global(5, dc)) < TOL


def test_non_positive_centre_weight_raises_numeric():
    """HHG_ERR_NUMERIC (include/hhg.h): a fitted surrogate whose centre weight
    is <= 0 somewhere cannot be used by the GS update (it divides by s_mc,
    eq. iteration-scheme): the fit reports it, apply still
    works, every smoother call refuses it; a good refit clears it."""
    import paper_1608_06473_b200 as hhg
    mesh = synth.single_tet()
    L = 4
    ctx = hhg.Ctx.from_mesh(mesh, L)
    ctx.fit(2)
    smp = ctx.sample_nodes(L)
    good = ctx.eval_stencils(L, 0)
    I = G.interior_ijk(2 ** L)
    pos = {tuple(p): x for x, p in enumerate(I)}
    samples = np.stack([good[[pos[tuple(p)] for p in smp]]])
    bad = samples.copy()
    bad[0, :, 7] = 1.0 - smp[:, 0] / 4.0          # centre weight linear in i, < 0 for i > 4
    with pytest.raises(hhg.HHGError) as e:
        ctx.fit_from_samples(L, bad)
    assert e.value.status == 4
    u, f, y = ctx.zeros(L), ctx.zeros(L), ctx.zeros(L)
    ctx.apply(L, u, y)                              # apply does not divide
    with pytest.raises(hhg.HHGError) as e:
        ctx.gs_sweep(L, u, f, 1)
    assert e.value.status == 4
    with pytest.raises(hhg.HHGError) as e:
        ctx.vcycle(L, u, f, n_cycles=1)
    assert e.value.status == 4
    ctx.fit_from_samples(L, samples)                # the exact samples again: fine
    ctx.gs_sweep(L, u, f, 1)
    ctx.close()


@pytest.mark.parametrize("kernel", ["front", "front6", "wide4", "wide6", "prod", "prodw", "default"])
@pytest.mark.parametrize("mesh_name,L", [("tet", 7), ("shell480", 5), ("shell60", 4), ("tet", 3)])
def test_gs_kernels_bit_identical(mesh_name, L, kernel, monkeypatch):
    """Every volume GS kernel -- the persistent 4-pass sweep (default), the
    single-pass wavefronts ("front", "front6", "wide4", "wide6"), the
    producer-warp sweeps with per-plane progress ("prod", "prodw") and the 4
    colour launches ("passes", the reference here) -- computes the same
    4-colour sweep bit for bit (same per-node arithmetic gs_node_value, same
    colour order); surrogate and constant-stencil smoothers."""
    import torch
    mesh, num, *_ = oracle_case(mesh_name, L)
    ctx = gpu_ctx(mesh_name, L)
    u, f = vecs(num)
    du, df = to_local(ctx, L, u), to_local(ctx, L, f)
    for op in ("surrogate", "const"):
        ref = du.clone()
        monkeypatch.setenv("HHG_GS_KERNEL", "passes")
        ctx.gs_sweep(L, ref, df, 2, op=op)
        if kernel == "default":
            monkeypatch.delenv("HHG_GS_KERNEL")
        else:
            monkeypatch.setenv("HHG_GS_KERNEL", kernel)
        got = du.clone()
        ctx.gs_sweep(L, got, df, 2, op=op)
        assert torch.equal(got, ref), (op, (got - ref).abs().max().item())


def test_coarse_cg_through_operator_calls_matches_oracle(monkeypatch):
    """HHG_COARSE=ops (the coarse solver used for levels too large to
    replicate, coarse.cu::coarse_replicable): the same 50-iteration CG from
    zero through the library's operator calls; V(3,3) history as the oracle's
    to 1e-10."""
    H = oracle_hierarchy("shell60", 4)
    num = H.num[4]
    u0, f = vecs(num, (7, 8))
    u_ref, hist_ref = H.solve(u0.copy(), f, 2)
    ctx = gpu_ctx("shell60", 4)
    monkeypatch.setenv("HHG_COARSE", "ops")
    du, df = to_local(ctx, 4, u0), to_local(ctx, 4, f)
    hist = ctx.vcycle(4, du, df, n_cycles=2)
    assert np.all(np.abs(hist - hist_ref) <= 1e-10 * hist_ref), (hist, hist_ref)
    assert rel(ctx.gather_global(4, du), u_ref) < 1e-10


@pytest.mark.parametrize("kernel", ["default", "front", "wide4", "prod", "prodw"])
@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("mesh_name,L", [("tet", 7), ("shell480", 5)])
def test_gs_flag_protocol_stress(mesh_name, L, seed, kernel, monkeypatch):
    """Stress of the cross-CTA protocols of the persistent GS kernels
    (completion flags of the 4-pass sweep; LL halo words and progress words of
    the wavefront; per-plane progress words of the producer-warp sweeps,
    PAPER.md:1306-1315 update order): bands of every macro
    handed out in reverse order (odd seeds) and random delays of up to ~8 us
    before passes / steps -- the sweep stays bit-identical to the 4 colour
    launches, which have no cross-CTA waits at all."""
    import torch
    mesh, num, *_ = oracle_case(mesh_name, L)
    ctx = gpu_ctx(mesh_name, L)
    u, f = vecs(num)
    du, df = to_local(ctx, L, u), to_local(ctx, L, f)
    ref = du.clone()
    monkeypatch.setenv("HHG_GS_KERNEL", "passes")
    ctx.gs_sweep(L, ref, df, 2)
    if kernel == "default":
        monkeypatch.delenv("HHG_GS_KERNEL")
    else:
        monkeypatch.setenv("HHG_GS_KERNEL", kernel)
    monkeypatch.setenv("HHG_GS_STRESS", str(seed))
    got = du.clone()
    ctx.gs_sweep(L, got, df, 2)
    assert torch.equal(got, ref)
