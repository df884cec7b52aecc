"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (480-macro shell, q = 2 LSQP j = 2, one apply, one residual, one GS
sweep through the C-ABI), checked on SAMPLED outputs that the oracle computes
one by one from its own definitions:

* apply / residual at volume nodes: y_I = sum_w P s_w(I) u_(I+w) with the
  oracle's own LSQP fit of the node's macro;
* apply at face / edge / vertex nodes: the exact FEM row by node-wise
  assembly over the macros containing the node;
* the on-the-fly FEM operator at volume nodes: the oracle's node stencils
  from the 24 incident fine tets (fem.volume_stencils);
* one GS sweep at sampled vertex, edge, face (near-edge and interior) and
  volume nodes (interior and next to macro faces / edges): the class-step
  order (R13/R14) replayed on the node's dependency cone with the
  oracle's rows (surrogate at volume nodes, exact FEM at the others).

Tolerance: |gpu - oracle| <= 1e-12 * sum_w |s_w u_w| per sampled node (the
row's natural scale; north_star's 1e-12 relative).
"""
import functools

import numpy as np
import pytest

import synth
from oracle import fem, geometry as G, surrogate as S

pytestmark = pytest.mark.gpu
TOL = 1e-12
DIRS = np.array(G.DIRS)
MC = 7


def _mesh(t, nr):
    # t = None: the single curved tet (BASELINE configs 1/2) at the largest
    # level the ABI accepts (L = 8, N = 256: the widest bands and rings)
    return synth.single_tet() if t is None else synth.shell_mesh(0.55, 1.0, t, nr)


@functools.lru_cache(maxsize=None)
def case(t, nr, L):
    import torch

    import paper_1608_06473_b200 as hhg
    mesh = _mesh(t, nr)
    num = G.Numbering(mesh, 2 ** L)
    ctx = hhg.Ctx.from_mesh(mesh, L)
    ctx.fit(2, "lsqp", 2)
    g = np.arange(num.n_total)
    u = synth.uniform_pm1(0, g) * num.unknown_mask
    f = synth.uniform_pm1(1, g) * num.unknown_mask
    del g
    du, df = ctx.zeros(L), ctx.zeros(L)
    ctx.scatter_global(L, torch.from_numpy(u).cuda(), du)
    ctx.scatter_global(L, torch.from_numpy(f).cuda(), df)
    dy, dr = ctx.zeros(L), ctx.zeros(L)
    ctx.apply(L, du, dy)
    ctx.residual(L, du, df, dr)
    dfem = ctx.zeros(L)
    ctx.apply(L, du, dfem, op="fem")
    ctx.gs_sweep(L, du, df, 1)
    torch.cuda.synchronize()
    out = {"y": ctx.gather_global(L, dy), "r": ctx.gather_global(L, dr), "ug": ctx.gather_global(L, du),
           "yfem": ctx.gather_global(L, dfem)}
    ctx.close()
    return mesh, num, u, f, out


@functools.lru_cache(maxsize=None)
def coeffs(t, nr, L, T):
    mesh = _mesh(t, nr)
    return S.fit_macro(mesh, T, L, 2, "lsqp", 2, blended=True)


def sample_volume(rng, N, nt, n, min_dist):
    out = []
    while len(out) < n:
        T = int(rng.integers(nt))
        i, j, k = (int(x) for x in rng.integers(min_dist, N - min_dist, 3))
        if i + j + k <= N - min_dist:
            out.append((T, i, j, k))
    return out


@pytest.mark.parametrize("t,nr,L", [(1, 2, 6), (1, 2, 7), (None, None, 8)])
def test_fullsize_apply_residual_sampled(t, nr, L):
    mesh, num, u, f, out = case(t, nr, L)
    N = 2 ** L
    rng = np.random.default_rng(1234 + L)
    pts = sample_volume(rng, N, mesh.nt, 96, 1)
    # include nodes next to every macro face and the farthest corners
    pts += [(0, 1, 1, 1), (mesh.nt - 1, N - 3, 1, 1), (mesh.nt // 2, 1, N - 3, 1), (min(7, mesh.nt - 1), 1, 1, N - 3)]
    for T, i, j, k in pts:
        ijk = np.array([[i, j, k]])
        sw = S.eval_weights(coeffs(t, nr, L, T), ijk, N, 2)[0]
        gI = int(num.gids(T, ijk)[0])
        gn = num.gids(T, ijk + DIRS)
        un = u[gn]
        ref = float(np.dot(sw, un))
        scale = float(np.abs(sw * un).sum())
        assert abs(out["y"][gI] - ref) <= TOL * scale, (T, i, j, k, out["y"][gI], ref)
        assert abs(out["r"][gI] - (f[gI] - ref)) <= TOL * (scale + abs(f[gI])), (T, i, j, k)


def _containing(mesh, verts):
    return [T for T in range(mesh.nt) if all(v in set(int(x) for x in mesh.tets[T]) for v in verts)]


@pytest.mark.parametrize("t,nr,L", [(1, 2, 6), (1, 2, 7), (None, None, 8)])
def test_fullsize_lower_primitive_rows_sampled(t, nr, L):
    mesh, num, u, f, out = case(t, nr, L)
    N = 2 ** L
    rng = np.random.default_rng(99 + L)
    gids = []
    unk_f = np.nonzero(num.unknown_mask[num.base_f:num.base_v])[0] + num.base_f
    unk_e = np.nonzero(num.unknown_mask[num.base_e:num.base_f])[0] + num.base_e
    unk_v = np.nonzero(num.unknown_mask[:num.base_e])[0]
    for pool, n in ((unk_f, 12), (unk_e, 4), (unk_v, 2)):
        if len(pool):
            gids += [int(x) for x in rng.choice(pool, n, replace=False)]
    if t is None:  # single tet: every face Dirichlet -> lower-primitive outputs are 0
        lp = slice(0, num.base_v)
        assert not np.any(out["y"][lp]) and not np.any(out["r"][lp]) and not np.any(out["ug"][lp])
    for g in gids:
        if g >= num.base_f:
            verts = num.faces[(g - num.base_f) // num.nfi]
        elif g >= num.base_e:
            verts = num.edges[(g - num.base_e) // (N - 1)]
        else:
            verts = [g]
        row = fem.fem_row(mesh, num, g, blended=True, macros=_containing(mesh, [int(v) for v in verts]))
        cols = np.array(list(row.keys()))
        vals = np.array([row[c] for c in cols])
        un = u[cols]
        ref = float(np.dot(vals, un))
        scale = float(np.abs(vals * un).sum())
        assert abs(out["y"][g] - ref) <= TOL * scale, (g, out["y"][g], ref)
        assert abs(out["r"][g] - (f[g] - ref)) <= TOL * (scale + abs(f[g])), g


def _gs_replay(mesh, num, t, nr, L, u, f):
    """new_value(g): node g after ONE hybrid GS sweep, replayed on its
    dependency cone from the class-step definition (R13/R14,
    oracle.Numbering.step_of): a node of step s is updated from the values
    after step s-1 -- a neighbour of a lower step contributes its new value
    (recursively), every other neighbour its old value; Dirichlet nodes are 0.
    Rows: the surrogate at volume nodes (the oracle's fit of the node's macro),
    the exact FEM row (node-wise assembly over every macro holding the node,
    oracle.fem.fem_row) at face / edge / vertex nodes.
    Returns (value, scale) with scale = (|f| + sum_w |s_w v_w|) / |s_mc|."""
    N = 2 ** L
    memo = {}

    def row(g):
        if g >= num.base_v:
            T, ijk = num.locate(g)[0]
            sw = S.eval_weights(coeffs(t, nr, L, T), ijk[None, :], N, 2)[0]
            cols = num.gids(T, ijk[None, :] + DIRS)
            return dict(zip((int(x) for x in cols), sw))
        return fem.fem_row(mesh, num, g, blended=True, locs=num.locate(g))

    def new_value(g):
        if g in memo:
            return memo[g]
        sg = num.step_of(g)
        acc, mag, diag = 0.0, 0.0, None
        for c, w in row(g).items():
            if c == g:
                diag = w
                continue
            sc = num.step_of(c)
            if sc < 0:
                continue
            v = new_value(c)[0] if sc < sg else u[c]
            acc += w * v
            mag += abs(w * v)
        memo[g] = ((f[g] - acc) / diag, (abs(f[g]) + mag) / abs(diag))
        return memo[g]
    return new_value


@pytest.mark.parametrize("t,nr,L", [(1, 2, 6), (1, 2, 7), (None, None, 8)])
def test_fullsize_gs_sweep_sampled(t, nr, L):
    """One hybrid GS sweep on the bench workload, sampled on EVERY node class
    the smoother couples: vertex, edge and face nodes (face
    nodes next to an edge -- the near-edge write path -- and in the face
    interior), volume nodes next to a macro face or edge, and interior volume
    nodes -- each replayed on its dependency cone by _gs_replay."""
    mesh, num, u, f, out = case(t, nr, L)
    N = 2 ** L
    rng = np.random.default_rng(4321 + L)
    gids = []
    # volume nodes: deep interior, within 1..3 steps of a macro face, and next to a macro edge
    for T, i, j, k in sample_volume(rng, N, mesh.nt, 16, 5):
        gids.append(int(num.gids(T, np.array([[i, j, k]]))[0]))
    for x in range(16):
        T = int(rng.integers(mesh.nt))
        d = 1 + x % 3
        ijk = [(d, 5 + x, 7), (9, d, 3 + x), (4 + x, 6, d), (d, d, 10 + x), (1, N - 3 - x, 1)][x % 5]
        if sum(ijk) <= N - 1:
            gids.append(int(num.gids(T, np.array([ijk]))[0]))
    if t is not None:
        unk_f = np.nonzero(num.unknown_mask[num.base_f:num.base_v])[0] + num.base_f
        unk_e = np.nonzero(num.unknown_mask[num.base_e:num.base_f])[0] + num.base_e
        unk_v = np.nonzero(num.unknown_mask[:num.base_e])[0]
        # face nodes near an edge (s, t or N-s-t in {1, 2}) and in the interior of the face
        near, far = [], []
        for g in rng.choice(unk_f, 4000, replace=False):
            s_, t_ = num._face_st(int(g - num.base_f) % num.nfi)
            (near if min(s_, t_, N - s_ - t_) <= 2 else far).append(int(g))
        gids += near[:10] + far[:4]
        gids += [int(x) for x in rng.choice(unk_e, 6, replace=False)]
        gids += [int(x) for x in rng.choice(unk_v, 3, replace=False)]
    new_value = _gs_replay(mesh, num, t, nr, L, u, f)
    for g in gids:
        ref, scale = new_value(g)
        assert abs(out["ug"][g] - ref) <= TOL * scale, (g, num.step_of(g), out["ug"][g], ref)


@pytest.mark.parametrize("t,nr,L", [(1, 2, 6), (1, 2, 7), (None, None, 8)])
def test_fullsize_fem_operator_sampled(t, nr, L):
    mesh, num, u, f, out = case(t, nr, L)
    N = 2 ** L
    rng = np.random.default_rng(777 + L)
    pts = sample_volume(rng, N, mesh.nt, 48, 1)
    for T, i, j, k in pts:
        ijk = np.array([[i, j, k]])
        sw = fem.volume_stencils(mesh, T, ijk, N, blended=True)[0]
        gI = int(num.gids(T, ijk)[0])
        un = u[num.gids(T, ijk + DIRS)]
        ref = float(np.dot(sw, un))
        scale = float(np.abs(sw * un).sum())
        assert abs(out["yfem"][gI] - ref) <= TOL * scale, (T, i, j, k, out["yfem"][gI], ref)


@pytest.mark.parametrize("t,nr,L,kernel", [(1, 2, 7, "default"), (1, 2, 7, "prodw"), (1, 2, 7, "wide4"),
                                           (None, None, 8, "default")])
def test_fullsize_gs_kernels_bit_identical(t, nr, L, kernel, monkeypatch):
    """At the bench size (480-macro shell, L = 7, 167 M unknowns, the launch
    configuration bench.py times) and on the widest lattice the ABI accepts
    (single tet, L = 8: the 16-plane ring, refill every step), two GS sweeps
    of the persistent kernels are bit-identical to the 4 colour launches
    (HHG_GS_KERNEL=passes), which have no cross-CTA waits at all."""
    import torch

    import paper_1608_06473_b200 as hhg
    mesh = _mesh(t, nr)
    ctx = hhg.Ctx.from_mesh(mesh, L)
    ctx.fit(2, "lsqp", 2)
    n_local, n_owned, n_global = ctx.layout(L)
    g = np.arange(n_global)
    u, f = ctx.zeros(L), ctx.zeros(L)
    ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(0, g)).cuda(), u)
    ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(1, g)).cuda(), f)
    del g
    ref = u.clone()
    monkeypatch.setenv("HHG_GS_KERNEL", "passes")
    ctx.gs_sweep(L, ref, f, 2)
    if kernel == "default":
        monkeypatch.delenv("HHG_GS_KERNEL")
    else:
        monkeypatch.setenv("HHG_GS_KERNEL", kernel)
    ctx.gs_sweep(L, u, f, 2)
    torch.cuda.synchronize()
    assert torch.equal(u, ref)
    ctx.close()
