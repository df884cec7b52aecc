"""Pins for oracle/surrogate.py: paper counts, row-sum lemma, LS properties,
planted fields, affine special case, O(H^(q+1)) decay, forward differencing."""
import os

import numpy as np
import pytest

import synth
from oracle import fem, geometry as G, surrogate as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line.split())
    return rows


def _sampling_sizes(L, rule):
    l = L - 2
    if rule == "ipoly":
        return len(S.ipoly_samples(L))
    j = {"2": 2, "l-1": l - 1, "l": l}[rule]
    return len(S.lsqp_samples(L, j))


def test_table_setup_sampling_counts():
    # PAPER.md Table setup is at paper level L = 5, i.e. BASELINE L = 7; sum over l = 1..5
    g = {(r[0], r[1]): int(r[2]) for r in _golden("paper_counts.txt") if r[0] in ("sumS", "SL", "m_q")}
    assert S.n_coeffs(2) == g[("m_q", "2")] == len(S.exponents(2))
    for rule in ("ipoly", "2", "l-1", "l"):
        if rule == "ipoly":
            sizes = [10] * 5
        else:
            sizes = []
            for Lb in range(3, 8):
                l = Lb - 2
                j = {"2": 2, "l-1": l - 1, "l": l}[rule]
                m = S.sampling_level(Lb, j)
                sizes.append(G.n_interior(2 ** (m + 2)))
        assert sizes[-1] == g[("SL", rule)]
        assert sum(sizes) == g[("sumS", rule)]
    # the sample sets themselves have those sizes and lie in the interior
    for Lb in (3, 4, 5):
        Sm = S.lsqp_samples(Lb, 2)
        N = 2 ** Lb
        assert np.all(Sm >= 1) and np.all(Sm.sum(1) <= N - 1)
        assert len({tuple(x) for x in Sm}) == len(Sm)
    assert _sampling_sizes(4, "ipoly") == 10


def test_full_rank_up_to_q4_on_M1():
    # A has full rank for q <= 4 on any M_k, k >= 1
    for q in range(0, 5):
        A = S.basis(S.lsqp_samples(3, 1), 8, q)
        assert np.linalg.matrix_rank(A) == S.n_coeffs(q)
    A = S.basis(S.lsqp_samples(3, 1), 8, 5)
    assert np.linalg.matrix_rank(A) < S.n_coeffs(5)        # m_5 = 56 > n_1 = 35


@pytest.mark.parametrize("q", [1, 2, 3])
def test_planted_polynomial_recovered_exactly(q):
    rng = np.random.default_rng(q)
    L = 5
    N = 2 ** L
    Sm = S.lsqp_samples(L, 2)
    a_true = rng.normal(size=(S.n_coeffs(q), 15))
    b = S.basis(Sm, N, q) @ a_true
    a = S.fit_values(Sm, b, N, q)
    I = G.interior_ijk(N)
    assert np.abs(S.eval_weights(a, I, N, q) - S.eval_weights(a_true, I, N, q)).max() < 1e-12


def test_lsqp_row_sum_lemma_and_normal_equations():
    m = synth.single_tet()
    L = 5
    N = 2 ** L
    a = S.fit_macro(m, 0, L, 2, "lsqp", 2)
    # row sum lemma: sum_w a_w = 0
    assert np.abs(a.sum(1)).max() < 1e-14 * np.abs(a).max() * 15
    Sm = S.lsqp_samples(L, 2)
    b = fem.volume_stencils(m, 0, Sm, N)
    A = S.basis(Sm, N, 2)
    ne = A.T @ (A @ a - b)
    assert np.abs(ne).max() < 1e-13 * np.abs(A.T @ b).max()
    # IPOLY: interpolates its 10 points exactly, row sum preserved
    ai = S.fit_macro(m, 0, L, 2, "ipoly")
    Si = S.ipoly_samples(L)
    bi = fem.volume_stencils(m, 0, Si, N)
    assert np.abs(S.eval_weights(ai, Si, N, 2) - bi).max() < 1e-13
    assert np.abs(ai.sum(1)).max() < 1e-12


def test_affine_macro_surrogate_equals_fem():
    m = synth.single_tet()
    flat = synth.MacroMesh(m.vertices, None, m.tets, m.dirichlet)
    L = 5
    N = 2 ** L
    I = G.interior_ijk(N)
    a = S.fit_macro(flat, 0, L, 2, "lsqp", 2, blended=False)
    s = fem.volume_stencils(flat, 0, I[:50], N)
    assert np.abs(S.eval_weights(a, I, N, 2) - s[0]).max() < 1e-13


def _family(s, r1=0.55):
    """Shrinking curved tets: H -> H 2^-s around the radial edge of the config-1 tet."""
    p = (1 + 5 ** 0.5) / 2
    f = np.array([(0.0, 1.0, p), (0.0, -1.0, p), (p, 0.0, 1.0)])
    f /= np.linalg.norm(f, axis=1, keepdims=True)
    h = 2.0 ** -s
    n0 = f[0]
    n1 = n0 + (f[1] - n0) * h
    n2 = n0 + (f[2] - n0) * h
    n1 /= np.linalg.norm(n1)
    n2 /= np.linalg.norm(n2)
    ri = 1 - (1 - r1) * h
    V = np.stack([ri * n0, n0, n1, n2])
    return synth.MacroMesh(V, np.array([ri, 1, 1, 1.0]), np.array([[0, 1, 2, 3]]),
                           np.ones((1, 4), np.uint8))


@pytest.mark.parametrize("q", [1, 2, 3])
def test_surrogate_error_decays_like_H_q_plus_1(q):
    # A priori assumption L~ = L (Id + H^(q+1) B): the
    # relative stencil error of the LS fit decays by 2^(q+1) per halving of H.
    L = 4
    N = 2 ** L
    I = G.interior_ijk(N)
    errs = []
    for s in (2, 3, 4):
        m = _family(s)
        sx = fem.volume_stencils(m, 0, I, N)
        a = S.fit_values(I, sx, N, q)
        errs.append(np.abs(S.eval_weights(a, I, N, q) - sx).max() / np.abs(sx).max())
    ratio = errs[-2] / errs[-1]
    assert 0.75 * 2 ** (q + 1) < ratio < 1.6 * 2 ** (q + 1)


def test_forward_difference_golden_and_exact():
    g = {r[0]: r[1:] for r in _golden("forward_difference.txt")}
    vals = S.forward_difference(float(g["p0"][0]), float(g["dp0"][0]), float(g["dk"][0]), 4)
    assert list(vals) == [float(v) for v in g["values"]]
    # incremental vs direct along a line of a fitted surrogate polynomial
    m = synth.single_tet()
    L = 7
    N = 2 ** L
    a = S.fit_macro(m, 0, L, 2, "lsqp", 2)
    j0, k0 = 3, 5
    n = N - 1 - j0 - k0
    line = np.stack([np.arange(n), np.full(n, j0), np.full(n, k0)], 1)
    direct = S.eval_weights(a, line, N, 2)
    for w in range(15):
        p = direct[:, w]
        # seeds analytically: p(0), p'(0) and p''(0) of the quadratic in i
        c = np.polyfit(np.arange(n, dtype=float), p, 2)
        dk = 2 * c[0]
        inc = S.forward_difference(c[2], c[1] + dk / 2, dk, n)
        assert np.abs(inc - p).max() <= 1e-13 * np.abs(p).max()


def test_surrogate_operator_structure():
    m = synth.shell_mesh(0.55, 1.0, 0, 1)
    L = 3
    num = G.Numbering(m, 2 ** L)
    Lt, Lx, cf = S.surrogate_operator(m, L, 2, num=num)
    cls = num.node_class(np.arange(num.n_total))
    lower = np.nonzero(cls < 3)[0]
    assert abs(Lt[lower] - Lx[lower]).max() == 0.0
    vol = np.nonzero(cls == 3)[0]
    rs = Lt[vol] @ np.ones(num.n_total)
    assert np.abs(rs).max() < 1e-13
    # not symmetric on volume rows, but close: relative Frobenius asymmetry small
    asym = abs(Lt - Lt.T).power(2).sum() ** 0.5 / (Lx.power(2).sum() ** 0.5)
    assert 0 < asym < 0.05
    Lt2, Lx2, _ = S.surrogate_operator(m, 2, 2)
    assert abs(Lt2 - Lx2).max() == 0.0


def test_face_surrogate_special_cases():
    """Surrogate face rows.  Pins: on an
    affine macro mesh every face row is constant along the face, so the fit
    reproduces the exact rows (PAPER.md:638-641 analogue); fitted rows keep
    zero row sums (the fit is linear and the exact rows sum to zero,
    PAPER.md:696-717 analogue); on the curved shell the surrogate faces change
    the operator by a small relative amount that shrinks with H (more macros)."""
    import numpy as np
    import synth
    from oracle import geometry as G, surrogate as S
    m = synth.shell_mesh(0.55, 1.0, 0, 1)
    flat = synth.MacroMesh(m.vertices, None, m.tets, m.dirichlet)
    L = 4
    num = G.Numbering(flat, 2 ** L)
    Lt, A, cf = S.surrogate_operator(flat, L, 2, num=num)
    Lf, _, _ = S.surrogate_operator_faces(flat, L, 2, num=num, A_exact=A, coeffs=cf)
    unk = np.nonzero(num.unknown_mask)[0]  # Dirichlet rows are not part of the operator
    assert abs((Lf - Lt)[unk]).max() <= 1e-13 * abs(Lt).max()
    rel = []
    for t in (0, 1):  # 60 -> 240 macros: the faces shrink tangentially
        mc = synth.shell_mesh(0.55, 1.0, t, 1)
        numc = G.Numbering(mc, 2 ** L)
        Ltc, Ac, cfc = S.surrogate_operator(mc, L, 2, num=numc)
        Lfc, _, _ = S.surrogate_operator_faces(mc, L, 2, num=numc, A_exact=Ac, coeffs=cfc)
        rows = np.nonzero(numc.unknown_mask[numc.base_f:numc.base_v])[0] + numc.base_f
        rs = np.asarray(Lfc[rows].sum(axis=1)).ravel()
        assert np.abs(rs).max() <= 1e-13 * abs(Lfc).max()
        rel.append(abs(Lfc[rows] - Ltc[rows]).max() / abs(Ltc[rows]).max())
    assert 0 < rel[1] < rel[0] < 0.1, rel
