"""Oracle surrogate operator: IPOLY / LSQP fit and the two-scale operator L~.

PAPER.md:458-534 (surrogate polynomial eq. quadraticPolynomial, m_q, IPOLY
sampling points, LSQP, sampling sets S_l = M_m(l,j))
(definition of L~: volume rows from the surrogate, lower primitives from FEM;
15 polynomials per macro and level), PAPER.md:696-717 (row-sum lemma).

Basis (R9): monomials x^l y^m z^n with x = i/N, y = j/N, z = k/N.
Weights are compared, never coefficients.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .fem import assemble, volume_stencils
from .geometry import DIRS, Numbering, interior_ijk


def exponents(q: int):
    """(l,m,n) with l+m+n <= q; m_q = (q+3)(q+2)(q+1)/6 of them (eq. numPolyCoeffs)."""
    out = []
    for d in range(q + 1):
        for l in range(d, -1, -1):
            for m in range(d - l, -1, -1):
                out.append((l, m, d - l - m))
    return out


def n_coeffs(q: int) -> int:
    return (q + 3) * (q + 2) * (q + 1) // 6


def basis(ijk: np.ndarray, N: int, q: int) -> np.ndarray:
    """Rows of A: lambda_lmn(i,j,k) = (i/N)^l (j/N)^m (k/N)^n."""
    x = np.asarray(ijk, dtype=np.float64) / N
    return np.stack([x[:, 0] ** l * x[:, 1] ** m * x[:, 2] ** n for (l, m, n) in exponents(q)], axis=1)


def sampling_level(L: int, j: int = 2) -> int:
    """m(l, j) = min{l, max{1, j}} (eq. samplingSetFunctions), l = L-2."""
    l = L - 2
    return min(l, max(1, j))


def lsqp_samples(L: int, j: int = 2) -> np.ndarray:
    """S_l = M_m(l,j) embedded at level-l indices (R10): the interior
    nodes of the N_m = 2^(m+2) lattice, scaled by 2^(l-m)."""
    l = L - 2
    m = sampling_level(L, j)
    return interior_ijk(2 ** (m + 2)) * (2 ** (l - m))


def ipoly_samples(L: int) -> np.ndarray:
    """The 10 IPOLY points for q = 2: a = 2^(l+2)-3, b = 2^(l+1)-1."""
    l = L - 2
    a = 2 ** (l + 2) - 3
    b = 2 ** (l + 1) - 1
    return np.array([(1, 1, 1), (1, 1, a), (1, a, 1), (a, 1, 1), (1, 1, b), (1, b, 1),
                     (b, 1, 1), (1, b, b), (b, 1, b), (b, b, 1)], dtype=np.int64)


def fit_macro(mesh, T: int, L: int, q: int = 2, method: str = "lsqp", j: int = 2,
              blended=True) -> np.ndarray:
    """Coefficients a [m_q, 15] of the 15 surrogate polynomials of macro T at
    level L (l = L-2 >= 1).  LSQP: argmin |A z - b_w|_2 by
    LAPACK least squares (DGELS-equivalent; never normal equations).  IPOLY:
    square solve at the 10 points (q = 2 only, as the paper defines them)."""
    if L < 3:
        raise ValueError("surrogate only on l >= 1 (L >= 3), PAPER.md:466-469")
    N = 2 ** L
    if method == "lsqp":
        S = lsqp_samples(L, j)
    elif method == "ipoly":
        if q != 2:
            raise ValueError("IPOLY points are given for q = 2 only (PAPER.md:490-499)")
        S = ipoly_samples(L)
    else:
        raise ValueError(method)
    b = volume_stencils(mesh, T, S, N, blended)          # [|S|, 15]
    return fit_values(S, b, N, q, square=(method == "ipoly"))


def fit_values(S: np.ndarray, b: np.ndarray, N: int, q: int, square=False) -> np.ndarray:
    """Solve A a = b (IPOLY, square, DGESV-equivalent) or a = argmin |A a - b|_2
    (LSQP) for sampled values b [|S|, n_rhs]."""
    A = basis(S, N, q)
    if square:
        return np.linalg.solve(A, b)
    a, *_ = np.linalg.lstsq(A, b, rcond=None)
    return a


def forward_difference(p0: float, dp0: float, dk: float, n: int) -> np.ndarray:
    """Incremental evaluation along a line, eq. linearstencilupdate
    (PAPER.md:1359-1371): s^d = p(0) + d*dp(0) + (d-1)d/2 * dk with
    dp(0) = p'(0) + dk/2, dk = p''(0).  Returned for d = 0..n-1."""
    d = np.arange(n, dtype=np.float64)
    return p0 + d * dp0 + (d - 1) * d / 2.0 * dk


def eval_weights(a: np.ndarray, ijk: np.ndarray, N: int, q: int) -> np.ndarray:
    """Direct evaluation P s_w(i,j,k) = sum a_lmn x^l y^m z^n (eq.
    quadraticPolynomial), all 15 w, centre included (R12)."""
    return basis(ijk, N, q) @ a


def surrogate_operator(mesh, L: int, q: int = 2, method: str = "lsqp", j: int = 2,
                       num: Numbering | None = None, A_exact=None, coeffs=None):
    """L~ over all canonical nodes (no BC): volume-primitive rows from the
    surrogate (column I+w gets P s_w(I); rows not symmetrised,
    PAPER.md:719-730); lower-primitive rows copied from the exact FEM matrix
    (PAPER.md:632-636).  For L = 2 (l = 0) L~ = L.
    Returns (L~, L, coeffs[nt, m_q, 15] or None)."""
    N = 2 ** L
    if num is None:
        num = Numbering(mesh, N)
    if A_exact is None:
        A_exact = assemble(mesh, N, num)
    if L < 3:
        return A_exact.copy(), A_exact, None
    inter = interior_ijk(N)
    cls = num.node_class(np.arange(num.n_total))
    lower = sp.diags((cls < 3).astype(np.float64)) @ A_exact
    rows, cols, vals = [], [], []
    cf = []
    for T in range(mesh.nt):
        a = coeffs[T] if coeffs is not None else fit_macro(mesh, T, L, q, method, j)
        cf.append(a)
        W = eval_weights(a, inter, N, q)                  # [n,15]
        gI = num.gids(T, inter)
        for w, d in enumerate(DIRS):
            rows.append(gI)
            cols.append(num.gids(T, inter + d))
            vals.append(W[:, w])
    vol = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                        shape=A_exact.shape).tocsr()
    return (lower + vol).tocsr(), A_exact, np.stack(cf)


# ---------------------------------------------------------------------------
# Surrogate face stencils: "all our techniques can also be
# applied to the construction of stencil entries associated with face and
# edge nodes".  Per macro face and per neighbour entry --
# the same neighbour relative to the face node everywhere on the face: an
# in-face offset (ds, dt) in the face's sorted-vertex frame, or a lattice
# direction into one of its two macros -- a degree-q polynomial in the face
# coordinates (s/N, t/N) is fitted by least squares to the exact weights at
# the face sample nodes: the interior nodes of the 2^(m+2) face lattice
# (m = m(l, j), the 2-D analogue of S_l, R10), embedded at level l.
# ---------------------------------------------------------------------------
def face_exponents(q: int):
    """(a, b) with a + b <= q, ordered by total degree, then a descending."""
    return [(d - b, b) for d in range(q + 1) for b in range(d + 1)]


def face_samples(L: int, j: int = 2) -> np.ndarray:
    """Face sample nodes (s, t): interior nodes of the N_m = 2^(m+2) face lattice
    (s, t >= 1, s + t <= N_m - 1, t outer), scaled by 2^(l-m)."""
    l = L - 2
    m = sampling_level(L, j)
    Nm = 2 ** (m + 2)
    st = [(s, t) for t in range(1, Nm - 1) for s in range(1, Nm - t)]
    return np.array(st, dtype=np.int64) * (2 ** (l - m))


def face_basis(st: np.ndarray, N: int, q: int) -> np.ndarray:
    x = np.asarray(st, dtype=np.float64) / N
    return np.stack([x[:, 0] ** a * x[:, 1] ** b for (a, b) in face_exponents(q)], axis=1)


def _face_node_ijk(mesh, T: int, fverts, s, t, N):
    """Lattice coordinates in macro T of face node (s, t) of the face with
    sorted global vertices fverts = (a < b < c): weight N-s-t on a, s on b, t on c."""
    w = np.zeros((len(s), 4), dtype=np.int64)
    loc = [int(np.nonzero(mesh.tets[T] == v)[0][0]) for v in fverts]
    w[:, loc[0]] = N - s - t
    w[:, loc[1]] = s
    w[:, loc[2]] = t
    return w[:, 1:]


def face_surrogate_rows(mesh, num: Numbering, A_exact, L: int, q: int = 2, j: int = 2):
    """Sparse matrix holding, for every face-node row (all faces with two
    macros), the surrogate weights; other rows empty."""
    N = 2 ** L
    from .geometry import DIRS as _DIRS
    rows, cols, vals = [], [], []
    S = face_samples(L, j)
    Bs = face_basis(S, N, q)
    st_all = np.array([(s, t) for t in range(1, N - 1) for s in range(1, N - t)], dtype=np.int64)
    Ba = face_basis(st_all, N, q)
    P = np.linalg.pinv(Bs)  # least squares (full column rank)
    A = A_exact.tocsr()
    for f, key in enumerate(num._fkey):
        c = key % num.mesh.nv
        ab = key // num.mesh.nv
        a, b = ab // num.mesh.nv, ab % num.mesh.nv
        fverts = (int(a), int(b), int(c))
        macros = [T for T in range(mesh.nt) if all(v in set(int(x) for x in mesh.tets[T]) for v in fverts)]
        if len(macros) != 2:
            continue
        gI_all = num.base_f + f * num.nfi + (st_all[:, 1] - 1) * (N - 1) - (st_all[:, 1] - 1) * st_all[:, 1] // 2 \
            + (st_all[:, 0] - 1)
        # neighbour entries: key -> (macro, direction) realising it
        entries = {("c",): (macros[0], 7)}
        for T in macros:
            loc = [int(np.nonzero(mesh.tets[T] == v)[0][0]) for v in fverts]
            lf = 6 - sum(loc)
            for w, d in enumerate(_DIRS):
                if w == 7:
                    continue
                dw = [-sum(d), d[0], d[1], d[2]]
                if dw[lf] == 0:
                    entries[("f", dw[loc[1]], dw[loc[2]])] = (T, w)
                elif dw[lf] > 0:
                    entries[("m", T, w)] = (T, w)
        assert len(entries) == 15, entries
        for ekey, (T, w) in entries.items():
            ijk_all = _face_node_ijk(mesh, T, fverts, st_all[:, 0], st_all[:, 1], N)
            gJ_all = num.gids(T, ijk_all + np.array(_DIRS[w]))
            # exact weights at the sample nodes
            idx = {(int(s), int(t)): x for x, (s, t) in enumerate(st_all)}
            sx = np.array([idx[(int(s), int(t))] for s, t in S])
            bvals = np.asarray(A[gI_all[sx], gJ_all[sx]]).ravel()
            coef = P @ bvals
            rows.append(gI_all)
            cols.append(gJ_all)
            vals.append(Ba @ coef)
    if not rows:
        return sp.csr_matrix(A_exact.shape)
    M = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=A_exact.shape)
    return M.tocsr()


def surrogate_operator_faces(mesh, L: int, q: int = 2, method: str = "lsqp", j: int = 2,
                             num: Numbering | None = None, A_exact=None, coeffs=None):
    """L~ with surrogate face rows as well: volume rows as in
    surrogate_operator, face-node rows from face_surrogate_rows, edge and vertex
    rows exact.  L = 2: exact (l = 0)."""
    N = 2 ** L
    if num is None:
        num = Numbering(mesh, N)
    Lt, A, cf = surrogate_operator(mesh, L, q, method, j, num=num, A_exact=A_exact, coeffs=coeffs)
    if L < 3:
        return Lt, A, cf
    cls = num.node_class(np.arange(num.n_total))
    keep = sp.diags((cls != 2).astype(np.float64))   # drop the exact face rows
    Fs = face_surrogate_rows(mesh, num, A, L, q, j)
    return (keep @ Lt + Fs).tocsr(), A, cf
