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
