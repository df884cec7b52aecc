"""Oracle solver operations: apply, residual, multicolour GS, transfers, CG, V-cycle.

PAPER.md:1306-1315 (eq. iteration-scheme: u_I = (f_I - sum_{w != mc} s_w
u_{I_w}) / s_mc), PAPER.md:852-860 (V(3,3), hybrid GS smoother),
PAPER.md:862-871 (residual).  Multicolour ordering, class steps,
transfers and the coarse CG are DESIGN.md readings R13, R14, R18, R19.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .geometry import Numbering, lattice_ijk

# parity-class -> coarse-edge direction for fine nodes not coinciding with a
# coarse node (R18; pinned by brute force in tests).
_PARITY_DIR = {
    (1, 0, 0): (1, 0, 0), (0, 1, 0): (0, 1, 0), (0, 0, 1): (0, 0, 1),
    (1, 1, 0): (-1, 1, 0), (1, 0, 1): (-1, 0, 1), (0, 1, 1): (0, -1, 1),
    (1, 1, 1): (1, -1, 1),
}


def mask(num: Numbering) -> np.ndarray:
    return num.unknown_mask.astype(np.float64)


def apply(Lt, num: Numbering, u: np.ndarray) -> np.ndarray:
    """y = L~ u over unknowns; Dirichlet entries of u ignored, of y zero."""
    m = mask(num)
    return m * (Lt @ (m * u))


def residual(Lt, num: Numbering, u, f) -> np.ndarray:
    """r = f - L~ u over unknowns."""
    m = mask(num)
    return m * (f - Lt @ (m * u))


class GS:
    """Multicolour Gauss-Seidel in class steps (vertices, edges c0..1, faces
    c0..2, volumes c0..3); within a step all selected nodes update
    simultaneously by eq. iteration-scheme with an IEEE division."""

    def __init__(self, Lt, num: Numbering):
        self.num = num
        m = sp.diags(mask(num))
        Lm = (m @ Lt @ m).tocsr()
        self.diag = Lm.diagonal().copy()
        self.off = (Lm - sp.diags(self.diag)).tocsr()
        self.steps = [s for s in num.gs_steps() if len(s)]
        self.offrows = [self.off[s] for s in self.steps]

    def sweep(self, u, f, n=1):
        u = u * mask(self.num)
        for _ in range(n):
            for s, O in zip(self.steps, self.offrows):
                u[s] = (f[s] - O @ u) / self.diag[s]
        return u

    def sweep_lex(self, u, f, n=1):
        """The paper's hybrid smoother with a LEXICOGRAPHIC volume ordering
        (PAPER.md:1317-1330): the lower-primitive class steps as in `sweep`
        (R13), then the volume nodes of every macro one at a time,
        west to east, south to north, bottom to top (i fastest, then j, then k
        -- the order of the volume ids, `interior_ijk`), each from the newest
        values (eq. iteration-scheme, IEEE division).  Volume nodes of
        different macros never couple, so the macro order is immaterial."""
        u = u * mask(self.num)
        base_v = self.num.base_v
        lp = [(s, O) for s, O in zip(self.steps, self.offrows) if s[0] < base_v]
        ip, ix, dv = self.off.indptr, self.off.indices, self.off.data
        for _ in range(n):
            for s, O in lp:
                u[s] = (f[s] - O @ u) / self.diag[s]
            for g in range(base_v, self.num.n_total):
                a, b = ip[g], ip[g + 1]
                u[g] = (f[g] - dv[a:b] @ u[ix[a:b]]) / self.diag[g]
        return u


def prolongation(mesh, num_c: Numbering, num_f: Numbering, masked=True) -> sp.csr_matrix:
    """P: coarse (N/2) -> fine (N), index-space linear interpolation per macro:
    all-even fine node (v) takes coarse v/2; otherwise 1/2 from each endpoint of
    its unique coarse edge (v -+ d)/2.  Rows/cols restricted to unknowns."""
    Nf = num_f.N
    lat = lattice_ijk(Nf)
    par = lat % 2
    rows, cols, vals = [], [], []
    for T in range(mesh.nt):
        gf = num_f.gids(T, lat)
        even = np.all(par == 0, axis=1)
        rows.append(gf[even])
        cols.append(num_c.gids(T, lat[even] // 2))
        vals.append(np.ones(even.sum()))
        for p, d in _PARITY_DIR.items():
            sel = np.all(par == np.array(p), axis=1)
            if not sel.any():
                continue
            v = lat[sel]
            d = np.array(d)
            for sgn in (-1, 1):
                rows.append(gf[sel])
                cols.append(num_c.gids(T, (v + sgn * d) // 2))
                vals.append(np.full(sel.sum(), 0.5))
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = np.concatenate(vals)
    # each (fine, coarse) pair appears once per macro containing the fine node:
    # keep one copy
    key = r * num_c.n_total + c
    _, first = np.unique(key, return_index=True)
    P = sp.coo_matrix((v[first], (r[first], c[first])), shape=(num_f.n_total, num_c.n_total)).tocsr()
    if not masked:
        return P
    mf = sp.diags(mask(num_f))
    mc = sp.diags(mask(num_c))
    return (mf @ P @ mc).tocsr()


def cg(A, b, iters: int, x0=None):
    """Plain conjugate gradients (Hestenes-Stiefel), fixed iteration count."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - A @ x
    p = r.copy()
    rr = r @ r
    for _ in range(iters):
        if rr == 0.0:
            break
        Ap = A @ p
        alpha = rr / (p @ Ap)
        x += alpha * p
        r -= alpha * Ap
        rr_new = r @ r
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x


class Hierarchy:
    """Levels L_coarse..L_max with L~ per level, GS, P; V(nu1,nu2) cycle."""

    def __init__(self, mesh, L_max: int, L_coarse: int = 2, q: int = 2, method="lsqp", j=2):
        from .surrogate import surrogate_operator
        self.mesh = mesh
        self.L_max, self.L_coarse = L_max, L_coarse
        self.num, self.Lt, self.L, self.gs, self.P = {}, {}, {}, {}, {}
        for L in range(L_coarse, L_max + 1):
            num = Numbering(mesh, 2 ** L)
            Lt, Lx, _ = surrogate_operator(mesh, L, q, method, j, num=num)
            self.num[L], self.Lt[L], self.L[L] = num, Lt, Lx
            self.gs[L] = GS(Lt, num)
            if L > L_coarse:
                self.P[L] = prolongation(mesh, self.num[L - 1], num)
        m = sp.diags(mask(self.num[L_coarse]))
        self.A_coarse = (m @ self.L[L_coarse] @ m).tocsr()

    def _res_op(self, L, dd):
        # double discretisation: the surrogate L~ smooths,
        # the exact operator L computes the residuals
        return self.L[L] if dd else self.Lt[L]

    def vcycle(self, L, u, f, nu1=3, nu2=3, cg_iters=50, dd=False, lex=False):
        """lex: the paper's lexicographic hybrid smoother (GS.sweep_lex,
        PAPER.md:1317-1330) instead of the 4-colour one."""
        if L == self.L_coarse:
            m = mask(self.num[L])
            return m * cg(self.A_coarse, m * f, cg_iters)
        smooth = self.gs[L].sweep_lex if lex else self.gs[L].sweep
        u = smooth(u, f, nu1)
        r = residual(self._res_op(L, dd), self.num[L], u, f)
        fc = self.P[L].T @ r
        uc = self.vcycle(L - 1, np.zeros_like(fc), fc, nu1, nu2, cg_iters, dd, lex)
        u = u + self.P[L] @ uc
        return smooth(u, f, nu2)

    def solve(self, u, f, n_cycles, nu1=3, nu2=3, cg_iters=50, dd=False, lex=False):
        """n_cycles V(nu1, nu2) cycles; history = ||f - A u||_2 after each, A
        the residual operator (L~, or L with double discretisation)."""
        L = self.L_max
        A = self._res_op(L, dd)
        hist = [np.linalg.norm(residual(A, self.num[L], u, f))]
        for _ in range(n_cycles):
            u = self.vcycle(L, u, f, nu1, nu2, cg_iters, dd, lex)
            hist.append(np.linalg.norm(residual(A, self.num[L], u, f)))
        return u, np.array(hist)
