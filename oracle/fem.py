"""Oracle FEM: local stiffness, global Galerkin matrix, node-wise stencils.

PAPER.md:183-193, 265-291 (Galerkin P1, L_l u_l = f_l, (L_l)_IJ = a_l(phi_I,
phi_J)); PAPER.md:385-394 (node stencil = sum over the 24 adjacent fine tets
of their local stiffness matrices); PAPER.md:380-384 (affine macro => constant
stencil, 2^-l scaling).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .geometry import (DIRS, MC, Numbering, incident_kuhn_tets, kuhn_tets,
                       lattice_ijk, node_coords)


def local_stiffness(P: np.ndarray) -> np.ndarray:
    """K[a][b] = |T| grad(lambda_a) . grad(lambda_b) for tets P [...,4,3]
    (a(u,v) = <grad u, grad v> on P1)."""
    P = np.asarray(P, dtype=np.float64)
    E = np.stack([P[..., 1, :] - P[..., 0, :], P[..., 2, :] - P[..., 0, :],
                  P[..., 3, :] - P[..., 0, :]], axis=-1)          # columns = edges
    det = np.linalg.det(E)
    Einv = np.linalg.inv(E)                                        # rows = grad lambda_1..3
    g = np.concatenate([-Einv.sum(axis=-2, keepdims=True), Einv], axis=-2)  # [...,4,3]
    vol = np.abs(det) / 6.0
    return vol[..., None, None] * np.einsum("...ad,...bd->...ab", g, g)


def macro_element_data(mesh, T: int, N: int, blended=True):
    """Fine tets of macro T: (lattice index [N^3,4], lattice ijk, K [N^3,4,4])."""
    lat = lattice_ijk(N)
    tets = kuhn_tets(N)                                  # [n,4,3]
    # lattice position index for gathering coordinates
    key = lambda a: (a[..., 2] * (N + 1) + a[..., 1]) * (N + 1) + a[..., 0]
    lut = -np.ones((N + 1) ** 3, dtype=np.int64)
    lut[key(lat)] = np.arange(len(lat))
    X = node_coords(mesh, T, lat, N, blended)
    li = lut[key(tets)]                                  # [n,4]
    K = local_stiffness(X[li])
    return li, lat, K


def assemble(mesh, N: int, num: Numbering | None = None, blended=True) -> sp.csr_matrix:
    """Global Galerkin matrix over ALL canonical nodes (no BC applied):
    L[I][J] = sum over fine tets T containing I,J of K_T[I][J]."""
    if num is None:
        num = Numbering(mesh, N)
    rows, cols, vals = [], [], []
    for T in range(mesh.nt):
        li, lat, K = macro_element_data(mesh, T, N, blended)
        g = num.gids(T, lat)[li]                          # [n,4]
        rows.append(np.repeat(g, 4, axis=1).ravel())
        cols.append(np.tile(g, (1, 4)).ravel())
        vals.append(K.reshape(len(g), 16).ravel())
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(num.n_total, num.n_total))
    return A.tocsr()


def apply_dirichlet(A: sp.csr_matrix, num: Numbering) -> sp.csr_matrix:
    """Restrict to unknowns: rows and columns of Dirichlet nodes zeroed
    (u = 0 on the boundary; R15)."""
    d = sp.diags(num.unknown_mask.astype(np.float64))
    B = (d @ A @ d).tocsr()
    B.eliminate_zeros()
    return B


def volume_stencils(mesh, T: int, ijk: np.ndarray, N: int, blended=True) -> np.ndarray:
    """Exact FEM node stencils s_w(I), w in DIRS order, for interior nodes
    `ijk` [n,3] of macro T: sum over the 24 incident fine tets
    (PAPER.md:385-394).  Node-wise on-the-fly assembly (paper's FEM)."""
    ijk = np.asarray(ijk, dtype=np.int64).reshape(-1, 3)
    out = np.zeros((len(ijk), 15))
    # the 24 incident tets of an interior node are translates of a fixed
    # pattern (relative offsets) -- build it once from the node (1,1,1)@N=4
    pat = incident_kuhn_tets(np.array([1, 1, 1]), 4)
    assert len(pat) == 24
    pat = np.stack(pat) - np.array([1, 1, 1])           # [24,4,3] relative
    dir_index = {tuple(d): w for w, d in enumerate(DIRS)}
    for t in range(24):
        verts = ijk[:, None, :] + pat[t][None, :, :]    # [n,4,3]
        P = np.stack([node_coords(mesh, T, verts[:, a], N, blended) for a in range(4)], axis=1)
        K = local_stiffness(P)                           # [n,4,4]
        a0 = int(np.nonzero(np.all(pat[t] == 0, axis=1))[0][0])   # position of node
        for b in range(4):
            w = dir_index[tuple(pat[t][b])]
            out[:, w] += K[:, a0, b]
    return out


def fem_row(mesh, num: Numbering, gid: int, blended=True, macros=None, locs=None) -> dict:
    """Row `gid` of the global FEM matrix (no BC) by node-wise assembly over
    every fine tet of every macro containing the node: {gid_J: value}.
    `macros` (optional) lists the candidate macros to search, ascending (a
    superset of those containing the node); the sum is the same.  `locs`
    (optional) gives the node's (macro, ijk) positions directly (e.g.
    `num.locate(gid)`), ascending macro order, instead of the search."""
    N = num.N
    row = {}
    if locs is None:
        lat = lattice_ijk(N)
        locs = []
        for T in (range(mesh.nt) if macros is None else macros):
            hit = np.nonzero(num.gids(T, lat) == gid)[0]
            if len(hit):
                locs.append((T, lat[hit[0]]))
    for T, ijk in locs:
        for tet in incident_kuhn_tets(ijk, N, inside_only=True):
            P = node_coords(mesh, T, tet, N, blended)
            K = local_stiffness(P)
            tg = num.gids(T, tet)
            a0 = int(np.nonzero(tg == gid)[0][0])
            for b in range(4):
                row[int(tg[b])] = row.get(int(tg[b]), 0.0) + K[a0, b]
    return row


def rhs_lumped(mesh, num: Numbering, func, blended=True) -> np.ndarray:
    """Lumped load vector f_I = func(x_I) * sum_{T ∋ I} |T|/4 over blended
    fine tets (R20; (f_l)_I = <f, phi_I>)."""
    N = num.N
    f = np.zeros(num.n_total)
    X = num.coords(blended)
    for T in range(mesh.nt):
        li, lat, K = macro_element_data(mesh, T, N, blended)
        P = node_coords(mesh, T, lat, N, blended)[li]     # [n,4,3]
        E = np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]], axis=-1)
        vol = np.abs(np.linalg.det(E)) / 6.0
        g = num.gids(T, lat)[li]
        np.add.at(f, g.ravel(), np.repeat(vol / 4.0, 4))
    f *= func(X[:, 0], X[:, 1], X[:, 2])
    f[num.dirichlet_mask] = 0.0
    return f


def stencil_from_matrix(A: sp.csr_matrix, num: Numbering, T: int, ijk: np.ndarray) -> np.ndarray:
    """Read interior-node stencils off a global matrix through the DIRS offsets."""
    ijk = np.asarray(ijk, dtype=np.int64).reshape(-1, 3)
    gI = num.gids(T, ijk)
    out = np.zeros((len(ijk), 15))
    for w, d in enumerate(DIRS):
        gJ = num.gids(T, ijk + d)
        out[:, w] = np.asarray(A[gI, gJ]).ravel()
    return out


__all__ = ["local_stiffness", "assemble", "apply_dirichlet", "volume_stencils",
           "fem_row", "rhs_lumped", "stencil_from_matrix", "MC"]
