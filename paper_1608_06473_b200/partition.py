"""Macro partition for the multi-rank path (SURVEY 8(e) "Partition"; host logic).

Recursive coordinate bisection of the radial columns of a spherical shell:
every macro tet is assigned to the column of its surface triangle (its vertices
projected onto the unit sphere span the triangle's three directions), the
columns are cut recursively along the axis of largest extent of their
direction centroids at the weighted median (weights = tets per column), so
every rank owns whole radial columns (cut faces are radial, no cut crosses a
prism) and the tet counts are balanced to within one column.  Meshes that are
not shells (e.g. a single tet) fall back to bisection of the tet centroids.
"""
from __future__ import annotations

import numpy as np


def _rcb(points: np.ndarray, weights: np.ndarray, idx: np.ndarray, nparts: int, first: int,
         out: np.ndarray) -> None:
    if nparts == 1:
        out[idx] = first
        return
    p = points[idx]
    axis = int(np.argmax(p.max(axis=0) - p.min(axis=0)))
    order = idx[np.lexsort((idx, p[:, axis]))]  # stable: ties by index
    left = nparts // 2
    w = np.cumsum(weights[order])
    target = w[-1] * left / nparts
    cut = int(np.searchsorted(w, target, side="left"))
    # the closer of the two candidate cuts to the target weight
    if cut < len(w) and cut > 0 and abs(w[cut - 1] - target) <= abs(w[cut] - target):
        cut -= 1
    cut = min(max(cut + 1, 1), len(order) - 1)
    _rcb(points, weights, order[:cut], left, first, out)
    _rcb(points, weights, order[cut:], nparts - left, first + left, out)


def radial_columns(vertices: np.ndarray, tets: np.ndarray):
    """Column id per tet (tets sharing their set of vertex directions), or None
    if the mesh is not a shell (some tet spans other than 3 directions)."""
    r = np.linalg.norm(vertices, axis=1)
    if np.any(r <= 0):
        return None
    d = np.round(vertices / r[:, None] * 1e9).astype(np.int64)
    _, dir_id = np.unique(d, axis=0, return_inverse=True)
    dir_id = dir_id.reshape(-1)
    td = np.sort(dir_id[tets], axis=1)
    # exactly 3 distinct directions per tet (a prism's tets)
    ndist = 1 + (td[:, 1] != td[:, 0]) + (td[:, 2] != td[:, 1]) + (td[:, 3] != td[:, 2])
    if np.any(ndist != 3):
        return None
    key = np.stack([td[:, 0], np.where(td[:, 1] != td[:, 0], td[:, 1], td[:, 2]), td[:, 3]], axis=1)
    _, col = np.unique(key, axis=0, return_inverse=True)
    return col.reshape(-1)


def partition_rcb(vertices, tets, nparts: int) -> np.ndarray:
    """owner[nt] in [0, nparts): recursive coordinate bisection of radial
    columns (shells) or of tet centroids (anything else)."""
    vertices = np.asarray(vertices, dtype=np.float64)
    tets = np.asarray(tets, dtype=np.int64)
    nt = tets.shape[0]
    if nparts < 1:
        raise ValueError("nparts must be >= 1")
    owner = np.zeros(nt, dtype=np.int32)
    if nparts == 1 or nt == 0:
        return owner
    col = radial_columns(vertices, tets)
    if col is None:
        pts = vertices[tets].mean(axis=1)
        w = np.ones(nt)
        part = np.zeros(nt, dtype=np.int32)
        _rcb(pts, w, np.arange(nt), min(nparts, nt), 0, part)
        return part
    ncol = int(col.max()) + 1
    u = vertices / np.linalg.norm(vertices, axis=1)[:, None]
    cen = np.zeros((ncol, 3))
    np.add.at(cen, col, u[tets].mean(axis=1))
    w = np.bincount(col, minlength=ncol).astype(np.float64)
    cen /= w[:, None]
    cpart = np.zeros(ncol, dtype=np.int32)
    _rcb(cen, w, np.arange(ncol), min(nparts, ncol), 0, cpart)
    return cpart[col]
