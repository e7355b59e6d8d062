"""Python/scipy restatement of the reference stencil builder -- TEST
INFRASTRUCTURE (the checker of the native builder), never imported by the
product package.

Follows reference pkg/src/kmf/geometry.py:315-570 (k-nearest and radius
neighbour rows, the visibility filter, the CSR assembly and deficiency
scan, the widening pass of build_stencils :453-518) on scipy's cKDTree,
whose tie behaviour at the k-th distance defines the reference stencils.
The product's builder (paper_2108_07031_b200/builder.py + csrc/kmf_build.cpp)
must equal it bit for bit (tests/test_builder.py); both share the host
boundary-frame construction (builder.frames, geometry.py:573-646).
"""

from __future__ import annotations

import numpy as np
from scipy.spatial import cKDTree

from paper_2108_07031_b200.builder import Parts, frames
from paper_2108_07031_b200.geometry import (
    DEGENERACY_FACTOR,
    INTERIOR,
    KNN_CAP,
    KNN_DEFAULT,
    RADIUS_MIN_NEIGHBORS,
    WALL,
    Connectivity,
    PointCloud,
    StencilDeficiencyError,
    StencilSet,
    _owners,
    _select,
)


def _rows_to_lists(ptr: np.ndarray, idx: np.ndarray):
    return [idx[ptr[i]:ptr[i + 1]] for i in range(ptr.shape[0] - 1)]


def knn_lists(x, y, k, subset=None):
    """Tie-inclusive k-nearest neighbours, self excluded, ascending index.

    Semantics of geometry.py:315-346: every point at distance <= the k-th
    neighbour's distance (self counted as the 0th) is kept; when all padded
    candidates tie with the cut the query widens until the plateau ends.
    Returns a list of int64 arrays.
    """
    n = x.shape[0]
    pts = np.column_stack([x, y])
    tree = cKDTree(pts)
    query = np.arange(n) if subset is None else np.asarray(subset, dtype=np.int64)
    k_eff = min(k + 1, n)
    pad = min(k_eff + 8, n)
    dist, nbr = tree.query(pts[query], k=pad)
    dist = np.atleast_2d(dist).reshape(query.size, pad)
    nbr = np.atleast_2d(nbr).reshape(query.size, pad)
    keep = dist <= dist[:, k_eff - 1:k_eff]
    plateau = np.flatnonzero(keep.all(axis=1)) if pad < n else np.empty(0, dtype=np.int64)
    keep &= nbr != query[:, None]
    cnt = keep.sum(axis=1)
    rows = np.where(keep, nbr, n)
    rows.sort(axis=1)
    out = [rows[r, :cnt[r]].astype(np.int64) for r in range(query.size)]
    for r in plateau:
        qi = int(query[r])
        width = pad
        while True:
            width = min(width * 2, n)
            d, nb = tree.query(pts[qi], k=width)
            sel = d <= d[k_eff - 1]
            if width == n or not sel.all():
                break
        cand = nb[sel]
        out[r] = np.sort(cand[cand != qi]).astype(np.int64)
    return out


def radius_lists(x, y, eps):
    """All neighbours with squared distance < eps^2, ascending (geometry.py:349-374)."""
    n = x.shape[0]
    tree = cKDTree(np.column_stack([x, y]))
    cands = tree.query_ball_point(np.column_stack([x, y]), r=eps * (1.0 + 1e-9))
    eps2 = eps * eps
    out = []
    for i in range(n):
        c = np.asarray(cands[i], dtype=np.int64)
        d2 = (x[c] - x[i]) ** 2 + (y[c] - y[i]) ** 2
        out.append(np.sort(c[(d2 < eps2) & (c != i)]))
    return out


def visibility_filter(cloud: PointCloud, lists, owners=None):
    """Drop edges that cut through the body behind the wall (geometry.py:396-450).

    An edge survives when each of its 1/4, 1/2, 3/4 sample points is either
    more than two local wall spacings from the nearest wall point or lies no
    deeper behind that point's tangent plane than the tolerance
    min(0.2 spacing, 0.45 local thickness).
    """
    wall = np.flatnonzero(cloud.flag == WALL)
    if wall.size < 2:
        return lists
    wx, wy = cloud.x[wall], cloud.y[wall]
    wnx, wny = cloud.nx[wall], cloud.ny[wall]
    wpts = np.column_stack([wx, wy])
    tree = cKDTree(wpts)
    spacing = tree.query(wpts, k=2)[0][:, 1]
    d16, c16 = tree.query(wpts, k=min(16, wall.size))
    facing = wnx[:, None] * wnx[c16] + wny[:, None] * wny[c16] < -0.5
    thick = np.where(facing, d16, np.inf).min(axis=1)
    tol = np.minimum(0.2 * spacing, 0.45 * thick)

    sizes = np.fromiter((len(v) for v in lists), dtype=np.int64, count=len(lists))
    if not sizes.sum():
        return lists
    nbr = np.concatenate(lists).astype(np.int64)
    base = np.arange(len(lists)) if owners is None else np.asarray(owners)
    own = np.repeat(base, sizes)
    ok = np.ones(nbr.shape[0], dtype=bool)
    x0, y0 = cloud.x[own], cloud.y[own]
    ddx, ddy = cloud.x[nbr] - x0, cloud.y[nbr] - y0
    for frac in (0.25, 0.5, 0.75):
        px = x0 + frac * ddx
        py = y0 + frac * ddy
        dist, near = tree.query(np.column_stack([px, py]))
        depth = (px - wx[near]) * wnx[near] + (py - wy[near]) * wny[near]
        ok &= (dist > 2.0 * spacing[near]) | (depth > -tol[near])
    if ok.all():
        return lists
    ptr = np.concatenate([[0], np.cumsum(sizes)])
    return [nbr[ptr[i]:ptr[i + 1]][ok[ptr[i]:ptr[i + 1]]] for i in range(len(lists))]



def _csr(cloud: PointCloud, lists) -> StencilSet:
    sizes = np.fromiter((len(v) for v in lists), dtype=np.int64, count=len(lists))
    ptr = np.concatenate([[0], np.cumsum(sizes)])
    idx = np.concatenate(lists).astype(np.int64) if ptr[-1] else np.empty(0, dtype=np.int64)
    own = np.repeat(np.arange(len(lists)), sizes)
    return StencilSet(ptr=ptr, idx=idx, dx=cloud.x[idx] - cloud.x[own], dy=cloud.y[idx] - cloud.y[own])


def _assemble(cloud: PointCloud, lists) -> Parts:
    full = _csr(cloud, lists)
    n = cloud.n_points
    own = _owners(full.ptr)
    length = np.hypot(full.dx, full.dy)
    d_min = np.full(n, np.inf)
    np.minimum.at(d_min, own, length)
    d_mean = np.bincount(own, weights=length, minlength=n) / np.maximum(full.counts(), 1)
    split = {
        "x+": _select(full, full.dx <= 0.0),
        "x-": _select(full, full.dx >= 0.0),
        "y+": _select(full, full.dy <= 0.0),
        "y-": _select(full, full.dy >= 0.0),
    }
    failures = []
    interior = cloud.flag == INTERIOR
    thresh = DEGENERACY_FACTOR * d_mean ** 4
    cnt = full.counts()
    for i in np.flatnonzero(cnt < 3):
        failures.append((int(i), "full", f"only {cnt[i]} neighbors"))
    for i in np.flatnonzero((cnt >= 3) & (np.abs(full.det) < thresh)):
        failures.append((int(i), "full", f"degenerate LS matrix (det {full.det[i]:.3e})"))
    for kind, s in split.items():
        sc = s.counts()
        for i in np.flatnonzero(interior & (sc < 3)):
            failures.append((int(i), kind, f"only {sc[i]} neighbors"))
        for i in np.flatnonzero(interior & (sc >= 3) & (np.abs(s.det) < thresh)):
            failures.append((int(i), kind, f"degenerate LS matrix (det {s.det[i]:.3e})"))
    wall_frame = frames(cloud, full, thresh, cloud.wall, +1.0, failures)
    outer_frame = frames(cloud, full, thresh, cloud.outer, -1.0, failures)
    return Parts(full, split, d_min, d_mean, wall_frame, outer_frame, failures)



def build_stencils_ref(cloud: PointCloud, epsilon: float | None = None, k: int | None = None) -> Connectivity:
    """geometry.py:453-518 restated: full, split and boundary-frame stencils
    with cached sums; StencilDeficiencyError (after widening failing points
    to k=25) exactly where the reference raises it."""
    cloud.validate()
    if epsilon is not None and k is not None:
        raise ValueError("give either epsilon or k, not both")
    if epsilon is not None and epsilon <= 0.0:
        raise ValueError("epsilon must be positive")
    if k is not None and k < 6:
        raise ValueError("k must be at least 6")
    if epsilon is not None:
        lists = radius_lists(cloud.x, cloud.y, epsilon)
        thin = [i for i, v in enumerate(lists) if len(v) < RADIUS_MIN_NEIGHBORS]
        if thin:
            for i, row in zip(thin, knn_lists(cloud.x, cloud.y, KNN_DEFAULT, thin)):
                lists[i] = row
    else:
        lists = knn_lists(cloud.x, cloud.y, min(k or KNN_DEFAULT, KNN_CAP))
    lists = visibility_filter(cloud, lists)
    parts = _assemble(cloud, lists)
    if parts.failures:
        grow = sorted({i for i, _, _ in parts.failures if len(lists[i]) < KNN_CAP})
        if grow:
            rows = visibility_filter(cloud, knn_lists(cloud.x, cloud.y, KNN_CAP, grow), owners=grow)
            for i, row in zip(grow, rows):
                lists[i] = row
            parts = _assemble(cloud, lists)
    if parts.failures:
        raise StencilDeficiencyError(parts.failures)
    interior = cloud.flag == INTERIOR
    det_safe = {kind: np.where(interior, s.det, 1.0) for kind, s in parts.split.items()}
    return Connectivity(
        cloud=cloud, full=parts.full, split=parts.split, d_min=parts.d_min, d_mean=parts.d_mean,
        wall_frame=parts.wall_frame, outer_frame=parts.outer_frame, det_safe=det_safe,
    )
