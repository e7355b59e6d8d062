"""Native stencil builder: ``build_stencils`` at 10M/40M.

Same result, bit for bit, as the reference builder (geometry.py:453-518;
its scipy restatement oracle/builder_ref.py is the tests' checker); the
heavy loops run in ``libkmf_build.so`` (csrc/kmf_build.cpp, C++/OpenMP, C
ABI in include/kmf_build.h):

* tie-inclusive kNN rows (geometry.py:315-346) and radius rows
  (geometry.py:349-374) from a 2-d tree;
* the visibility filter's edge loop (geometry.py:396-450) -- the wall
  statistics (spacing, thickness, tolerance) stay on cKDTree here because
  the 16-nearest tie order is part of their definition;
* CSR offsets, full and sign-split LS sums, d_min / d_mean
  (geometry.py:375-393, 532-560).

The deficiency scan, boundary frames (``frames``, geometry.py:573-646) and
the widening pass are the host builder's own code.  Split families are never materialised: their sums,
determinants and counts come from the native pass and their CSR arrays are
derived from the full stencil on first access (``SplitView``), which keeps
the host footprint at 40M points to the full stencil (~14 GB).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np
from scipy.spatial import cKDTree

from . import geometry as G

LIB_PATH = Path(__file__).resolve().parent / "libkmf_build.so"
_lib = None

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH.name} is not built (make -C paper_2108_07031_b200/csrc)")
        L = C.CDLL(str(LIB_PATH))
        L.kmfb_threads.restype = C.c_int
        L.kmfb_set_threads.restype = C.c_int
        L.kmfb_set_threads.argtypes = [C.c_int]
        L.kmfb_knn.argtypes = [C.c_int64, _dp, _dp, C.c_int, C.c_int64, _i64p, _i64p, _i64p, _i64p]
        L.kmfb_visibility.argtypes = [C.c_int64, _dp, _dp, C.c_int64, _i64p, _dp, _dp, _dp, _dp, C.c_int64, _i64p,
                                      _i64p, _i64p, _u8p, _i64p]
        L.kmfb_assemble.argtypes = [C.c_int64, _dp, _dp, _i64p, _i64p, _dp, _dp, _dp, _dp, _dp, _dp, _i64p]
        L.kmfb_radius.argtypes = [C.c_int64, _dp, _dp, C.c_double, _i64p, _i64p, _i64p]
        for f in (L.kmfb_knn, L.kmfb_visibility, L.kmfb_assemble, L.kmfb_radius):
            f.restype = C.c_int
        _lib = L
    return _lib


def available() -> bool:
    try:
        lib()
        return True
    except (RuntimeError, OSError):
        return False


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(_i64p)


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"{what}: invalid argument (code {rc})")


# ------------------------------------------------------------------ pieces


def _frame_family(rows_idx, rows_dt, rows_dn) -> StencilSet:
    cnt = np.array([r.shape[0] for r in rows_idx], dtype=np.int64)
    ptr = np.concatenate([[0], np.cumsum(cnt)])
    if ptr[-1]:
        idx = np.concatenate(rows_idx).astype(np.int64)
        dt = np.concatenate(rows_dt)
        dn = np.concatenate(rows_dn)
    else:
        idx, dt, dn = np.empty(0, dtype=np.int64), np.empty(0), np.empty(0)
    return G.StencilSet(ptr=ptr, idx=idx, dx=dt, dy=dn)


def frames(cloud, full, thresh, points, side, failures):
    """Rotated boundary stencils for one class (geometry.py:573-646).

    ``side`` +1 keeps dn >= 0 for the one-sided normal family (wall: fluid
    along +n), -1 keeps dn <= 0 (outer).  A tangent-split family that is
    too thin or degenerate falls back to the full stencil.  The usability
    test sums with np.sum exactly as the reference does (its result decides
    fallbacks, so its summation order is part of the bit-exact contract).
    """
    if points.size == 0:
        return None
    nx, ny = cloud.nx[points], cloud.ny[points]
    tx, ty = -ny, nx
    label = "wall" if side > 0 else "outer"
    fam = {"tp": ([], [], []), "tm": ([], [], []), "nr": ([], [], [])}
    fallback = {}

    def usable(dts, dns, limit):
        stt = float(np.sum(dts ** 2))
        snn = float(np.sum(dns ** 2))
        stn = float(np.sum(dts * dns))
        return dts.shape[0] >= 3 and abs(stt * snn - stn * stn) >= limit

    for loc, gi in enumerate(points):
        lo, hi = full.ptr[gi], full.ptr[gi + 1]
        nb = full.idx[lo:hi]
        ex, ey = full.dx[lo:hi], full.dy[lo:hi]
        dt = ex * tx[loc] + ey * ty[loc]
        dn = ex * nx[loc] + ey * ny[loc]
        lim = thresh[gi]
        every = np.ones(dt.shape[0], dtype=bool)
        tag = ""
        for key, mask, mark in (("tp", dt <= 0.0, "+"), ("tm", dt >= 0.0, "-")):
            if not usable(dt[mask], dn[mask], lim):
                mask = every
                tag += mark
            fam[key][0].append(nb[mask])
            fam[key][1].append(dt[mask])
            fam[key][2].append(dn[mask])
        if tag:
            fallback[int(gi)] = tag
        nmask = dn >= 0.0 if side > 0 else dn <= 0.0
        if not usable(dt[nmask], dn[nmask], lim):
            failures.append((int(gi), f"{label}-normal", f"unusable one-sided stencil ({int(nmask.sum())} pts)"))
        fam["nr"][0].append(nb[nmask])
        fam["nr"][1].append(dt[nmask])
        fam["nr"][2].append(dn[nmask])
    return G.FrameStencils(
        points=points, tx=tx, ty=ty, nx=nx, ny=ny,
        tplus=_frame_family(*fam["tp"]), tminus=_frame_family(*fam["tm"]),
        normal=_frame_family(*fam["nr"]), fallback=fallback,
    )


@dataclass
class Parts:
    full: G.StencilSet
    split: dict
    d_min: np.ndarray
    d_mean: np.ndarray
    wall_frame: G.FrameStencils | None
    outer_frame: G.FrameStencils | None
    failures: list


def radius_csr(cloud: G.PointCloud, eps: float):
    """geometry.py:349-374 rows as CSR (ptr, idx int64)."""
    x, y = np.ascontiguousarray(cloud.x), np.ascontiguousarray(cloud.y)
    n = x.shape[0]
    counts = np.zeros(n, dtype=np.int64)
    L = lib()
    _check(L.kmfb_radius(n, _d(x), _d(y), float(eps), _i(counts), None, None), "kmfb_radius")
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    idx = np.empty(int(ptr[-1]), dtype=np.int64)
    _check(L.kmfb_radius(n, _d(x), _d(y), float(eps), _i(counts), _i(ptr), _i(idx)), "kmfb_radius")
    return ptr, idx



def knn_csr(cloud: G.PointCloud, k: int, subset=None):
    """geometry.py:315-346 rows as CSR (ptr, idx int64)."""
    x, y = np.ascontiguousarray(cloud.x), np.ascontiguousarray(cloud.y)
    n = x.shape[0]
    q = None if subset is None else np.ascontiguousarray(subset, dtype=np.int64)
    nq = n if q is None else q.shape[0]
    counts = np.zeros(nq, dtype=np.int64)
    L = lib()
    _check(L.kmfb_knn(n, _d(x), _d(y), int(k), nq, _i(q), _i(counts), None, None), "kmfb_knn")
    ptr = np.zeros(nq + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    idx = np.empty(int(ptr[-1]), dtype=np.int64)
    _check(L.kmfb_knn(n, _d(x), _d(y), int(k), nq, _i(q), _i(counts), _i(ptr), _i(idx)), "kmfb_knn")
    return ptr, idx


def wall_statistics(cloud: G.PointCloud):
    """spacing and tolerance of every wall point (geometry.py:418-431), on
    cKDTree like the reference (its tie order defines the 16-neighbour set)."""
    w = np.flatnonzero(cloud.flag == G.WALL)
    if w.size < 2:
        return w, None, None
    wpts = np.column_stack([cloud.x[w], cloud.y[w]])
    wnx, wny = cloud.nx[w], cloud.ny[w]
    tree = cKDTree(wpts)
    spacing = tree.query(wpts, k=2)[0][:, 1]
    d16, c16 = tree.query(wpts, k=min(16, w.size))
    facing = wnx[:, None] * wnx[c16] + wny[:, None] * wny[c16] < -0.5
    thick = np.where(facing, d16, np.inf).min(axis=1)
    return w, spacing, np.minimum(0.2 * spacing, 0.45 * thick)


def visibility_keep(cloud: G.PointCloud, ptr, idx, owners=None, wall_stats=None):
    """geometry.py:396-450 edge mask (1 keep) for CSR rows owned by owners."""
    w, spacing, tol = wall_stats if wall_stats is not None else wall_statistics(cloud)
    keep = np.ones(idx.shape[0], dtype=np.uint8)
    if spacing is None or idx.shape[0] == 0:
        return keep.astype(bool)
    x, y = np.ascontiguousarray(cloud.x), np.ascontiguousarray(cloud.y)
    wnx, wny = np.ascontiguousarray(cloud.nx[w]), np.ascontiguousarray(cloud.ny[w])
    own = None if owners is None else np.ascontiguousarray(owners, dtype=np.int64)
    amb = C.c_int64(0)
    _check(lib().kmfb_visibility(x.shape[0], _d(x), _d(y), w.shape[0], _i(np.ascontiguousarray(w)), _d(wnx), _d(wny),
                                 _d(np.ascontiguousarray(spacing)), _d(np.ascontiguousarray(tol)), ptr.shape[0] - 1,
                                 _i(own), _i(ptr), _i(idx), keep.ctypes.data_as(_u8p), C.byref(amb)),
           "kmfb_visibility")
    if amb.value:
        # nearest-wall ties with disagreeing outcomes: settle these edges on
        # cKDTree, whose first-found tie order is the reference's
        und = np.flatnonzero(keep == 2)
        own_e = np.repeat(np.arange(ptr.shape[0] - 1) if own is None else own, np.diff(ptr))[und]
        tree = cKDTree(np.column_stack([cloud.x[w], cloud.y[w]]))
        ok = np.ones(und.shape[0], dtype=bool)
        x0, y0 = cloud.x[own_e], cloud.y[own_e]
        ddx, ddy = cloud.x[idx[und]] - x0, cloud.y[idx[und]] - y0
        for frac in (0.25, 0.5, 0.75):
            px, py = x0 + frac * ddx, y0 + frac * ddy
            dist, near = tree.query(np.column_stack([px, py]))
            depth = (px - cloud.x[w][near]) * wnx[near] + (py - cloud.y[w][near]) * wny[near]
            ok &= (dist > 2.0 * spacing[near]) | (depth > -tol[near])
        keep[und] = ok
    return keep.astype(bool)


def _compress(ptr, idx, keep):
    if keep.all():
        return ptr, idx
    own = np.repeat(np.arange(ptr.shape[0] - 1), np.diff(ptr))
    cnt = np.bincount(own[keep], minlength=ptr.shape[0] - 1)
    nptr = np.zeros_like(ptr)
    np.cumsum(cnt, out=nptr[1:])
    return nptr, idx[keep]


class SplitView:
    """Sign-split family of the full stencil (geometry.py:387-393) with its
    sums from the native pass; ptr/idx/dx/dy are derived on first access."""

    def __init__(self, full: G.StencilSet, family: int, counts, sxx, sxy, syy, det):
        self._full, self._family, self._counts = full, family, counts
        self.sxx, self.sxy, self.syy, self.det = sxx, sxy, syy, det
        self._csr = None

    def mask(self) -> np.ndarray:
        f = self._full
        return (f.dx <= 0.0, f.dx >= 0.0, f.dy <= 0.0, f.dy >= 0.0)[self._family]

    def _materialise(self):
        if self._csr is None:
            m = self.mask()
            ptr = np.zeros(self._counts.shape[0] + 1, dtype=np.int64)
            np.cumsum(self._counts, out=ptr[1:])
            self._csr = (ptr, self._full.idx[m], self._full.dx[m], self._full.dy[m])
        return self._csr

    ptr = property(lambda self: self._materialise()[0])
    idx = property(lambda self: self._materialise()[1])
    dx = property(lambda self: self._materialise()[2])
    dy = property(lambda self: self._materialise()[3])

    @property
    def n_owners(self) -> int:
        return self._counts.shape[0]

    def counts(self) -> np.ndarray:
        return self._counts

    def neighbors(self, i: int):
        p = self.ptr
        return self.idx[p[i]:p[i + 1]]

    def offsets(self, i: int):
        p = self.ptr
        return self.dx[p[i]:p[i + 1]], self.dy[p[i]:p[i + 1]]


def assemble(cloud: G.PointCloud, ptr, idx) -> Parts:
    """geometry.py:532-570 on the native sums; same failure list, same order."""
    n = cloud.n_points
    x, y = np.ascontiguousarray(cloud.x), np.ascontiguousarray(cloud.y)
    m = idx.shape[0]
    dx, dy = np.empty(m), np.empty(m)
    sums = np.empty((4, n))
    d_min, d_mean = np.empty(n), np.empty(n)
    ssum = np.empty((4, 4, n))
    scnt = np.empty((4, n), dtype=np.int64)
    _check(lib().kmfb_assemble(n, _d(x), _d(y), _i(ptr), _i(idx), _d(dx), _d(dy), _d(sums), _d(d_min), _d(d_mean),
                               _d(ssum), _i(scnt)), "kmfb_assemble")
    full = G.StencilSet(ptr=ptr, idx=idx, dx=dx, dy=dy, sxx=sums[0], sxy=sums[1], syy=sums[2], det=sums[3])
    split = {kind: SplitView(full, f, scnt[f], *ssum[f]) for f, kind in enumerate(G.SPLIT_KINDS)}
    failures = []
    interior = cloud.flag == G.INTERIOR
    thresh = G.DEGENERACY_FACTOR * d_mean ** 4
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


def _splice(ptr, idx, rows_of: np.ndarray, rptr, ridx):
    """Replace the rows `rows_of` (ascending, few) of a CSR by the rows of (rptr, ridx)."""
    n = ptr.shape[0] - 1
    cnt = np.diff(ptr)
    cnt[rows_of] = np.diff(rptr)
    nptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=nptr[1:])
    nidx = np.empty(int(nptr[-1]), dtype=np.int64)
    prev = 0  # first row not yet copied
    for r, i in enumerate(rows_of):
        nidx[nptr[prev]:nptr[i]] = idx[ptr[prev]:ptr[i]]  # untouched run [prev, i)
        nidx[nptr[i]:nptr[i + 1]] = ridx[rptr[r]:rptr[r + 1]]
        prev = i + 1
    nidx[nptr[prev]:] = idx[ptr[prev]:]
    return nptr, nidx


def build_stencils_native(cloud: G.PointCloud, k: int | None = None, epsilon: float | None = None) -> G.Connectivity:
    """geometry.py:453-518 with the native loops, k-nearest or radius mode
    (radius rows with fewer than 8 neighbours take their 15 nearest,
    geometry.py:480-486)."""
    cloud.validate()
    if epsilon is not None and k is not None:
        raise ValueError("give either epsilon or k, not both")
    if epsilon is not None and epsilon <= 0.0:
        raise ValueError("epsilon must be positive")
    if k is not None and k < 6:
        raise ValueError("k must be at least 6")
    ws = wall_statistics(cloud)
    if epsilon is not None:
        ptr, idx = radius_csr(cloud, epsilon)
        thin = np.flatnonzero(np.diff(ptr) < G.RADIUS_MIN_NEIGHBORS).astype(np.int64)
        if thin.size:
            tptr, tidx = knn_csr(cloud, G.KNN_DEFAULT, thin)
            ptr, idx = _splice(ptr, idx, thin, tptr, tidx)
    else:
        ptr, idx = knn_csr(cloud, min(k or G.KNN_DEFAULT, G.KNN_CAP))
    ptr, idx = _compress(ptr, idx, visibility_keep(cloud, ptr, idx, wall_stats=ws))
    parts = assemble(cloud, ptr, idx)
    if parts.failures:
        cnt = np.diff(ptr)
        grow = np.array(sorted({i for i, _, _ in parts.failures if cnt[i] < G.KNN_CAP}), dtype=np.int64)
        if grow.size:
            rptr, ridx = knn_csr(cloud, G.KNN_CAP, grow)
            rptr, ridx = _compress(rptr, ridx, visibility_keep(cloud, rptr, ridx, owners=grow, wall_stats=ws))
            ptr, idx = _splice(ptr, idx, grow, rptr, ridx)
            parts = assemble(cloud, ptr, idx)
    if parts.failures:
        raise G.StencilDeficiencyError(parts.failures)
    interior = cloud.flag == G.INTERIOR
    det_safe = {kind: np.where(interior, s.det, 1.0) for kind, s in parts.split.items()}
    return G.Connectivity(cloud=cloud, full=parts.full, split=parts.split, d_min=parts.d_min, d_mean=parts.d_mean,
                          wall_frame=parts.wall_frame, outer_frame=parts.outer_frame, det_safe=det_safe)
