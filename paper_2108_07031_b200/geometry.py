"""Point clouds, stencils and the NACA 0012 cloud generator (host-side setup).

Drop-in for reference ``kmf.geometry``: same types and field names
(geometry.py:56-312), same builder semantics (geometry.py:315-646) and same
generator (geometry.py:652-770).  This is SETUP, not the timed hot path: it
runs once on the host before the device context is created.  Its outputs
must be bit-identical to the reference's (they fix the summation order of
every least-squares sum on the device), which tests/test_geometry_parity.py
checks against sha256 digests of the reference's own arrays
(tests/golden/*.json).  scipy's cKDTree is used for the neighbour queries
because its tie behaviour at the k-th distance defines the reference
stencils.

Beyond the reference the builder is vectorised (one batched kNN query and
row-sorted CSR assembly instead of per-point Python lists), which matters at
the 2.5M/10M-point configurations.
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
from scipy.spatial import cKDTree

INTERIOR, WALL, OUTER = 0, 1, 2
SPLIT_KINDS = ("x+", "x-", "y+", "y-")
DEGENERACY_FACTOR = 1e-12   # geometry.py:32
RADIUS_MIN_NEIGHBORS = 8    # geometry.py:35
KNN_DEFAULT = 15
KNN_CAP = 25
_BINARY_MAGIC = b"KMF1"


class StencilDeficiencyError(ValueError):
    """Unusable stencils; ``failures`` lists (point, kind, reason) (geometry.py:40-53)."""

    def __init__(self, failures):
        self.failures = list(failures)
        shown = "; ".join(f"point {p} [{k}]: {r}" for p, k, r in self.failures[:8])
        extra = "" if len(self.failures) <= 8 else f" (+{len(self.failures) - 8} more)"
        super().__init__(f"{len(self.failures)} deficient stencil(s): {shown}{extra}")


# --------------------------------------------------------------------- types


@dataclass
class PointCloud:
    """Scattered 2D points, class flags, boundary normals (geometry.py:56-112)."""

    x: np.ndarray
    y: np.ndarray
    flag: np.ndarray
    nx: np.ndarray
    ny: np.ndarray

    def __post_init__(self):
        self.x = np.asarray(self.x, dtype=np.float64)
        self.y = np.asarray(self.y, dtype=np.float64)
        self.flag = np.asarray(self.flag, dtype=np.int64)
        self.nx = np.asarray(self.nx, dtype=np.float64)
        self.ny = np.asarray(self.ny, dtype=np.float64)

    @property
    def n_points(self) -> int:
        return self.x.shape[0]

    @property
    def interior(self) -> np.ndarray:
        return np.flatnonzero(self.flag == INTERIOR)

    @property
    def wall(self) -> np.ndarray:
        return np.flatnonzero(self.flag == WALL)

    @property
    def outer(self) -> np.ndarray:
        return np.flatnonzero(self.flag == OUTER)

    def validate(self) -> None:
        n = self.n_points
        for name in ("x", "y", "nx", "ny"):
            a = getattr(self, name)
            if a.shape != (n,):
                raise ValueError(f"field {name} has shape {a.shape}, expected ({n},)")
            if not np.isfinite(a).all():
                raise ValueError(f"field {name} contains non-finite values")
        if self.flag.shape != (n,):
            raise ValueError("flag shape mismatch")
        bad = ~np.isin(self.flag, (INTERIOR, WALL, OUTER))
        if bad.any():
            raise ValueError(f"invalid class flag at point {np.flatnonzero(bad)[0]}")
        if not (self.flag == INTERIOR).any():
            raise ValueError("cloud has no interior points")
        bnd = np.flatnonzero(self.flag != INTERIOR)
        if bnd.size:
            length = np.hypot(self.nx[bnd], self.ny[bnd])
            off = np.flatnonzero(np.abs(length - 1.0) > 1e-12)
            if off.size:
                i = bnd[off[0]]
                raise ValueError(
                    f"boundary normal at point {i} is not unit length "
                    f"(|n| = {np.hypot(self.nx[i], self.ny[i]):.17g})"
                )


def _owners(ptr: np.ndarray) -> np.ndarray:
    return np.repeat(np.arange(ptr.shape[0] - 1), np.diff(ptr))


@dataclass
class StencilSet:
    """One CSR stencil family with cached LS sums (geometry.py:222-266).

    The sums are np.bincount accumulations in CSR order -- that order is the
    one the device kernels reproduce.
    """

    ptr: np.ndarray
    idx: np.ndarray
    dx: np.ndarray
    dy: np.ndarray
    sxx: np.ndarray = field(default=None)
    sxy: np.ndarray = field(default=None)
    syy: np.ndarray = field(default=None)
    det: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.sxx is None:
            self._refresh_sums()

    def _refresh_sums(self):
        m = self.ptr.shape[0] - 1
        own = _owners(self.ptr)
        self.sxx = np.bincount(own, weights=self.dx * self.dx, minlength=m)
        self.sxy = np.bincount(own, weights=self.dx * self.dy, minlength=m)
        self.syy = np.bincount(own, weights=self.dy * self.dy, minlength=m)
        self.det = self.sxx * self.syy - self.sxy * self.sxy

    @property
    def n_owners(self) -> int:
        return self.ptr.shape[0] - 1

    def counts(self) -> np.ndarray:
        return np.diff(self.ptr)

    def neighbors(self, i: int) -> np.ndarray:
        return self.idx[self.ptr[i]:self.ptr[i + 1]]

    def offsets(self, i: int):
        lo, hi = self.ptr[i], self.ptr[i + 1]
        return self.dx[lo:hi], self.dy[lo:hi]


@dataclass
class FrameStencils:
    """Tangent/normal-frame stencils of one boundary class (geometry.py:269-291)."""

    points: np.ndarray
    tx: np.ndarray
    ty: np.ndarray
    nx: np.ndarray
    ny: np.ndarray
    tplus: StencilSet
    tminus: StencilSet
    normal: StencilSet
    fallback: dict


@dataclass
class Connectivity:
    """Full + split + boundary-frame stencils (geometry.py:294-312)."""

    cloud: PointCloud
    full: StencilSet
    split: dict
    d_min: np.ndarray
    d_mean: np.ndarray
    wall_frame: FrameStencils | None = None
    outer_frame: FrameStencils | None = None
    det_safe: dict = field(default_factory=dict)

    def ls_matrix(self, i: int, kind: str = "full"):
        s = self.full if kind == "full" else self.split[kind]
        return s.sxx[i], s.sxy[i], s.syy[i], s.det[i]


# ---------------------------------------------------------------- cloud IO


def read_point_cloud(source) -> PointCloud:
    """Text or KMF1-binary grid from a path, bytes or file object (geometry.py:115-191)."""
    if isinstance(source, (str, Path)):
        data = Path(source).read_bytes()
    elif isinstance(source, bytes):
        data = source
    else:
        data = source.read()
        if isinstance(data, str):
            data = data.encode()
    if data[:4] == _BINARY_MAGIC:
        n = int(np.frombuffer(data[4:12], dtype="<i8")[0])
        body = np.frombuffer(data[12:], dtype="<f8")
        if body.size != 5 * n:
            raise ValueError(f"binary grid: expected {5 * n} floats, found {body.size}")
        x, y, fl, nx, ny = body.reshape(5, n)
        flag = fl.astype(np.int64)
        if not np.all(fl == flag):
            raise ValueError("binary grid: non-integer class flag")
        cloud = PointCloud(x.copy(), y.copy(), flag, nx.copy(), ny.copy())
        cloud.validate()
        return cloud
    return _parse_text(data.decode())


def _parse_text(text: str) -> PointCloud:
    header = None
    recs = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        body = raw.split("#", 1)[0].strip()
        if not body:
            continue
        tok = body.split()
        if header is None:
            if len(tok) != 1:
                raise ValueError(f"line {lineno}: expected point count, got {raw!r}")
            header = int(tok[0])
            if header <= 0:
                raise ValueError(f"line {lineno}: point count must be positive")
            continue
        try:
            px, py, fl = float(tok[0]), float(tok[1]), int(tok[2])
        except (IndexError, ValueError) as exc:
            raise ValueError(f"line {lineno}: malformed point record {raw!r}") from exc
        if fl == INTERIOR:
            if len(tok) != 3:
                raise ValueError(f"line {lineno}: interior point takes exactly 'x y flag'")
            recs.append((px, py, fl, 0.0, 0.0))
        else:
            if len(tok) != 5:
                raise ValueError(f"line {lineno}: boundary point needs 'x y flag nx ny'")
            recs.append((px, py, fl, float(tok[3]), float(tok[4])))
    if header is None:
        raise ValueError("empty grid file")
    if len(recs) != header:
        raise ValueError(f"header says {header} points, file has {len(recs)}")
    a = np.array(recs, dtype=np.float64)
    cloud = PointCloud(a[:, 0], a[:, 1], a[:, 2].astype(np.int64), a[:, 3], a[:, 4])
    cloud.validate()
    return cloud


def write_point_cloud(cloud: PointCloud, path, binary: bool = False) -> None:
    """Write text (17 significant digits, round-trips doubles) or KMF1 binary."""
    cloud.validate()
    path = Path(path)
    if binary:
        cols = np.concatenate([cloud.x, cloud.y, cloud.flag.astype(np.float64), cloud.nx, cloud.ny])
        path.write_bytes(_BINARY_MAGIC + np.array([cloud.n_points], dtype="<i8").tobytes()
                         + cols.astype("<f8").tobytes())
        return
    out = io.StringIO()
    out.write(f"{cloud.n_points}\n")
    for i in range(cloud.n_points):
        if cloud.flag[i] == INTERIOR:
            out.write(f"{cloud.x[i]:.17g} {cloud.y[i]:.17g} 0\n")
        else:
            out.write(f"{cloud.x[i]:.17g} {cloud.y[i]:.17g} {int(cloud.flag[i])} "
                      f"{cloud.nx[i]:.17g} {cloud.ny[i]:.17g}\n")
    path.write_text(out.getvalue())


# ----------------------------------------------------------- neighbour search


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


# ----------------------------------------------------------------- assembly


def _csr(cloud: PointCloud, lists) -> StencilSet:
    sizes = np.fromiter((len(v) for v in lists), dtype=np.int64, count=len(lists))
    ptr = np.concatenate([[0], np.cumsum(sizes)])
    idx = np.concatenate(lists).astype(np.int64) if ptr[-1] else np.empty(0, dtype=np.int64)
    own = np.repeat(np.arange(len(lists)), sizes)
    return StencilSet(ptr=ptr, idx=idx, dx=cloud.x[idx] - cloud.x[own], dy=cloud.y[idx] - cloud.y[own])


def _select(full: StencilSet, mask: np.ndarray) -> StencilSet:
    """Order-preserving sub-stencil (geometry.py:387-393)."""
    cnt = np.bincount(_owners(full.ptr)[mask], minlength=full.n_owners)
    ptr = np.concatenate([[0], np.cumsum(cnt)])
    return StencilSet(ptr=ptr, idx=full.idx[mask], dx=full.dx[mask], dy=full.dy[mask])


def _frame_family(rows_idx, rows_dt, rows_dn) -> StencilSet:
    cnt = np.array([r.shape[0] for r in rows_idx], dtype=np.int64)
    ptr = np.concatenate([[0], np.cumsum(cnt)])
    if ptr[-1]:
        idx = np.concatenate(rows_idx).astype(np.int64)
        dt = np.concatenate(rows_dt)
        dn = np.concatenate(rows_dn)
    else:
        idx, dt, dn = np.empty(0, dtype=np.int64), np.empty(0), np.empty(0)
    return StencilSet(ptr=ptr, idx=idx, dx=dt, dy=dn)


def _frames(cloud, full, thresh, points, side, failures):
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
    return FrameStencils(
        points=points, tx=tx, ty=ty, nx=nx, ny=ny,
        tplus=_frame_family(*fam["tp"]), tminus=_frame_family(*fam["tm"]),
        normal=_frame_family(*fam["nr"]), fallback=fallback,
    )


@dataclass
class _Parts:
    full: StencilSet
    split: dict
    d_min: np.ndarray
    d_mean: np.ndarray
    wall_frame: FrameStencils | None
    outer_frame: FrameStencils | None
    failures: list


def _assemble(cloud: PointCloud, lists) -> _Parts:
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
    wall_frame = _frames(cloud, full, thresh, cloud.wall, +1.0, failures)
    outer_frame = _frames(cloud, full, thresh, cloud.outer, -1.0, failures)
    return _Parts(full, split, d_min, d_mean, wall_frame, outer_frame, failures)


def build_stencils(cloud: PointCloud, epsilon: float | None = None, k: int | None = None,
                   native: bool | None = None) -> Connectivity:
    """Full, split and boundary-frame stencils with cached sums (geometry.py:453-518).

    Raises StencilDeficiencyError (after widening failing points to k=25)
    exactly where the reference does.  In k-nearest mode the heavy loops run
    in the native builder (builder.py, libkmf_build.so) unless native=False;
    native=None uses it when the library is built.  Both paths give
    bit-identical connectivities (tests/test_builder.py).
    """
    if epsilon is None and native is not False:
        from . import builder

        if native or builder.available():
            return builder.build_stencils_native(cloud, k)
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


# ------------------------------------------------------------ the generator

_T = 0.12  # NACA 0012 thickness ratio
_COEF = (0.2969, -0.1260, -0.3516, 0.2843, -0.1036)  # closed trailing edge
_CLUSTER = 0.6


def _half_thickness(xc):
    a0, a1, a2, a3, a4 = _COEF
    return 5.0 * _T * (a0 * np.sqrt(xc) + xc * (a1 + xc * (a2 + xc * (a3 + xc * a4))))


def _half_thickness_slope(xc):
    a0, a1, a2, a3, a4 = _COEF
    return 5.0 * _T * (0.5 * a0 / np.sqrt(xc) + a1 + xc * (2.0 * a2 + xc * (3.0 * a3 + xc * 4.0 * a4)))


def _mirror_ring(first, upper, middle, lower_sign):
    """[first, upper..., middle, sign * reversed(upper)...] -- exact y-mirror."""
    return np.concatenate([[first], upper, [middle], lower_sign * upper[::-1]])


def generate_naca_cloud(chord_points: int = 80, layers: int = 30, growth: float = 1.15,
                        far_field: float = 20.0) -> PointCloud:
    """O-type cloud around a NACA 0012 (geometry.py:672-770), bit-identical.

    ``chord_points`` wall points (equal-arc-length with mild clustering),
    ``layers`` rings blended to a far-field circle with geometric gap growth.
    Ring 0 is the wall, the last ring the outer boundary; points are stored
    ring by ring (ring j occupies [j*m, (j+1)*m)).
    """
    if chord_points < 40:
        raise ValueError("chord_points must be at least 40")
    if chord_points % 2:
        raise ValueError("chord_points must be even (mirror-symmetric surface)")
    if layers < 4:
        raise ValueError("layers must be at least 4")
    if growth < 1.0:
        raise ValueError("growth must be >= 1")
    if far_field <= 2.0:
        raise ValueError("far_field must exceed 2 chords")
    m = chord_points
    half = m // 2
    # arc-length table on a sqrt-stretched abscissa, then targets
    xt = np.linspace(0.0, 1.0, 4001) ** 2
    arc = np.concatenate([[0.0], np.cumsum(np.hypot(np.diff(xt), np.diff(_half_thickness(xt))))])
    t = np.arange(1, half) / half
    targets = arc[-1] * (1.0 - (t - _CLUSTER * np.sin(2.0 * np.pi * t) / (2.0 * np.pi)))
    xu = np.interp(targets, arc, xt)
    yu = _half_thickness(xu)
    slope = _half_thickness_slope(xu)
    norm = np.hypot(slope, 1.0)
    surf_x = _mirror_ring(1.0, xu, 0.0, 1.0)
    surf_y = _mirror_ring(0.0, yu, 0.0, -1.0)
    wall_nx = _mirror_ring(1.0, -slope / norm, -1.0, 1.0)
    wall_ny = _mirror_ring(0.0, 1.0 / norm, 0.0, -1.0)
    phi = np.pi * np.arange(1, half) / half
    cphi, sphi = np.cos(phi), np.sin(phi)
    far_x = _mirror_ring(0.5 + far_field, 0.5 + far_field * cphi, 0.5 - far_field, 1.0)
    far_y = _mirror_ring(0.0, far_field * sphi, 0.0, -1.0)
    outer_nx = _mirror_ring(1.0, cphi, -1.0, 1.0)
    outer_ny = _mirror_ring(0.0, sphi, 0.0, -1.0)
    gaps = growth ** np.arange(layers - 1)
    s = (np.concatenate([[0.0], np.cumsum(gaps)]) / np.sum(gaps))[:, None]
    x = ((1.0 - s) * surf_x + s * far_x).ravel()
    y = ((1.0 - s) * surf_y + s * far_y).ravel()
    flag = np.full((layers, m), INTERIOR, dtype=np.int64)
    flag[0], flag[-1] = WALL, OUTER
    nx = np.zeros((layers, m))
    ny = np.zeros((layers, m))
    nx[0], ny[0] = wall_nx, wall_ny
    nx[-1], ny[-1] = outer_nx, outer_ny
    cloud = PointCloud(x, y, flag.ravel(), nx.ravel(), ny.ravel())
    cloud.validate()
    return cloud


def growth_for_window(m: int, layers: int, ratio: float = 0.0735) -> float:
    """Ring growth g with first-ring anisotropy R = m (g-1)/(g^(L-1)-1) = ratio.

    SURVEY.md section 8(d): trailing-edge split stencils stay usable for
    R in [0.067, 0.079]; bisection on the monotone map g -> R.
    """
    lo, hi = 1.0 + 1e-12, 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        r = m * (mid - 1.0) / (mid ** (layers - 1) - 1.0)
        if r > ratio:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)
