"""Point clouds, stencils and the NACA 0012 cloud generator (host-side setup).

Drop-in for reference ``kmf.geometry``: same types and field names
(geometry.py:56-312), same builder semantics (geometry.py:315-646, native: builder.py)
and same generator (geometry.py:652-770).  This is SETUP, not the timed hot path: it
runs once on the host before the device context is created.  Its outputs
must be bit-identical to the reference's (they fix the summation order of
every least-squares sum on the device), which tests/test_geometry_parity.py
checks against sha256 digests of the reference's own arrays
(tests/golden/*.json).
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

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


# ----------------------------------------------------------------- builder


def _select(full: StencilSet, mask: np.ndarray) -> StencilSet:
    """Order-preserving sub-stencil (geometry.py:387-393)."""
    cnt = np.bincount(_owners(full.ptr)[mask], minlength=full.n_owners)
    ptr = np.concatenate([[0], np.cumsum(cnt)])
    return StencilSet(ptr=ptr, idx=full.idx[mask], dx=full.dx[mask], dy=full.dy[mask])


def build_stencils(cloud: PointCloud, epsilon: float | None = None, k: int | None = None) -> Connectivity:
    """Full, split and boundary-frame stencils with cached sums (geometry.py:453-518):
    the native builder (builder.py, libkmf_build.so), bit-identical to the
    reference's (tests/test_builder.py, tests/test_geometry_parity.py);
    StencilDeficiencyError (after widening failing points to k=25) exactly
    where the reference raises it."""
    from .builder import build_stencils_native

    return build_stencils_native(cloud, k=k, epsilon=epsilon)


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
