"""The host set-up is bit-exact against the reference: generator, stencil
builder (kNN ties, visibility filter, widening, frames) and initial state,
compared by sha256 digests of the reference's own arrays.  CPU only.
"""

import hashlib

import numpy as np
import pytest

from conftest import channel_cloud, golden, lattice_cloud
from paper_2108_07031_b200.geometry import (
    PointCloud,
    StencilDeficiencyError,
    build_stencils,
    generate_naca_cloud,
    read_point_cloud,
    write_point_cloud,
)
from paper_2108_07031_b200.solver import SolverConfig, initial_primitives


def digest(a) -> str:
    a = np.asarray(a)
    a = a.astype("<i8") if a.dtype.kind in "biu" else a.astype("<f8")
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def conn_digests(cloud, conn) -> dict:
    out = {f"cloud.{k}": digest(getattr(cloud, k)) for k in ("x", "y", "flag", "nx", "ny")}

    def st(prefix, s):
        for k in ("ptr", "idx", "dx", "dy", "sxx", "sxy", "syy", "det"):
            out[f"{prefix}.{k}"] = digest(getattr(s, k))

    st("full", conn.full)
    for kind, s in conn.split.items():
        st(f"split[{kind}]", s)
        out[f"det_safe[{kind}]"] = digest(conn.det_safe[kind])
    out["d_min"] = digest(conn.d_min)
    out["d_mean"] = digest(conn.d_mean)
    for fname in ("wall_frame", "outer_frame"):
        fr = getattr(conn, fname)
        if fr is None:
            out[fname] = None
            continue
        for k in ("points", "tx", "ty", "nx", "ny"):
            out[f"{fname}.{k}"] = digest(getattr(fr, k))
        for sn in ("tplus", "tminus", "normal"):
            st(f"{fname}.{sn}", getattr(fr, sn))
        out[f"{fname}.fallback"] = sorted([int(k), v] for k, v in fr.fallback.items())
    out["n_points"] = int(cloud.n_points)
    out["n_edges"] = int(conn.full.idx.size)
    return out


def assert_digests(mine: dict, ref: dict):
    bad = [k for k, v in mine.items() if ref.get(k) != v]
    assert not bad, f"mismatching arrays vs reference: {bad[:10]}"


def test_small_naca_bitexact(small_naca, small_naca_conn):
    _, meta = golden("small")
    assert_digests(conn_digests(small_naca, small_naca_conn), meta["digests"])


@pytest.mark.parametrize("tag,mach,aoa", [("m63a2", 0.63, 2.0), ("m63a0", 0.63, 0.0), ("m85a1", 0.85, 1.0)])
def test_initial_state_bitexact(tag, mach, aoa, small_naca):
    _, meta = golden("small")
    ip = initial_primitives(SolverConfig(mach=mach, aoa_deg=aoa), small_naca)
    assert digest(np.stack([ip.rho, ip.u1, ip.u2, ip.p])) == meta["digests"][f"init.{tag}"]


def test_lattice_and_channel_bitexact():
    _, meta = golden("lattice")
    cases = {
        "lat5_k8": (lattice_cloud(5, 0.01, True), 8),
        "lat7_k15": (lattice_cloud(7, 1.0, True), None),
        "chan_k8": (channel_cloud(), 8),
    }
    for tag, (cloud, k) in cases.items():
        assert_digests(conn_digests(cloud, build_stencils(cloud, k=k)), meta["digests"][tag])


def test_config2_160k_bitexact():
    """Config 2 (800, 200, 1.03): 160,000 points, 2.4M edges."""
    _, meta = golden("c160k")
    m, L, g, ff = meta["params"]
    cloud = generate_naca_cloud(m, L, g, ff)
    conn = build_stencils(cloud)
    d = conn_digests(cloud, conn)
    assert_digests(d, meta["digests"])
    ip = initial_primitives(SolverConfig(mach=meta["mach"], aoa_deg=meta["aoa"]), cloud)
    assert digest(np.stack([ip.rho, ip.u1, ip.u2, ip.p])) == meta["digests"]["init"]


def test_mirror_symmetric_stencil_membership(small_naca, small_naca_conn):
    """Reference tests/test_geometry.py:258-274: mirrored points have
    mirrored stencils (tie-inclusive kNN)."""
    m = 80
    mirror = np.concatenate([r * m + (m - np.arange(m)) % m for r in range(30)])
    s = small_naca_conn.full
    for i in range(0, small_naca.n_points, 37):
        a = set(s.neighbors(i).tolist())
        b = set(mirror[s.neighbors(mirror[i])].tolist())
        assert a == b


def test_deficient_cloud_raises():
    # three collinear interior points cannot support any 2x2 LS solve
    cloud = PointCloud(np.array([0.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0]), np.zeros(8),
                       np.zeros(8, dtype=np.int64), np.zeros(8), np.zeros(8))
    with pytest.raises(StencilDeficiencyError):
        build_stencils(cloud, k=6)


def test_builder_argument_validation(small_naca):
    with pytest.raises(ValueError):
        build_stencils(small_naca, epsilon=0.1, k=8)
    with pytest.raises(ValueError):
        build_stencils(small_naca, k=5)
    with pytest.raises(ValueError):
        build_stencils(small_naca, epsilon=-1.0)


def test_generator_validation():
    for args in ((39, 30, 1.1, 20.0), (81, 30, 1.1, 20.0), (80, 3, 1.1, 20.0), (80, 30, 0.9, 20.0),
                 (80, 30, 1.1, 2.0)):
        with pytest.raises(ValueError):
            generate_naca_cloud(*args)


@pytest.mark.parametrize("binary", [False, True])
def test_grid_io_round_trip(tmp_path, small_naca, binary):
    p = tmp_path / ("g.bin" if binary else "g.txt")
    write_point_cloud(small_naca, p, binary=binary)
    back = read_point_cloud(p)
    for k in ("x", "y", "flag", "nx", "ny"):
        assert np.array_equal(getattr(back, k), getattr(small_naca, k))


def test_text_grid_errors():
    with pytest.raises(ValueError):
        read_point_cloud(b"")
    with pytest.raises(ValueError):
        read_point_cloud(b"2\n0 0 0\n")
    with pytest.raises(ValueError):
        read_point_cloud(b"1\n0 0 1\n")


def test_hilbert_permutation_is_local_and_deterministic(small_naca):
    from paper_2108_07031_b200 import reorder

    p = reorder.permutation(small_naca, "hilbert")
    assert np.array_equal(np.sort(p), np.arange(small_naca.n_points))
    assert np.array_equal(p, reorder.permutation(small_naca, "hilbert"))
    assert reorder.permutation(small_naca, "natural") is None
    # the 2x2 grid in Hilbert order visits (0,0),(0,1),(1,1),(1,0)
    k = reorder.hilbert_keys(np.array([0.0, 0.0, 1.0, 1.0]), np.array([0.0, 1.0, 1.0, 0.0]), bits=1)
    assert list(k) == [0, 1, 2, 3]
