"""Native stencil builder (libkmf_build.so, builder.py) == the scipy
restatement of the reference builder (oracle/builder_ref.py, test
infrastructure), bit for bit.  CPU only.

The reference digests in test_geometry_parity.py already run through the
native path (it is build_stencils' default); these tests pin the two paths
against each other on the cases the digests do not cover (other k, the
widening pass, deficiency errors, degenerate and tie-heavy clouds).
"""

import numpy as np
import pytest

from conftest import channel_cloud, lattice_cloud
from paper_2108_07031_b200 import builder
from oracle.builder_ref import build_stencils_ref, knn_lists, radius_lists
from paper_2108_07031_b200.geometry import (
    PointCloud,
    StencilDeficiencyError,
    build_stencils,
    generate_naca_cloud,
)

pytestmark = pytest.mark.skipif(not builder.available(), reason="libkmf_build.so not built")

FIELDS = ("ptr", "idx", "dx", "dy", "sxx", "sxy", "syy", "det")


def assert_same(a, b):
    for nm in FIELDS:
        assert np.array_equal(getattr(a.full, nm), getattr(b.full, nm)), f"full.{nm}"
    for kind in a.split:
        for nm in FIELDS:
            assert np.array_equal(getattr(a.split[kind], nm), getattr(b.split[kind], nm)), f"{kind}.{nm}"
        assert np.array_equal(a.split[kind].counts(), b.split[kind].counts())
        assert np.array_equal(a.det_safe[kind], b.det_safe[kind])
    assert np.array_equal(a.d_min, b.d_min) and np.array_equal(a.d_mean, b.d_mean)
    for fr in ("wall_frame", "outer_frame"):
        fa, fb = getattr(a, fr), getattr(b, fr)
        assert (fa is None) == (fb is None)
        if fa is None:
            continue
        for k in ("points", "tx", "ty", "nx", "ny"):
            assert np.array_equal(getattr(fa, k), getattr(fb, k))
        for st in ("tplus", "tminus", "normal"):
            for nm in FIELDS:
                assert np.array_equal(getattr(getattr(fa, st), nm), getattr(getattr(fb, st), nm)), f"{fr}.{st}.{nm}"
        assert fa.fallback == fb.fallback


@pytest.mark.parametrize("args,k", [((80, 30, 1.15), None), ((80, 30, 1.15), 8), ((80, 30, 1.15), 25),
                                    ((120, 40, 1.1), 6), ((400, 100, 1.06), None)])
def test_naca_native_equals_scipy(args, k):
    cloud = generate_naca_cloud(*args, 20.0)
    assert_same(build_stencils(cloud, k=k), build_stencils_ref(cloud, k=k))


@pytest.mark.parametrize("n,h,k", [(5, 0.01, 8), (7, 1.0, None), (9, 0.5, 12), (4, 1.0, 6)])
def test_lattice_ties_native_equals_scipy(n, h, k):
    cloud = lattice_cloud(n, h, True)
    assert_same(build_stencils(cloud, k=k), build_stencils_ref(cloud, k=k))


def test_channel_native_equals_scipy():
    cloud = channel_cloud()
    assert_same(build_stencils(cloud, k=8), build_stencils_ref(cloud, k=8))


def test_knn_rows_match_scipy_including_plateaus():
    # a lattice has exact distance ties at every shell: the cut is tie-inclusive
    cloud = lattice_cloud(11, 0.3, False)
    for k in (4, 8, 12, 20):
        ptr, idx = builder.knn_csr(cloud, k)
        ref = knn_lists(cloud.x, cloud.y, k)
        assert [list(idx[ptr[i]:ptr[i + 1]]) for i in range(cloud.n_points)] == [list(r) for r in ref]
    sub = np.array([0, 5, 60, 120], dtype=np.int64)
    ptr, idx = builder.knn_csr(cloud, 25, sub)
    ref = knn_lists(cloud.x, cloud.y, 25, sub)
    assert [list(idx[ptr[i]:ptr[i + 1]]) for i in range(sub.size)] == [list(r) for r in ref]


def test_random_cloud_native_equals_scipy():
    rng = np.random.default_rng(7)
    n = 3000
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    cloud = PointCloud(x, y, np.zeros(n, dtype=np.int64), np.zeros(n), np.zeros(n))
    for k in (6, 15):
        ptr, idx = builder.knn_csr(cloud, k)
        ref = knn_lists(x, y, k)
        assert np.array_equal(idx, np.concatenate(ref))


def test_deficiency_error_identical():
    cloud = PointCloud(np.arange(8, dtype=float), np.zeros(8), np.zeros(8, dtype=np.int64), np.zeros(8), np.zeros(8))
    with pytest.raises(StencilDeficiencyError) as a:
        build_stencils(cloud, k=6)
    with pytest.raises(StencilDeficiencyError) as b:
        build_stencils_ref(cloud, k=6)
    assert a.value.failures == b.value.failures


def test_split_view_materialises_the_sign_subsets():
    cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
    conn = build_stencils(cloud)
    f = conn.full
    for kind, m in zip(("x+", "x-", "y+", "y-"), (f.dx <= 0, f.dx >= 0, f.dy <= 0, f.dy >= 0)):
        s = conn.split[kind]
        assert isinstance(s, builder.SplitView)
        assert np.array_equal(s.idx, f.idx[m])
        assert s.ptr[-1] == m.sum()
        i = 100
        assert np.array_equal(s.neighbors(i), s.idx[s.ptr[i]:s.ptr[i + 1]])


def test_store_round_trip_memory_mapped(tmp_path):
    from paper_2108_07031_b200 import store

    cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
    conn = build_stencils(cloud)
    store.save(conn, tmp_path / "c", extra={"init": np.arange(6.0)})
    back, extra = store.load(tmp_path / "c")
    assert isinstance(back.full.idx, np.memmap)
    assert np.array_equal(extra["init"], np.arange(6.0))
    for k in ("x", "y", "flag", "nx", "ny"):
        assert np.array_equal(getattr(back.cloud, k), getattr(cloud, k))
    assert_same(back, conn)


@pytest.mark.parametrize("n,h,eps", [(7, 1.0, 1.5), (9, 0.5, 1.2), (6, 1.0, 1.01), (8, 0.25, 0.3)])
def test_radius_mode_native_equals_scipy(n, h, eps):
    """epsilon mode (geometry.py:349-374 + the thin-row kNN fallback and
    the widening pass): rows, sums and frames bit for bit."""
    cloud = lattice_cloud(n, h, True)
    try:
        ref = build_stencils_ref(cloud, epsilon=eps)
    except StencilDeficiencyError:
        with pytest.raises(StencilDeficiencyError):
            build_stencils(cloud, epsilon=eps)
        return
    assert_same(build_stencils(cloud, epsilon=eps), ref)


def test_radius_rows_native_equal_scipy():
    rng = np.random.default_rng(3)
    x, y = rng.uniform(0, 1, 3000), rng.uniform(0, 1, 3000)
    cloud = PointCloud(x, y, np.zeros(3000, dtype=np.int64), np.zeros(3000), np.zeros(3000))
    for eps in (0.01, 0.03, 0.07):
        ptr, idx = builder.radius_csr(cloud, eps)
        ref = radius_lists(x, y, eps)
        assert np.array_equal(np.diff(ptr), [len(r) for r in ref])
        assert np.array_equal(idx, np.concatenate(ref))


def test_argument_errors_match_the_reference():
    cloud = lattice_cloud(5, 1.0, True)
    with pytest.raises(ValueError, match="either epsilon or k"):
        build_stencils(cloud, epsilon=1.5, k=8)
    with pytest.raises(ValueError, match="epsilon must be positive"):
        build_stencils(cloud, epsilon=-1.0)
    with pytest.raises(ValueError, match="at least 6"):
        build_stencils(cloud, k=5)
