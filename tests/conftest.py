"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built
libkmf_b200.so; everything else runs on the CPU (the oracle and host logic).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

# before CUDA initialises in this process: the peer-linked group tests run
# up to 4 ranks concurrently on one device, each on two streams that spin on
# each other (kmf_peer_link refuses fewer hardware queues than 2 per rank)
import os  # noqa: E402

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2108_07031_b200.geometry import (  # noqa: E402
    INTERIOR,
    OUTER,
    WALL,
    PointCloud,
    build_stencils,
    generate_naca_cloud,
)
from paper_2108_07031_b200.state import Primitives, free_stream  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libkmf_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden(name: str):
    """(arrays, meta) of tests/golden/<name>.{npz,json} (tools/make_golden.py)."""
    npz = GOLDEN / f"{name}.npz"
    arrays = dict(np.load(npz)) if npz.exists() else {}
    meta = json.loads((GOLDEN / f"{name}.json").read_text())
    return arrays, meta


def lattice_cloud(n: int = 5, h: float = 1.0, classify_boundary: bool = False) -> PointCloud:
    """n x n lattice, rim optionally outer (reference tests/conftest.py:7-28)."""
    gx, gy = np.meshgrid(np.arange(n) * h, np.arange(n) * h, indexing="ij")
    x, y = gx.ravel(), gy.ravel()
    flag = np.full(x.size, INTERIOR, dtype=np.int64)
    nx = np.zeros(x.size)
    ny = np.zeros(x.size)
    if classify_boundary:
        lim = (n - 1) * h
        rim = (x == 0.0) | (y == 0.0) | (x == lim) | (y == lim)
        flag[rim] = OUTER
        nx[x == 0.0] -= 1.0
        nx[x == lim] += 1.0
        ny[y == 0.0] -= 1.0
        ny[y == lim] += 1.0
        norm = np.hypot(nx, ny)
        ok = norm > 0
        nx[ok] /= norm[ok]
        ny[ok] /= norm[ok]
    return PointCloud(x, y, flag, nx, ny)


def channel_cloud(nx=9, ny=6, h=0.1) -> PointCloud:
    """Flat-wall channel lattice (reference tests/test_solver.py:74-95)."""
    gx, gy = np.meshgrid(np.arange(nx) * h, np.arange(ny) * h, indexing="ij")
    x, y = gx.ravel(), gy.ravel()
    flag = np.zeros(x.size, dtype=np.int64)
    mx = np.zeros(x.size)
    my = np.zeros(x.size)
    bottom = y < 0.5 * h
    top = y > (ny - 1.5) * h
    left = x < 0.5 * h
    right = x > (nx - 1.5) * h
    flag[bottom] = WALL
    my[bottom] = 1.0
    for side, (sx, sy) in ((top, (0.0, 1.0)), (left, (-1.0, 0.0)), (right, (1.0, 0.0))):
        sel = side & ~bottom
        flag[sel] = OUTER
        mx[sel], my[sel] = sx, sy
    corner = (left | right) & top
    nrm = np.hypot(np.where(left, -1.0, 1.0), 1.0)
    mx[corner] = np.where(left, -1.0, 1.0)[corner] / nrm[corner]
    my[corner] = 1.0 / nrm[corner]
    return PointCloud(x, y, flag, mx, my)


def perturbed_state(cloud, mach=0.63, aoa=2.0, gamma=1.4, amp=0.02) -> Primitives:
    """Free stream plus a smooth bump (reference tests/test_solver.py:98-102)."""
    fs = free_stream(mach, aoa, gamma, n=cloud.n_points)
    bump = amp * np.exp(-((cloud.x - 1.8) ** 2 + cloud.y ** 2) / 0.16)
    return Primitives(fs.rho * (1.0 + bump), fs.u1, fs.u2, fs.p * (1.0 + gamma * bump))


def fs_vec(mach, aoa, gamma=1.4):
    fs = free_stream(mach, aoa, gamma)
    return np.array([fs.rho[0], fs.u1[0], fs.u2[0], fs.p[0]])


@pytest.fixture(scope="session")
def small_naca():
    return generate_naca_cloud(80, 30, 1.15, 20.0)


@pytest.fixture(scope="session")
def small_naca_conn(small_naca):
    return build_stencils(small_naca)


@pytest.fixture(scope="session")
def small_golden():
    return golden("small")


@pytest.fixture(scope="session")
def oracle_small(small_naca_conn):
    from oracle import oracle as O

    return O.Packed(small_naca_conn)


def _has_gpu() -> bool:
    try:
        from paper_2108_07031_b200 import _lib

        return _lib.lib().kmf_device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    """Fail loudly (not skip) when a -m gpu test runs without the device path."""
    from paper_2108_07031_b200 import _lib

    _lib.require_device()
    return True
