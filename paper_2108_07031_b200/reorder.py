"""Space-filling-curve point ordering for the device layout.

The device stores every per-point field (and the sliced-ELL stencil) in a
permuted "slot" order; neighbour lists keep their reference order, so every
least-squares sum, every flux and the exact residue are bitwise identical
in any order (tests/test_gpu_reorder.py).  The order only changes memory
locality: a Hilbert order makes each 32-point warp and each 128-thread block
a compact 2D patch whose neighbour halo is small, so neighbour gathers hit L1
more often than in the generator's ring-by-ring order.

The permutation is a pure integer function of the quantised coordinates
(21 bits per axis over the cloud's bounding box, ties broken by the original
index), so it is reproducible bit for bit on any host.
"""

from __future__ import annotations

import numpy as np

ORDERS = ("natural", "hilbert", "ringtile2", "ringtile4", "ringtile8")
BITS = 21


def _quantise(v: np.ndarray, bits: int) -> np.ndarray:
    lo, hi = float(v.min()), float(v.max())
    span = hi - lo if hi > lo else 1.0
    scale = float((1 << bits) - 1) / span
    return np.floor((v - lo) * scale).astype(np.int64)


def hilbert_keys(x: np.ndarray, y: np.ndarray, bits: int = BITS) -> np.ndarray:
    """Hilbert-curve index of each point on a 2^bits x 2^bits grid."""
    xi = _quantise(np.asarray(x, dtype=np.float64), bits)
    yi = _quantise(np.asarray(y, dtype=np.float64), bits)
    d = np.zeros(xi.shape, dtype=np.int64)
    n = 1 << bits
    s = n >> 1
    while s > 0:
        rx = ((xi & s) > 0).astype(np.int64)
        ry = ((yi & s) > 0).astype(np.int64)
        d += s * s * ((3 * rx) ^ ry)
        # rotate the quadrant (classic xy2d)
        flip = ry == 0
        swap_r = flip & (rx == 1)
        xi = np.where(swap_r, n - 1 - xi, xi)
        yi = np.where(swap_r, n - 1 - yi, yi)
        xi, yi = np.where(flip, yi, xi), np.where(flip, xi, yi)
        s >>= 1
    return d


def ring_tiles(n: int, m: int, tile_rings: int = 4, width: int = 32) -> np.ndarray:
    """Tile order for ring-structured clouds (point r*m + a is angle a of
    ring r, as generate_naca_cloud numbers them): bands of `tile_rings`
    rings, each cut into `width`-point angular tiles stored ring by ring.
    A warp still owns `width` angularly consecutive points (so its slot-s
    neighbours stay consecutive and coalesced) while a block's warps stack
    radially and share their neighbour rings in L1."""
    if n % m:
        raise ValueError("ring tiling needs n to be a multiple of the ring size m")
    k = np.arange(n, dtype=np.int64)
    r, a = k // m, k % m
    return np.lexsort((a % width, r % tile_rings, a // width, r // tile_rings)).astype(np.int64)


def permutation(cloud, order: str = "hilbert", ring_size: int | None = None) -> np.ndarray | None:
    """perm[k] = caller point stored in device slot k (None for natural).

    "ringtile" needs the ring size m of a generator cloud (ring_size, or the
    number of wall points when the cloud has one wall ring)."""
    if order not in ORDERS:
        raise ValueError(f"order must be one of {ORDERS}")
    if order == "natural":
        return None
    if order.startswith("ringtile"):
        m = ring_size or int((cloud.flag == 1).sum())
        rows = int(order[len("ringtile"):] or 4)
        return ring_tiles(cloud.n_points, m, rows)
    keys = hilbert_keys(cloud.x, cloud.y)
    return np.lexsort((np.arange(keys.size), keys)).astype(np.int64)
