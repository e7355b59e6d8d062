"""Geometric domain decomposition with a deep halo (multi-GPU).

Rank r owns a contiguous range of the point order (the generator's ring
order: a band of rings).  Its local problem is the owned points plus
`depth = n_inner + 2` halo layers, L_k = N(L_{k-1}) minus earlier layers
(N = full-stencil neighbours).  With q exchanged for all halo points once
per RK stage:

  first order is exact on L0..L_{depth-1}, sweep s on L0..L_{depth-1-s},
  and after n_inner sweeps the gradients are exact on L0 and L1 -- all the
  owned flux residuals need.

Every owned point therefore runs exactly the single-GPU arithmetic, so
histories are bitwise identical for any rank count; the residue is the
exact limb sum all-reduced across ranks.  Local numbering: owned points
(in global order), then each halo layer sorted by global index; halo
points of the last layer get empty stencils (they only carry q).

`LocalPart.conn` is a regular Connectivity (sub-cloud, local CSR, split
families, sums, frames of the owned boundary points), so the same device
context -- and the CPU oracle in the tests -- runs it unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .geometry import (
    INTERIOR,
    Connectivity,
    FrameStencils,
    PointCloud,
    StencilSet,
    _select,
)


@dataclass
class LocalPart:
    rank: int
    nranks: int
    n_global: int
    n_owned: int
    layer_counts: np.ndarray      # cumulative local counts of layers 0..depth
    global_ids: np.ndarray        # local slot -> global point
    conn: Connectivity
    # halo exchange: for each peer, local slots to send (owned) and to fill (halo)
    send: dict = field(default_factory=dict)   # peer -> local owned slots (peer's recv order)
    recv: dict = field(default_factory=dict)   # peer -> local halo slots


def owner_ranges(n: int, nranks: int) -> np.ndarray:
    """Contiguous equal ranges: rank r owns [bounds[r], bounds[r+1])."""
    return np.array([r * n // nranks for r in range(nranks + 1)], dtype=np.int64)


def _neighbors_of(full: StencilSet, pts: np.ndarray) -> np.ndarray:
    if pts.size == 0:
        return np.empty(0, dtype=np.int64)
    lo, hi = full.ptr[pts], full.ptr[pts + 1]
    cnt = hi - lo
    starts = np.repeat(lo - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
    return full.idx[np.arange(cnt.sum()) + starts]


def halo_layers(full: StencilSet, owned: np.ndarray, depth: int):
    """[L0 = owned, L1, ..., L_depth] as sorted global index arrays."""
    n = full.n_owners
    have = np.zeros(n, dtype=bool)
    have[owned] = True
    layers = [owned]
    for _ in range(depth):
        nb = np.unique(_neighbors_of(full, layers[-1]))
        new = nb[~have[nb]]
        have[new] = True
        layers.append(new)
    return layers


def _sub_stencil(s: StencilSet, rows: np.ndarray, g2l: np.ndarray, keep_rows: np.ndarray) -> StencilSet:
    """Rows `rows` (global owners, in local order) of `s`, neighbours mapped
    to local slots; rows with keep_rows False get empty stencils."""
    cnt = np.where(keep_rows, s.ptr[rows + 1] - s.ptr[rows], 0)
    ptr = np.concatenate([[0], np.cumsum(cnt)])
    starts = np.repeat(s.ptr[rows] - ptr[:-1], cnt)
    e = np.arange(ptr[-1]) + starts
    idx = g2l[s.idx[e]]
    if (idx < 0).any():
        raise ValueError("stencil reaches outside the halo (depth too small)")
    return StencilSet(ptr=ptr, idx=idx, dx=s.dx[e], dy=s.dy[e])


def _sub_frame(fr: FrameStencils | None, g2l: np.ndarray, owned_mask: np.ndarray):
    if fr is None:
        return None
    sel = np.flatnonzero(owned_mask[fr.points])
    if sel.size == 0:
        return None
    fams = {}
    for name in ("tplus", "tminus", "normal"):
        s = getattr(fr, name)
        fams[name] = _sub_stencil(s, sel, g2l, np.ones(sel.size, dtype=bool))
    fb = {int(g2l[p]): v for p, v in fr.fallback.items() if owned_mask[p]}
    return FrameStencils(points=g2l[fr.points[sel]], tx=fr.tx[sel], ty=fr.ty[sel], nx=fr.nx[sel], ny=fr.ny[sel],
                         fallback=fb, **fams)


def build_part(conn: Connectivity, rank: int, nranks: int, depth: int) -> LocalPart:
    cl = conn.cloud
    n = cl.n_points
    b = owner_ranges(n, nranks)
    owned = np.arange(b[rank], b[rank + 1], dtype=np.int64)
    layers = halo_layers(conn.full, owned, depth)
    gid = np.concatenate(layers)
    g2l = np.full(n, -1, dtype=np.int64)
    g2l[gid] = np.arange(gid.size)
    counts = np.cumsum([l.size for l in layers]).astype(np.int64)
    inner = np.zeros(gid.size, dtype=bool)
    inner[: counts[-2] if depth > 0 else counts[-1]] = True  # last layer: q carriers only
    owned_mask = np.zeros(n, dtype=bool)
    owned_mask[owned] = True

    sub = PointCloud(cl.x[gid], cl.y[gid], cl.flag[gid], cl.nx[gid], cl.ny[gid])
    full = _sub_stencil(conn.full, gid, g2l, inner)
    split = {
        "x+": _select(full, full.dx <= 0.0),
        "x-": _select(full, full.dx >= 0.0),
        "y+": _select(full, full.dy <= 0.0),
        "y-": _select(full, full.dy >= 0.0),
    }
    interior = sub.flag == INTERIOR
    det_safe = {k: np.where(interior, s.det, 1.0) for k, s in split.items()}
    lconn = Connectivity(
        cloud=sub, full=full, split=split, d_min=conn.d_min[gid], d_mean=conn.d_mean[gid],
        wall_frame=_sub_frame(conn.wall_frame, g2l, owned_mask),
        outer_frame=_sub_frame(conn.outer_frame, g2l, owned_mask),
        det_safe=det_safe,
    )
    part = LocalPart(rank=rank, nranks=nranks, n_global=n, n_owned=int(owned.size), layer_counts=counts,
                     global_ids=gid, conn=lconn)
    # receive lists: halo points grouped by owner rank (local halo order kept)
    halo = gid[owned.size:]
    halo_owner = np.searchsorted(b, halo, side="right") - 1
    for peer in range(nranks):
        if peer == rank:
            continue
        sel = np.flatnonzero(halo_owner == peer)
        if sel.size:
            part.recv[peer] = owned.size + sel
    return part


def build_parts(conn: Connectivity, nranks: int, depth: int) -> list[LocalPart]:
    """All ranks' parts with matching send lists (send[peer] on rank r lists
    r's local slots of the points peer receives, in peer's receive order)."""
    parts = [build_part(conn, r, nranks, depth) for r in range(nranks)]
    b = owner_ranges(conn.cloud.n_points, nranks)
    for p in parts:
        for peer, slots in p.recv.items():
            glob = p.global_ids[slots]
            parts[peer].send[p.rank] = glob - b[peer]  # owned points are numbered first, in global order
    return parts


def send_lists_for(conn: Connectivity, rank: int, nranks: int, depth: int) -> dict:
    """send[peer] for one rank without building the other parts' connectivity."""
    b = owner_ranges(conn.cloud.n_points, nranks)
    out = {}
    for peer in range(nranks):
        if peer == rank:
            continue
        owned = np.arange(b[peer], b[peer + 1], dtype=np.int64)
        halo = np.concatenate(halo_layers(conn.full, owned, depth)[1:])
        mine = halo[(halo >= b[rank]) & (halo < b[rank + 1])]
        if mine.size:
            out[peer] = mine - b[rank]
    return out
