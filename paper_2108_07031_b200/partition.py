"""Geometric domain decomposition with a deep halo (multi-GPU).

Ownership (`owner_map`): "bands" -- contiguous ranges of the caller's point
order (the generator's ring order: a band of rings, cut along whole rings);
"sectors" -- equal-count angular sectors about the wall centroid (cut along
rays, so the halo grows with the number of rings L instead of the ring
length m: ~4x smaller at the 40M cloud).  Any ownership gives the same bits.

Rank r's local problem is its owned points plus `depth = n_inner + 2` halo
layers, L_k = N(L_{k-1}) minus earlier layers (N = full-stencil neighbours).
With q exchanged for all halo points once per RK stage, first order is
exact on L0..L_{depth-1}, sweep s on L0..L_{depth-1-s}, and after n_inner
sweeps the gradients are exact on L0 and L1 -- all the owned flux
residuals need.  Every owned point therefore runs exactly the single-GPU
arithmetic, so histories are bitwise identical for any rank count; the
residue is the exact limb sum all-reduced across ranks.

Local numbering: the owned points ordered by DEPTH -- the forward hop
distance to the nearest non-owned point, capped at depth + 1, deepest first
(ties in global order) -- then each halo layer sorted by global index;
halo points of the last layer get empty stencils (they only carry q).
Kernel k of a stage (0 first order, 1..n_inner sweeps, flux after them)
at an owned point of depth >= k + 2 reads only owned data of this stage,
so with this order it runs as a PREFIX of the slots before the stage's
halo exchange has arrived (the interior pass, overlapping the exchange)
and on the rest after it (the band pass): `stage_ranges` restates the
device schedule (kmf_b200.cu stage_range).

`LocalPart.conn` is a regular Connectivity (sub-cloud, local CSR, split
families, sums, frames of the owned boundary points), so the same device
context -- and the CPU oracle in the tests -- runs it unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .geometry import (
    INTERIOR,
    WALL,
    Connectivity,
    FrameStencils,
    PointCloud,
    StencilSet,
    _select,
)

SCHEMES = ("bands", "sectors")


@dataclass
class LocalPart:
    rank: int
    nranks: int
    n_global: int
    n_owned: int
    depth: int
    layer_counts: np.ndarray      # cumulative local counts of layers 0..depth (layer_end)
    interior_end: np.ndarray      # [k] owned slots at depth >= k, k = 0..depth+1 (non-increasing)
    global_ids: np.ndarray        # local slot -> global point
    conn: Connectivity
    scheme: str = "bands"
    # halo exchange: for each peer, local slots to send (owned) and to fill (halo)
    send: dict = field(default_factory=dict)   # peer -> local owned slots (peer's recv order)
    recv: dict = field(default_factory=dict)   # peer -> local halo slots

    def local_of_owned(self, gids: np.ndarray) -> np.ndarray:
        """Local slots of owned global points (any order)."""
        owned = self.global_ids[: self.n_owned]
        order = np.argsort(owned, kind="stable")
        pos = np.searchsorted(owned[order], gids)
        if pos.size and (pos.max() >= owned.size or not np.array_equal(owned[order][pos], gids)):
            raise ValueError("points not owned by this rank")
        return order[pos].astype(np.int64)


def owner_ranges(n: int, nranks: int) -> np.ndarray:
    """Contiguous equal ranges: rank r owns [bounds[r], bounds[r+1])."""
    return np.array([r * n // nranks for r in range(nranks + 1)], dtype=np.int64)


def owner_map(cloud: PointCloud, nranks: int, scheme: str = "bands") -> np.ndarray:
    """Owning rank of every point (int32, caller order)."""
    n = cloud.n_points
    if scheme not in SCHEMES:
        raise ValueError(f"scheme must be one of {SCHEMES}")
    own = np.empty(n, dtype=np.int32)
    if scheme == "bands" or nranks == 1:
        b = owner_ranges(n, nranks)
        for r in range(nranks):
            own[b[r]:b[r + 1]] = r
        return own
    wall = cloud.flag == WALL
    cx, cy = (float(np.mean(cloud.x[wall])), float(np.mean(cloud.y[wall]))) if wall.any() else (
        float(np.mean(cloud.x)), float(np.mean(cloud.y)))
    theta = np.arctan2(cloud.y - cy, cloud.x - cx)
    order = np.argsort(theta, kind="stable")
    b = owner_ranges(n, nranks)
    for r in range(nranks):
        own[order[b[r]:b[r + 1]]] = r
    return own


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


def owned_depth(full: StencilSet, owned: np.ndarray, cap: int) -> np.ndarray:
    """Forward hop distance from each owned point (sorted global ids) to the
    nearest non-owned point along stencil edges i -> j, j in N(i), capped at
    `cap`: a kernel reading neighbours k+1 hops out at a point of depth
    >= k + 2 touches owned data only.  Unit-weight Bellman-Ford relaxation
    over the owned rows (one gather per hop)."""
    n = full.n_owners
    d = np.zeros(n, dtype=np.int8)
    d[owned] = cap
    lo, hi = full.ptr[owned], full.ptr[owned + 1]
    cnt = (hi - lo).astype(np.int64)
    if owned.size and owned[-1] - owned[0] + 1 == owned.size:  # contiguous rows: a view
        idx = full.idx[lo[0]:hi[-1]]
        starts = lo - lo[0]
    else:
        starts = np.concatenate([[0], np.cumsum(cnt)[:-1]])
        idx = full.idx[np.arange(cnt.sum()) + np.repeat(lo - starts, cnt)]
    has = cnt > 0
    for _ in range(cap):
        nb = d[idx]
        m = np.full(owned.size, cap, dtype=np.int16)
        if has.any():
            m[has] = np.minimum.reduceat(nb, starts[has]).astype(np.int16) + 1
        new = np.minimum(d[owned], m).astype(np.int8)
        if np.array_equal(new, d[owned]):
            break
        d[owned] = new
    return d[owned].astype(np.int64)


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


def build_part(conn: Connectivity, rank: int, nranks: int, depth: int, scheme: str = "bands",
               owner: np.ndarray | None = None) -> LocalPart:
    cl = conn.cloud
    n = cl.n_points
    if owner is None:
        owner = owner_map(cl, nranks, scheme)
    owned = np.flatnonzero(owner == rank).astype(np.int64)
    layers = halo_layers(conn.full, owned, depth)
    dep = owned_depth(conn.full, owned, depth + 1)
    owned_sorted = owned[np.argsort(-dep, kind="stable")]
    gid = np.concatenate([owned_sorted] + layers[1:])
    g2l = np.full(n, -1, dtype=np.int64)
    g2l[gid] = np.arange(gid.size)
    counts = np.cumsum([l.size for l in layers]).astype(np.int64)
    interior_end = np.array([int((dep >= k).sum()) for k in range(depth + 2)], dtype=np.int64)
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
    part = LocalPart(rank=rank, nranks=nranks, n_global=n, n_owned=int(owned.size), depth=depth,
                     layer_counts=counts, interior_end=interior_end, global_ids=gid, conn=lconn, scheme=scheme)
    # receive lists: halo points grouped by owner rank (local halo order kept)
    halo_owner = owner[gid[owned.size:]]
    for peer in range(nranks):
        if peer == rank:
            continue
        sel = np.flatnonzero(halo_owner == peer)
        if sel.size:
            part.recv[peer] = owned.size + sel
    return part


def build_parts(conn: Connectivity, nranks: int, depth: int, scheme: str = "bands") -> list[LocalPart]:
    """All ranks' parts with matching send lists (send[peer] on rank r lists
    r's local slots of the points peer receives, in peer's receive order)."""
    owner = owner_map(conn.cloud, nranks, scheme)
    parts = [build_part(conn, r, nranks, depth, scheme, owner) for r in range(nranks)]
    for p in parts:
        for peer, slots in p.recv.items():
            parts[peer].send[p.rank] = parts[peer].local_of_owned(p.global_ids[slots])
    return parts


def send_lists_for(conn: Connectivity, part: LocalPart, owner: np.ndarray | None = None) -> dict:
    """send[peer] for one rank's part without building the other parts'
    connectivity: each peer's halo layers, restricted to this rank's owned
    points, in the peer's receive order."""
    if owner is None:
        owner = owner_map(conn.cloud, part.nranks, part.scheme)
    out = {}
    for peer in range(part.nranks):
        if peer == part.rank:
            continue
        peer_owned = np.flatnonzero(owner == peer).astype(np.int64)
        halo = np.concatenate(halo_layers(conn.full, peer_owned, part.depth)[1:])
        mine = halo[owner[halo] == part.rank]
        if mine.size:
            out[peer] = part.local_of_owned(mine)
    return out


def stage_ranges(part: LocalPart, n_inner: int) -> list:
    """The device schedule of one RK stage (kmf_b200.cu stage_range), as
    [(kernel, interior (lo, hi), band (lo, hi))] for the first order, the
    n_inner sweeps and the flux."""
    if n_inner + 2 > part.depth:
        raise ValueError(f"n_inner {n_inner} needs a halo of depth {n_inner + 2}, the partition has {part.depth}")
    out = []
    kernels = ([("first_order", 0)] + [(f"sweep{s}", s) for s in range(1, n_inner + 1)]) if n_inner > 0 else []
    kernels.append(("flux", n_inner + 1 if n_inner > 0 else 0))
    for name, k in kernels:
        cut = int(part.interior_end[min(k + 2, part.depth + 1)])
        end = part.n_owned if name == "flux" else int(part.layer_counts[max(0, part.depth - 1 - k)])
        out.append((name, (0, cut), (cut, max(cut, end))))
    return out
