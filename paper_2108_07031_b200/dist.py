"""Partitioned (multi-GPU) solve on top of the device contexts.

Two drivers share the partition of `partition.py` and the device kernels:

* `solve_group` -- one process, one context per rank (same GPU or several
  GPUs), halo q moved by device / peer copies (`kmf_run_group`).  Used by the
  multi-rank parity tests on a single B200 and as a one-process multi-GPU
  mode.
* `RankSolver` -- one process per GPU (torchrun), halo exchange and the
  residue limb all-reduce over NCCL inside the iteration graph
  (`kmf_nccl_init` + `kmf_run`).  torch.distributed only carries the NCCL
  unique id and the final error / state gathers (plumbing).

Both run the same per-stage schedule: an interior pass over the owned
points that read no halo data of this stage, the halo exchange (under NCCL
on a forked stream, overlapping the interior pass), then the band pass
(partition.stage_ranges).  Every rank runs the single-GPU arithmetic on its
owned points, so the residue history is bitwise identical to `solver.solve`
for any rank count and ownership scheme (tests/test_gpu_dist.py,
tests/test_partition.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._device import DeviceConnectivity
from .geometry import Connectivity
from .partition import LocalPart, build_part, owner_map, send_lists_for
from .solver import SolverConfig, _params, initial_primitives
from .state import PositivityError, Primitives, prims_array, raise_decode_flags


def attach_partition(dev: DeviceConnectivity, part: LocalPart) -> None:
    peers = sorted(set(part.send) | set(part.recv))
    layer_end = np.ascontiguousarray(part.layer_counts, dtype=np.int64)
    interior_end = np.ascontiguousarray(part.interior_end, dtype=np.int64)
    send_counts = np.array([part.send.get(p, np.empty(0)).size for p in peers], dtype=np.int64)
    recv_counts = np.array([part.recv.get(p, np.empty(0)).size for p in peers], dtype=np.int64)
    send = np.concatenate([part.send[p] for p in peers if p in part.send] or [np.empty(0, np.int64)]).astype(np.int64)
    recv = np.concatenate([part.recv[p] for p in peers if p in part.recv] or [np.empty(0, np.int64)]).astype(np.int64)
    pr = (C.c_int * max(len(peers), 1))(*peers)
    keep = (send_counts, recv_counts, send, recv)
    _lib.check(
        _lib.lib().kmf_set_partition(dev.handle, part.n_owned, part.n_global, part.rank, part.nranks, part.depth,
                                     _lib.i64ptr(layer_end), _lib.i64ptr(interior_end), len(peers), pr,
                                     _lib.i64ptr(keep[0]), _lib.i64ptr(keep[2]), _lib.i64ptr(keep[1]),
                                     _lib.i64ptr(keep[3])),
        "kmf_set_partition",
    )


class RankPart:
    """One rank's partition and its device context."""

    def __init__(self, conn: Connectivity, rank: int, nranks: int, n_inner: int = 3, device: int | None = None,
                 part: LocalPart | None = None, scheme: str = "bands", owner=None):
        depth = n_inner + 2
        if part is None:
            if owner is None:
                owner = owner_map(conn.cloud, nranks, scheme)
            part = build_part(conn, rank, nranks, depth, scheme, owner)
            part.send = send_lists_for(conn, part, owner)
        self.part = part
        self.dev = DeviceConnectivity(part.conn, device=device)
        attach_partition(self.dev, part)

    def set_state(self, prims_global: np.ndarray) -> None:
        self.dev.set_state(np.ascontiguousarray(prims_global[:, self.part.global_ids]))

    def owned_state(self):
        prims, U = self.dev.get_state()
        no = self.part.n_owned
        return self.part.global_ids[:no], prims[:, :no], U[:, :no]


def _rank_error(rp: RankPart) -> _lib.ErrorInfo:
    info = _lib.ErrorInfo()
    _lib.lib().kmf_last_error(rp.dev.handle, C.byref(info))
    return info


def _decode_failures(rp: RankPart, info, params) -> tuple:
    """(iteration, stage, global flags of this rank's owned points) of a
    conserved_to_primitives failure, for the cross-rank merge."""
    fl = rp.dev.stage_decode_flags(info.stage, params.gamma, rp.part.n_owned)
    return info.iteration, info.stage, rp.part.global_ids[: rp.part.n_owned], fl


def _raise_merged_decode(fails, n_global: int) -> None:
    """state.py:110-128 raised over the WHOLE state: the reference checks
    every point at once, so the failing (owned) points of all ranks that
    failed at the earliest (iteration, stage) are merged in global order."""
    first = min((it, st) for it, st, _, _ in fails)
    fl = np.zeros(n_global, dtype=np.uint8)
    for it, st, gid, f in fails:
        if (it, st) == first:
            fl[gid] |= f
    raise_decode_flags(fl, f"iteration {first[0]}: ")


_C2P = (_lib.CTX_C2P_DENSITY, _lib.CTX_C2P_PRESSURE)


def _check_depth(part: LocalPart, config) -> None:
    n_inner = config.n_inner if getattr(config, "order", 2) == 2 else 0
    if n_inner + 2 > part.depth:
        raise ValueError(f"n_inner {n_inner} needs a halo of depth {n_inner + 2}; the partition was built with "
                         f"depth {part.depth}")


def _raise_rank_error(rp: RankPart, params) -> None:
    info = _rank_error(rp)
    try:
        rp.dev.raise_positivity(info.context, info.stage, which=_lib.DIAG_LAST_RUN, mode=params.mode,
                                prefix=f"iteration {info.iteration}: ", gamma=params.gamma)
    except PositivityError as exc:
        idx = exc.indices
        if idx is not None and info.context >= _lib.CTX_WALL_TANGENT:
            idx = rp.part.global_ids[idx]  # point-level contexts: report global numbering
        raise PositivityError(str(exc), indices=idx) from None


TRANSPORTS = ("host", "peer")


def solve_group(config: SolverConfig, cloud, conn: Connectivity, nranks: int, initial_state: Primitives | None = None,
                devices=None, scheme: str = "bands", transport: str = "host"):
    """Partitioned solve in one process; returns (history, prims (4,n), U (4,n), converged).

    transport "host": kmf_run_group (the host moves the halo between the
    stages); "peer": the contexts are peer-linked (kmf_peer_link) and run
    concurrently with the device-side peer transport (kmf_run_linked)."""
    if transport not in TRANSPORTS:
        raise ValueError(f"transport must be one of {TRANSPORTS}")
    prims0 = (initial_state.copy() if initial_state is not None else initial_primitives(config, cloud))
    prims0.validate("initial state")
    devices = devices or [_lib.device_index()] * nranks
    owner = owner_map(cloud, nranks, scheme)
    ranks = [RankPart(conn, r, nranks, config.n_inner, devices[r], scheme=scheme, owner=owner) for r in range(nranks)]
    g = prims_array(prims0)
    for rp in ranks:
        rp.set_state(g)
    p = _params(config)
    handles = (C.c_void_p * nranks)(*[rp.dev.handle.value for rp in ranks])
    hist = np.zeros(config.n_outer)
    done, conv = C.c_int(0), C.c_int(0)
    if transport == "peer":
        _lib.check(_lib.lib().kmf_peer_link(handles, nranks), "kmf_peer_link")
        run = _lib.lib().kmf_run_linked
    else:
        run = _lib.lib().kmf_run_group
    rc = run(handles, nranks, C.byref(p), config.n_outer, _lib.dptr(hist), C.byref(done), C.byref(conv))
    if rc == _lib.KMF_EPEER:
        raise _lib.DeviceError("peer transport timed out; counters (pushes, bands, iterations | data | read | "
                               "limbs) per rank: " + "; ".join(str(peer_counters(rp)) for rp in ranks))
    if rc == _lib.KMF_EPOSITIVITY:
        # the reference raises at the earliest failing (iteration, stage)
        # over the whole cloud, and within a stage at its first raise site
        # (interior flux < wall < outer closures < decode: context order)
        failed = sorted(((rp, info) for rp in ranks for info in [_rank_error(rp)]
                         if info.code == _lib.KMF_EPOSITIVITY),
                        key=lambda f: (f[1].iteration, f[1].stage, f[1].context))
        first = (failed[0][1].iteration, failed[0][1].stage)
        earliest = [(rp, info) for rp, info in failed if (info.iteration, info.stage) == first]
        dec = [_decode_failures(rp, info, p) for rp, info in earliest if info.context in _C2P]
        if dec and len(dec) == len(earliest):
            _raise_merged_decode(dec, cloud.n_points)
        _raise_rank_error(earliest[0][0], p)
    _lib.check(rc, f"solve_group ({transport})")
    n = cloud.n_points
    prims, U = np.empty((4, n)), np.empty((4, n))
    for rp in ranks:
        gid, pr, u = rp.owned_state()
        prims[:, gid] = pr
        U[:, gid] = u
    return hist[: done.value], prims, U, bool(conv.value)


def peer_push_targets(part: LocalPart, recv_of: list) -> tuple:
    """Where this rank's halo pushes land (the kmf_peer_open lists): per
    peer in attach_partition's order (sorted peers), the peer's local halo
    slots for this rank's send list -- the peer's receive list for this
    rank, whose order the send list follows (exchange_send_lists).
    recv_of[p] is rank p's `recv` dict.  Returns (counts, slots) int64."""
    peers = sorted(set(part.send) | set(part.recv))
    dst = []
    for p in peers:
        d = np.asarray(recv_of[p].get(part.rank, np.empty(0)), dtype=np.int64) if p in part.send \
            else np.empty(0, np.int64)
        if d.size != (part.send[p].size if p in part.send else 0):
            raise ValueError(f"rank {p} receives {d.size} points from rank {part.rank}, which sends "
                             f"{part.send.get(p, np.empty(0)).size}")
        dst.append(d)
    counts = np.array([d.size for d in dst], dtype=np.int64)
    slots = np.ascontiguousarray(np.concatenate(dst) if dst else np.empty(0, np.int64), dtype=np.int64)
    return counts, slots


def peer_counters(rp: RankPart) -> list:
    """kmf_peer_counters of one rank (diagnostics)."""
    nr = rp.part.nranks
    out = (C.c_uint64 * (3 + 3 * nr))()
    _lib.check(_lib.lib().kmf_peer_counters(rp.dev.handle, out), "kmf_peer_counters")
    v = list(out)
    return [v[:3], v[3:3 + nr], v[3 + nr:3 + 2 * nr], v[3 + 2 * nr:]]


def exchange_send_lists(part: LocalPart, dist) -> None:
    """Fill part.send from the peers' receive lists: one object all-gather
    of halo global ids, instead of every rank recomputing every peer's halo
    (partition.send_lists_for, O(nranks) halo searches over the global
    stencil).  send[peer] lists this rank's local (owned) slots in the
    peer's receive order."""
    mine = {peer: part.global_ids[slots] for peer, slots in part.recv.items()}
    allrecv = [None] * part.nranks
    dist.all_gather_object(allrecv, mine)
    part.send = {peer: part.local_of_owned(np.asarray(r[part.rank])) for peer, r in enumerate(allrecv)
                 if peer != part.rank and part.rank in r}


RANK_TRANSPORTS = ("nccl", "peer")


class RankSolver:
    """This process's rank of a partitioned solve (torchrun, one GPU per
    process).  `dist` is an initialised torch.distributed module (plumbing:
    ids, handles, lists, errors).  transport "nccl": halo send/recv and the
    limb all-reduce by NCCL inside the iteration graph; "peer": the GPUs
    push the halo into each other's memory from the update kernel and
    all-gather the limbs over peer memory (CUDA IPC, csrc/kmf_peer.cuh)."""

    def __init__(self, conn: Connectivity, dist, n_inner: int = 3, device: int | None = None, scheme: str = "bands",
                 transport: str = "nccl"):
        if transport not in RANK_TRANSPORTS:
            raise ValueError(f"transport must be one of {RANK_TRANSPORTS}")
        self.rank, self.nranks = dist.get_rank(), dist.get_world_size()
        self.dist = dist
        self.transport = transport
        part = build_part(conn, self.rank, self.nranks, n_inner + 2, scheme)
        exchange_send_lists(part, dist)
        self.rp = RankPart(conn, self.rank, self.nranks, n_inner, device, part=part)
        if transport == "peer":
            self._open_peers()
            return
        uid = (C.c_char * 128)()
        if self.rank == 0:
            _lib.check(_lib.lib().kmf_nccl_get_unique_id(uid), "kmf_nccl_get_unique_id")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        uid = (C.c_char * 128).from_buffer_copy(box[0])
        _lib.check(_lib.lib().kmf_nccl_init(self.rp.dev.handle, uid, self.rank, self.nranks), "kmf_nccl_init")

    def _open_peers(self) -> None:
        """All-gather the ranks' IPC handles and receive lists, then map the
        peers (kmf_peer_open): this rank pushes its send list to peer p into
        the local slots of p's receive list for this rank."""
        L, part = _lib.lib(), self.rp.part
        h = (C.c_char * _lib.KMF_PEER_HANDLE_BYTES)()
        _lib.check(L.kmf_peer_handle(self.rp.dev.handle, h), "kmf_peer_handle")
        every = [None] * self.nranks
        self.dist.all_gather_object(every, (bytes(h), {p: np.asarray(s, np.int64) for p, s in part.recv.items()}))
        handles = (C.c_char * (_lib.KMF_PEER_HANDLE_BYTES * self.nranks)).from_buffer_copy(
            b"".join(e[0] for e in every))
        counts, slots = peer_push_targets(part, [e[1] for e in every])
        _lib.check(L.kmf_peer_open(self.rp.dev.handle, handles, _lib.i64ptr(counts), _lib.i64ptr(slots)),
                   "kmf_peer_open")

    @property
    def dev(self) -> DeviceConnectivity:
        return self.rp.dev

    def run(self, config: SolverConfig, prims_global: np.ndarray, n_iter: int):
        """Set the state and run; history is identical on every rank."""
        _check_depth(self.rp.part, config)
        self.rp.set_state(prims_global)
        p = _params(config)
        hist = np.zeros(max(n_iter, 1))
        done, conv = C.c_int(0), C.c_int(0)
        rc = _lib.lib().kmf_run(self.rp.dev.handle, C.byref(p), n_iter, _lib.dptr(hist), C.byref(done),
                                C.byref(conv))
        flags = [None] * self.nranks
        mine = None
        if rc == _lib.KMF_EPOSITIVITY:
            info = _rank_error(self.rp)
            mine = (int(info.context), _decode_failures(self.rp, info, p) if info.context in _C2P else None)
        self.dist.all_gather_object(flags, (rc, mine))
        if any(f[0] == _lib.KMF_EPOSITIVITY for f in flags):
            fails = [f[1] for f in flags if f[0] == _lib.KMF_EPOSITIVITY]
            if all(ctx in _C2P for ctx, _ in fails):
                _raise_merged_decode([d for _, d in fails], self.rp.part.n_global)
            if rc == _lib.KMF_EPOSITIVITY:
                _raise_rank_error(self.rp, p)
            raise PositivityError("positivity failure on another rank")
        _lib.check(rc, "kmf_run")
        return hist[: done.value], bool(conv.value)
