"""Multi-GPU domain decomposition, checked on the CPU with the oracle.

A partitioned solve -- every rank runs the single-GPU arithmetic on its
owned points plus an (n_inner + 2)-layer halo, exchanging q for the halo
once per RK stage and summing the residue exactly -- must reproduce the
global solve bit for bit.  The exchange runs in-process and, for
world_size 2, over torch.distributed gloo (the same protocol the NCCL
transport implements on the GPUs).
"""

import math
import os
import socket

import numpy as np
import pytest

from conftest import fs_vec, perturbed_state
from oracle import oracle as O
from paper_2108_07031_b200.geometry import Connectivity, StencilSet, _select
from paper_2108_07031_b200.partition import (
    build_part,
    build_parts,
    halo_layers,
    owner_map,
    owner_ranges,
    send_lists_for,
    stage_ranges,
)

DEPTH = 5  # n_inner 3 + 2


def flux_view(conn: Connectivity, n_owned: int) -> Connectivity:
    """Same local connectivity with stencils only on owned rows (what the
    device kernels restrict the flux / boundary / update launches to)."""
    f = conn.full
    keep = np.arange(f.n_owners) < n_owned
    cnt = np.where(keep, np.diff(f.ptr), 0)
    ptr = np.concatenate([[0], np.cumsum(cnt)])
    e = np.arange(ptr[-1]) + np.repeat(f.ptr[:-1][keep] - ptr[:-1][keep], cnt[keep])
    full = StencilSet(ptr=ptr, idx=f.idx[e], dx=f.dx[e], dy=f.dy[e])
    split = {"x+": _select(full, full.dx <= 0.0), "x-": _select(full, full.dx >= 0.0),
             "y+": _select(full, full.dy <= 0.0), "y-": _select(full, full.dy >= 0.0)}
    det_safe = {k: np.where(conn.cloud.flag == 0, s.det, 1.0) for k, s in split.items()}
    for k in det_safe:
        det_safe[k][~keep] = 1.0
    return Connectivity(cloud=conn.cloud, full=full, split=split, d_min=conn.d_min, d_mean=conn.d_mean,
                        wall_frame=conn.wall_frame, outer_frame=conn.outer_frame, det_safe=det_safe)


class RankState:
    def __init__(self, part, init_global, fs):
        self.p = part
        self.pk = O.Packed(part.conn)
        self.pkf = O.Packed(flux_view(part.conn, part.n_owned))
        self.fs = fs
        self.prims = init_global[:, part.global_ids].copy()
        self.q = O.primitives_to_q(self.prims)
        self.U = O.primitives_to_conserved(self.prims)

    def owned(self, a):
        return a[:, : self.p.n_owned]

    def stage(self, stage, U_outer, dt):
        qx, qy, _ = O.q_derivatives(self.pk, self.q, 3)
        R = O.flux_residual(self.pkf, self.q, qx, qy)
        R = O.apply_boundary(self.pkf, self.q, qx, qy, self.fs, R)
        no = self.p.n_owned
        Un = O.state_update_rk(U_outer[:, :no], self.U[:, :no], stage, dt[:no], R[:, :no])
        self.U[:, :no] = Un
        self.prims[:, :no] = O.conserved_to_primitives(Un)
        self.q[:, :no] = O.primitives_to_q(self.prims[:, :no])


def global_reference(conn, init, fs, iters):
    hist, prims, U, _, _ = O.solve(O.Packed(conn), init, fs, iters)
    return hist, prims


def test_layers_cover_the_dependency_cone(small_naca_conn):
    n = small_naca_conn.cloud.n_points
    b = owner_ranges(n, 3)
    layers = halo_layers(small_naca_conn.full, np.arange(b[1], b[2]), DEPTH)
    allpts = np.concatenate(layers)
    assert np.unique(allpts).size == allpts.size
    # every neighbour of layers 0..DEPTH-1 is inside the local set
    inside = np.zeros(n, dtype=bool)
    inside[allpts] = True
    f = small_naca_conn.full
    for L in layers[:-1]:
        for i in L[:: max(1, L.size // 50)]:
            assert inside[f.neighbors(i)].all()


@pytest.mark.parametrize("scheme", ["bands", "sectors"])
def test_send_lists_match(small_naca_conn, scheme):
    parts = build_parts(small_naca_conn, 3, DEPTH, scheme)
    for p in parts:
        ref = send_lists_for(small_naca_conn, p)
        assert ref.keys() == p.send.keys()
        for peer, s in p.send.items():
            assert np.array_equal(ref[peer], s)
            assert np.array_equal(p.global_ids[s], parts[peer].global_ids[parts[peer].recv[p.rank]])


def test_owner_maps_are_balanced_partitions(small_naca):
    n = small_naca.n_points
    for scheme in ("bands", "sectors"):
        own = owner_map(small_naca, 4, scheme)
        counts = np.bincount(own, minlength=4)
        assert counts.sum() == n and counts.max() - counts.min() <= 1


@pytest.mark.parametrize("scheme", ["bands", "sectors"])
def test_local_order_puts_deep_points_first(small_naca_conn, scheme):
    """Owned slots are ordered by depth (forward hops to the nearest halo
    point): every prefix interior_end[k] holds exactly the owned points of
    depth >= k, checked against a direct BFS on the global stencil."""
    part = build_part(small_naca_conn, 1, 3, DEPTH, scheme)
    f = small_naca_conn.full
    n = f.n_owners
    owner = owner_map(small_naca_conn.cloud, 3, scheme)
    # forward depth by brute force: d(p) = 1 + min_{j in N(p)} d(j), d = 0 off-rank
    d = np.where(owner == 1, 99, 0)
    for _ in range(DEPTH + 2):
        for i in np.flatnonzero(owner == 1):
            d[i] = min(d[i], 1 + d[f.neighbors(i)].min())
    d = np.minimum(d, DEPTH + 1)
    gid = part.global_ids[: part.n_owned]
    assert np.all(np.diff(d[gid]) <= 0)  # deepest first
    for k in range(DEPTH + 2):
        assert part.interior_end[k] == int((d[gid] >= k).sum())


def _np_first_order(f, q):
    """lsq.py:164-175 restated with np.bincount (CSR-order sums)."""
    n = f.n_owners
    owner = np.repeat(np.arange(n), np.diff(f.ptr))
    dq = q[:, f.idx] - q[:, owner]
    sx = np.stack([np.bincount(owner, weights=f.dx * dq[k], minlength=n) for k in range(4)])
    sy = np.stack([np.bincount(owner, weights=f.dy * dq[k], minlength=n) for k in range(4)])
    with np.errstate(invalid="ignore", divide="ignore"):
        return (f.syy * sx - f.sxy * sy) / f.det, (f.sxx * sy - f.sxy * sx) / f.det


def _np_sweep(f, q, qx, qy):
    """lsq.py:214-227 restated with np.bincount."""
    n = f.n_owners
    owner = np.repeat(np.arange(n), np.diff(f.ptr))
    ti = q[:, f.idx] - 0.5 * (f.dx * qx[:, f.idx] + f.dy * qy[:, f.idx])
    t0 = q[:, owner] - 0.5 * (f.dx * qx[:, owner] + f.dy * qy[:, owner])
    dq = ti - t0
    sx = np.stack([np.bincount(owner, weights=f.dx * dq[k], minlength=n) for k in range(4)])
    sy = np.stack([np.bincount(owner, weights=f.dy * dq[k], minlength=n) for k in range(4)])
    with np.errstate(invalid="ignore", divide="ignore"):
        return (f.syy * sx - f.sxy * sy) / f.det, (f.sxx * sy - f.sxy * sx) / f.det


@pytest.mark.parametrize("scheme", ["bands", "sectors"])
@pytest.mark.parametrize("n_inner", [0, 1, 3])
def test_interior_band_schedule_reads_no_pending_halo(small_naca, small_naca_conn, scheme, n_inner):
    """The device's per-stage schedule (stage_ranges): the interior pass runs
    while the halo q of this stage is still in flight -- poisoned with NaN
    here -- and writes only its ranges; the band pass completes the levels
    after the exchange.  Every level on its valid extent must equal the
    unsplit computation bit for bit (a single read of pending data would
    show up as NaN), and every flux row of the interior pass must read only
    gradients the interior pass produced."""
    part = build_part(small_naca_conn, 1, 3, DEPTH, scheme)
    f = part.conn.full
    q = O.primitives_to_q(perturbed_state(small_naca).as_array()[:, part.global_ids])
    q_pending = q.copy()
    q_pending[:, part.n_owned:] = np.nan
    sched = dict((name, (a, b)) for name, a, b in stage_ranges(part, n_inner))
    names = ["first_order"] + [f"sweep{s}" for s in range(1, n_inner + 1)] if n_inner else []
    levels = [(np.full_like(q, np.nan), np.full_like(q, np.nan)) for _ in names]

    def run_pass(qq, which):
        for k, name in enumerate(names):
            lo, hi = sched[name][which]
            gx, gy = _np_first_order(f, qq) if k == 0 else _np_sweep(f, qq, *levels[k - 1])
            levels[k][0][:, lo:hi] = gx[:, lo:hi]
            levels[k][1][:, lo:hi] = gy[:, lo:hi]

    run_pass(q_pending, 0)
    # flux interior rows read neighbours' final gradients: all produced already
    lo, hi = sched["flux"][0]
    for i in range(lo, hi):
        nb = np.append(f.neighbors(i), i)
        assert np.all(np.isfinite(q_pending[:, nb]))
        if names:
            assert np.all(np.isfinite(levels[-1][0][:, nb]))
    run_pass(q, 1)
    assert sched["flux"][1][1] == part.n_owned
    gx, gy = None, None
    for k, name in enumerate(names):
        gx, gy = _np_first_order(f, q) if k == 0 else _np_sweep(f, q, gx, gy)
        end = sched[name][1][1]
        assert end == part.layer_counts[DEPTH - 1 - k]
        assert np.array_equal(levels[k][0][:, :end], gx[:, :end]) and np.array_equal(levels[k][1][:, :end], gy[:, :end])


@pytest.mark.parametrize("scheme", ["bands", "sectors"])
@pytest.mark.parametrize("nranks", [2, 3])
def test_partitioned_solve_is_bitwise_global(nranks, scheme, small_naca, small_naca_conn):
    fs = fs_vec(0.63, 2.0)
    init = perturbed_state(small_naca).as_array()
    iters = 3
    ref_hist, ref_prims = global_reference(small_naca_conn, init, fs, iters)
    parts = build_parts(small_naca_conn, nranks, DEPTH, scheme)
    ranks = [RankState(p, init, fs) for p in parts]
    n = small_naca.n_points
    hist = []
    for it in range(iters):
        dts = [O.local_timestep(r.pk, r.prims, 0.2) for r in ranks]
        U_outer = [r.U.copy() for r in ranks]
        for stage in (1, 2, 3, 4):
            for r, dt, Uo in zip(ranks, dts, U_outer):
                r.stage(stage, Uo, dt)
            for r in ranks:  # halo exchange of q
                for peer, slots in r.p.recv.items():
                    r.q[:, slots] = ranks[peer].q[:, parts[peer].send[r.p.rank]]
        drho2 = np.concatenate([(r.U[0, : r.p.n_owned] - Uo[0, : r.p.n_owned]) ** 2 for r, Uo in zip(ranks, U_outer)])
        hist.append(math.sqrt(math.fsum(drho2.tolist()) / n))
    assert np.array_equal(np.array(hist), ref_hist)
    got = np.empty_like(ref_prims)
    for r in ranks:
        got[:, r.p.global_ids[: r.p.n_owned]] = r.owned(r.prims)
    assert np.array_equal(got, ref_prims)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from conftest import fs_vec as fsv, perturbed_state as ps
    from paper_2108_07031_b200 import build_stencils, generate_naca_cloud

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
    conn = build_stencils(cloud)
    part = build_part(conn, rank, world, DEPTH)
    part.send = send_lists_for(conn, part)
    r = RankState(part, ps(cloud).as_array(), fsv(0.63, 2.0))
    hist = []
    for it in range(2):
        dt = O.local_timestep(r.pk, r.prims, 0.2)
        Uo = r.U.copy()
        for stage in (1, 2, 3, 4):
            r.stage(stage, Uo, dt)
            reqs, bufs = [], {}
            for peer, slots in part.send.items():
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(r.q[:, slots])), peer))
            for peer, slots in part.recv.items():
                bufs[peer] = torch.empty((4, slots.size), dtype=torch.float64)
                reqs.append(dist.irecv(bufs[peer], peer))
            for q_ in reqs:
                q_.wait()
            for peer, slots in part.recv.items():
                r.q[:, slots] = bufs[peer].numpy()
        # exact residue: gather the owned drho^2 values (order-free fsum)
        mine = torch.from_numpy((r.U[0, : part.n_owned] - Uo[0, : part.n_owned]) ** 2)
        sizes = [None] * world
        dist.all_gather_object(sizes, mine.numel())
        chunks = [torch.empty(s, dtype=torch.float64) for s in sizes]
        dist.all_gather(chunks, mine)
        hist.append(math.sqrt(math.fsum(torch.cat(chunks).tolist()) / cloud.n_points))
    out[rank] = (hist, r.owned(r.prims).copy(), part.global_ids[: part.n_owned].copy())
    dist.destroy_process_group()


def test_gloo_two_ranks_bitwise_global(small_naca, small_naca_conn):
    import torch.multiprocessing as mp

    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gloo_worker, args=(2, port, out), nprocs=2, join=True)
    fs = fs_vec(0.63, 2.0)
    ref_hist, ref_prims = global_reference(small_naca_conn, perturbed_state(small_naca).as_array(), fs, 2)
    for rank in (0, 1):
        hist, prims, gid = out[rank]
        assert np.array_equal(np.array(hist), ref_hist)
        assert np.array_equal(prims, ref_prims[:, gid])


def _sendlist_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2108_07031_b200 import build_stencils, generate_naca_cloud
    from paper_2108_07031_b200.dist import exchange_send_lists

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    conn = build_stencils(generate_naca_cloud(80, 30, 1.15, 20.0))
    part = build_part(conn, rank, world, DEPTH)
    exchange_send_lists(part, dist)
    out[rank] = {k: v.copy() for k, v in part.send.items()}
    dist.destroy_process_group()


def test_gloo_send_lists_from_peer_receive_lists(small_naca_conn):
    """dist.exchange_send_lists (all-gather of receive lists) == the
    per-peer halo recomputation of send_lists_for, on 3 gloo ranks."""
    import torch.multiprocessing as mp

    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sendlist_worker, args=(3, port, out), nprocs=3, join=True)
    for rank in range(3):
        ref = send_lists_for(small_naca_conn, build_part(small_naca_conn, rank, 3, DEPTH))
        assert out[rank].keys() == ref.keys()
        for peer in ref:
            assert np.array_equal(out[rank][peer], ref[peer])


def _setup_worker(rank, world, port, out):
    import sys

    import torch.distributed as dist

    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
    import bench

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cloud, conn, cfg, init = bench.setup("c1", dist, rank)
    out[rank] = (np.asarray(conn.full.idx[::97]).copy(), np.asarray(conn.split["y-"].sxx[::13]).copy(),
                 init.as_array()[:, ::29].copy(), cfg.mach)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_shared_setup_store():
    """bench.setup under 2 ranks: rank 0 builds, both map the /dev/shm store;
    every rank sees the same connectivity and initial state as a direct build."""
    import sys

    import torch.multiprocessing as mp

    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
    import bench

    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_setup_worker, args=(2, port, out), nprocs=2, join=True)
    cloud, conn, cfg, init = bench.build_config("c1")
    for rank in (0, 1):
        idx, sxx, ini, mach = out[rank]
        assert np.array_equal(idx, conn.full.idx[::97])
        assert np.array_equal(sxx, conn.split["y-"].sxx[::13])
        assert np.array_equal(ini, init.as_array()[:, ::29]) and mach == cfg.mach


def test_oracle_n_act_equals_owned_flux_view(small_naca_conn, small_naca):
    """oracle n_act (flux and residue on a partition's owned rows, used for
    the bounded CPU samples of bench.py) == the owned-row flux view."""
    part = build_part(small_naca_conn, 1, 3, DEPTH)
    init = perturbed_state(small_naca).as_array()[:, part.global_ids]
    pk = O.Packed(part.conn)
    pk.c.n_act = part.n_owned
    ref = O.Packed(flux_view(part.conn, part.n_owned))
    q = O.primitives_to_q(init)
    qx, qy, _ = O.q_derivatives(pk, q, 3)
    a = O.flux_residual(pk, q, qx, qy)
    b = O.flux_residual(ref, q, qx, qy)
    no = part.n_owned
    assert np.array_equal(a[:, :no], b[:, :no]) and not a[:, no:].any()
    # a sampled solve runs without touching the (garbage) halo fluxes
    hist, _, _, its, _ = O.solve(pk, init, fs_vec(0.63, 2.0), 2)
    assert its == 2 and np.all(np.isfinite(hist))


@pytest.mark.parametrize("scheme", ["bands", "sectors"])
def test_peer_push_targets_reproduce_the_exchange(small_naca_conn, scheme):
    """The peer transport's push map (dist.peer_push_targets: each send
    point's destination slot in the peer's halo) writes exactly what the
    receive-side halo exchange writes, for 3 ranks of either ownership."""
    from paper_2108_07031_b200.dist import peer_push_targets

    parts = build_parts(small_naca_conn, 3, DEPTH, scheme)
    rng = np.random.default_rng(7)
    q = [rng.standard_normal((4, p.global_ids.size)) for p in parts]
    want = [x.copy() for x in q]
    for r, p in enumerate(parts):  # receive side: q[:, recv[peer]] = peer q[:, peer.send[r]]
        for peer, slots in p.recv.items():
            want[r][:, slots] = q[peer][:, parts[peer].send[r]]
    got = [x.copy() for x in q]
    recv_of = [p.recv for p in parts]
    for r, p in enumerate(parts):  # push side, in attach_partition's peer order
        counts, slots = peer_push_targets(p, recv_of)
        off = 0
        for peer, cnt in zip(sorted(set(p.send) | set(p.recv)), counts):
            if cnt:
                got[peer][:, slots[off:off + cnt]] = q[r][:, p.send[peer]]
            off += cnt
    for r in range(3):
        assert np.array_equal(got[r], want[r])
        # every halo slot is written by exactly one push
        n_halo = parts[r].global_ids.size - parts[r].n_owned
        assert sum(v.size for v in parts[r].recv.values()) == n_halo
