"""Partitioned device solve reproduces the single-domain solve bit for bit,
for both ownership schemes and every transport: the one-process group
runner with the host moving the halo ("host") or the contexts peer-linked
("peer": update kernels push into each other's halo, device counters order
the stages, limbs all-gathered over peer memory); multi-process NCCL and
multi-process peer transport (CUDA IPC), several ranks sharing one GPU."""

import numpy as np
import pytest

from conftest import perturbed_state
from paper_2108_07031_b200 import SolverConfig, solve
from paper_2108_07031_b200.dist import solve_group

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("transport", ["host", "peer"])
@pytest.mark.parametrize("scheme", ["bands", "sectors"])
@pytest.mark.parametrize("nranks", [2, 3])
def test_group_solve_bitwise(gpu, nranks, scheme, transport, small_naca, small_naca_conn):
    init = perturbed_state(small_naca)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=6)
    ref = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
    hist, prims, U, conv = solve_group(cfg, small_naca, small_naca_conn, nranks, initial_state=init, scheme=scheme,
                                       transport=transport)
    assert np.array_equal(hist, ref.residue_history)
    assert np.array_equal(prims, ref.primitives.as_array())
    assert np.array_equal(U, ref.conserved)


@pytest.mark.parametrize("transport", ["host", "peer"])
def test_group_solve_default_init_transonic(gpu, transport, small_naca, small_naca_conn):
    cfg = SolverConfig(mach=0.85, aoa_deg=1.0, n_outer=20)
    ref = solve(cfg, small_naca, small_naca_conn, instrument=False)
    hist, prims, _, _ = solve_group(cfg, small_naca, small_naca_conn, 2, transport=transport)
    assert np.array_equal(hist, ref.residue_history)
    assert np.array_equal(prims, ref.primitives.as_array())


@pytest.mark.parametrize("transport", ["host", "peer"])
def test_group_solve_convergence_stop(gpu, transport, small_naca, small_naca_conn):
    from paper_2108_07031_b200 import free_stream

    init = free_stream(0.63, 2.0, n=small_naca.n_points)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=30, convergence_tol=1e-6)
    hist, _, _, conv = solve_group(cfg, small_naca, small_naca_conn, 2, initial_state=init, transport=transport)
    assert conv and hist.shape == (1,)


@pytest.mark.parametrize("transport", ["host", "peer"])
def test_group_solve_positivity(gpu, transport, small_naca, small_naca_conn):
    from paper_2108_07031_b200 import PositivityError

    init = perturbed_state(small_naca, amp=-0.64)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=5, cfl=1.0)
    with pytest.raises(PositivityError) as exc:
        solve_group(cfg, small_naca, small_naca_conn, 2, initial_state=init, transport=transport)
    assert str(exc.value).startswith("iteration 1: conserved_to_primitives: nonpositive density")
    assert list(exc.value.indices) == [880]


def test_nccl_rank_solver_world_one(gpu, small_naca, small_naca_conn, tmp_path):
    """The NCCL transport inside the iteration graph on one rank: kmf_nccl_init
    (+ its eager warm-up), the partitioned update that defers the iteration
    close, the limb all-reduce and k_close captured in the graph -- the same
    history and state as the single-domain solve, bit for bit."""
    import os

    import torch.distributed as dist

    from paper_2108_07031_b200.dist import RankSolver

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    store = dist.FileStore(str(tmp_path / "store"), 1)
    dist.init_process_group("gloo", store=store, rank=0, world_size=1)
    try:
        init = perturbed_state(small_naca)
        cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=6)
        ref = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
        rs = RankSolver(small_naca_conn, dist, n_inner=cfg.n_inner)
        hist, conv = rs.run(cfg, init.as_array(), cfg.n_outer)
        gid, prims, _ = rs.rp.owned_state()
        assert np.array_equal(hist, ref.residue_history)
        assert np.array_equal(prims, ref.primitives.as_array()[:, gid])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["host", "peer"])
@pytest.mark.parametrize("mode", ["fused", "split4"])
def test_group_solve_first_order_and_split4(gpu, mode, transport, small_naca, small_naca_conn):
    """First-order scheme (no q-gradient kernels: the flux's own interior
    range) and split4 under the partition schedule."""
    init = perturbed_state(small_naca)
    for order in (1, 2):
        cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=4, mode=mode, order=order)
        ref = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
        hist, prims, _, _ = solve_group(cfg, small_naca, small_naca_conn, 3, initial_state=init, scheme="sectors",
                                        transport=transport)
        assert np.array_equal(hist, ref.residue_history)
        assert np.array_equal(prims, ref.primitives.as_array())


def test_peer_linked_continuation(gpu, small_naca, small_naca_conn):
    """kmf_run_linked twice on the same peer-linked contexts (the second run
    seeds by refreshing q and pushing the send points: the continued-run
    protocol) equals one 7-iteration solve; the host-exchange group runner
    refuses peer-linked contexts."""
    import ctypes as C

    from paper_2108_07031_b200 import _lib
    from paper_2108_07031_b200.dist import RankPart
    from paper_2108_07031_b200.solver import _params

    init = perturbed_state(small_naca)
    ranks = [RankPart(small_naca_conn, r, 3, n_inner=3, scheme="sectors") for r in range(3)]
    for rp in ranks:
        rp.set_state(init.as_array())
    h = (C.c_void_p * 3)(*[rp.dev.handle.value for rp in ranks])
    _lib.check(_lib.lib().kmf_peer_link(h, 3), "link")
    one = _params(SolverConfig(mach=0.63, n_outer=1))
    assert _lib.lib().kmf_run_group(h, 3, C.byref(one), 1, None, None, None) == _lib.KMF_EINVAL
    # ... and not alone either (its peers would never start): refused, not a 30 s deadline
    d0, c0 = C.c_int(0), C.c_int(0)
    assert _lib.lib().kmf_run(ranks[0].dev.handle, C.byref(one), 1, None, C.byref(d0), C.byref(c0)) == _lib.KMF_EINVAL
    ref = solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=7), small_naca, small_naca_conn, initial_state=init,
                instrument=False)
    got = []
    for n in (3, 4):
        cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=n)
        hist = np.zeros(n)
        done, conv = C.c_int(0), C.c_int(0)
        _lib.check(_lib.lib().kmf_run_linked(h, 3, C.byref(_params(cfg)), n, _lib.dptr(hist), C.byref(done),
                                             C.byref(conv)), "linked")
        assert done.value == n
        got.extend(hist.tolist())
    assert np.array_equal(np.array(got), ref.residue_history)
    for rp in ranks:
        gid, prims, _ = rp.owned_state()
        assert np.array_equal(prims, ref.primitives.as_array()[:, gid])


def test_group_rejects_shallow_halo(gpu, small_naca, small_naca_conn):
    """A partition built for n_inner = 1 (depth 3) cannot run n_inner = 3:
    the halo gradients would be inexact (ValueError, not silent drift)."""
    import ctypes as C

    from paper_2108_07031_b200 import _lib
    from paper_2108_07031_b200.dist import RankPart
    from paper_2108_07031_b200.solver import _params

    ranks = [RankPart(small_naca_conn, r, 2, n_inner=1) for r in range(2)]
    init = perturbed_state(small_naca).as_array()
    for rp in ranks:
        rp.set_state(init)
    p = _params(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=2, n_inner=3))
    h = (C.c_void_p * 2)(*[rp.dev.handle.value for rp in ranks])
    hist = np.zeros(2)
    done, conv = C.c_int(0), C.c_int(0)
    rc = _lib.lib().kmf_run_group(h, 2, C.byref(p), 2, _lib.dptr(hist), C.byref(done), C.byref(conv))
    assert rc == _lib.KMF_EINVAL
    # one sweep fits the depth-3 halo and stays bitwise
    cfg1 = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=3, n_inner=1)
    ref = solve(cfg1, small_naca, small_naca_conn, initial_state=perturbed_state(small_naca), instrument=False)
    p1 = _params(cfg1)
    hist = np.zeros(3)
    _lib.check(_lib.lib().kmf_run_group(h, 2, C.byref(p1), 3, _lib.dptr(hist), C.byref(done), C.byref(conv)), "group")
    assert np.array_equal(hist, ref.residue_history)


def _rank_worker(rank, world, port, scheme, order, transport, q):
    import os

    import torch.distributed as dist

    from paper_2108_07031_b200 import SolverConfig as Cfg
    from paper_2108_07031_b200 import _lib, build_stencils, generate_naca_cloud
    from paper_2108_07031_b200.dist import RankSolver
    from paper_2108_07031_b200.state import prims_array

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    ndev = _lib.lib().kmf_device_count()
    if ndev < world and transport == "nccl":
        # fewer GPUs than ranks: each rank reports its own host, so NCCL
        # skips its same-host duplicate-device check and connects the ranks
        # through its socket transport (loopback) -- the same NCCL calls,
        # graphs and schedule as on NVLink, only the wire differs
        os.environ["NCCL_HOSTID"] = f"kmf-test-host-{rank}"
        os.environ["NCCL_SOCKET_IFNAME"] = "lo"
        os.environ["NCCL_IB_DISABLE"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
        conn = build_stencils(cloud)
        init = perturbed_state(cloud)
        cfg = Cfg(mach=0.63, aoa_deg=2.0, n_outer=6, order=order)
        rs = RankSolver(conn, dist, n_inner=3, device=rank % ndev, scheme=scheme, transport=transport)
        hist, conv = rs.run(cfg, prims_array(init), cfg.n_outer)
        gid, prims, _ = rs.rp.owned_state()
        # the streamed-cases path on the same communicator: two cases from
        # the same local state, each must equal the run above
        from paper_2108_07031_b200.solver import _params

        local = np.ascontiguousarray(prims_array(init)[:, rs.rp.part.global_ids])
        outs, hc, _, _, st = rs.dev.run_cases([_params(cfg)] * 2, [local, local], cfg.n_outer)
        no = rs.rp.part.n_owned
        cases_ok = st == [0, 0] and all(np.array_equal(hc[k], hist) and np.array_equal(outs[k][:, :no], prims)
                                        for k in range(2))
        q.put((rank, hist, gid, prims, None if cases_ok else "run_cases differs from run"))
    except Exception as exc:  # reported, never left hanging on the queue
        q.put((rank, None, None, None, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("world,scheme,order", [(2, "sectors", 2), (3, "bands", 2), (4, "sectors", 1)])
def test_ranks_bitwise(gpu, world, scheme, order, transport, small_naca, small_naca_conn):
    """N processes, the halo exchange and residue reduction inside the
    iteration graph -- NCCL (send/recv forked beside the interior pass,
    limb all-reduce) or the peer transport (CUDA IPC mappings of the peers'
    q and flag blocks, halo pushed by the update kernel) -- bitwise the
    single-domain solve.  With fewer GPUs than ranks the ranks share a GPU
    (NCCL over its socket transport, see _rank_worker; IPC on one device)."""
    import socket

    import torch.multiprocessing as mp

    from paper_2108_07031_b200.state import prims_array

    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, scheme, order, transport, q))
             for r in range(world)]
    for p_ in procs:
        p_.start()
    try:
        out = [q.get(timeout=300) for _ in range(world)]
    finally:
        for p_ in procs:
            p_.join(timeout=60)
            if p_.is_alive():
                p_.kill()
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=6, order=order)
    ref = solve(cfg, small_naca, small_naca_conn, initial_state=perturbed_state(small_naca), instrument=False)
    seen = np.zeros(small_naca.n_points, dtype=int)
    for rank, hist, gid, prims, err in out:
        assert err is None, f"rank {rank}: {err}"
        assert np.array_equal(hist, ref.residue_history)
        assert np.array_equal(prims, prims_array(ref.primitives)[:, gid])
        seen[gid] += 1
    assert np.all(seen == 1)  # the owned sets partition the cloud


def _deadline_worker(rank, world, port, q):
    import os
    import time as _t

    import torch.distributed as dist

    from paper_2108_07031_b200 import SolverConfig as Cfg
    from paper_2108_07031_b200 import _lib, build_stencils, generate_naca_cloud
    from paper_2108_07031_b200.dist import RankSolver
    from paper_2108_07031_b200.state import prims_array

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["KMF_PEER_TIMEOUT_S"] = "2"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
        conn = build_stencils(cloud)
        rs = RankSolver(conn, dist, n_inner=3, device=0, scheme="sectors", transport="peer")
        res = None
        if rank == 0:  # rank 1 never runs: rank 0 must come back with KMF_EPEER, not hang
            t0 = _t.perf_counter()
            try:
                rs.run(Cfg(mach=0.63, aoa_deg=2.0, n_outer=2), prims_array(perturbed_state(cloud)), 2)
                res = ("returned", _t.perf_counter() - t0)
            except _lib.DeviceError as e:
                res = (str(e), _t.perf_counter() - t0)
            # the context is now unusable (its ranks' counters disagree): refused at once
            try:
                rs.run(Cfg(mach=0.63, aoa_deg=2.0, n_outer=1), prims_array(perturbed_state(cloud)), 1)
            except _lib.DeviceError as e:
                res = res + ("re-create" in str(e),)
        else:  # the collective RankSolver.run ends with (error flags), without running
            for _ in range(2):
                flags = [None] * world
                dist.all_gather_object(flags, (0, None))
            res = ("idle", 0.0)
        dist.barrier()
        q.put((rank, res))
    except Exception as exc:
        q.put((rank, (repr(exc), -1.0)))
    finally:
        dist.destroy_process_group()


def test_peer_deadline_instead_of_hang(gpu):
    """A rank whose peer never runs gets KMF_EPEER after the wait deadline
    (2 s here) -- the GPU and the process come back instead of spinning."""
    import socket

    import torch.multiprocessing as mp

    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_deadline_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    try:
        out = dict(q.get(timeout=180) for _ in range(2))
    finally:
        for p_ in procs:
            p_.join(timeout=60)
            if p_.is_alive():
                p_.kill()
    msg, took, refused = out[0]
    assert "code 5" in msg and "did not arrive" in msg, msg
    assert 1.5 < took < 60 and refused


def test_solve_on_several_devices(gpu, small_naca, small_naca_conn):
    """solve(..., devices=[...]) partitions the cloud over the listed devices
    (here the same GPU three times) and runs the ranks concurrently over the
    peer transport: bitwise the one-GPU solve, PositivityError included."""
    from paper_2108_07031_b200 import PositivityError

    init = perturbed_state(small_naca)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=10)
    ref = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
    got = solve(cfg, small_naca, small_naca_conn, initial_state=init, devices=[0, 0, 0])
    assert np.array_equal(got.residue_history, ref.residue_history)
    assert np.array_equal(got.primitives.as_array(), ref.primitives.as_array())
    assert np.array_equal(got.conserved, ref.conserved)
    assert got.iterations == 10 and got.wall_seconds > 0
    bad = perturbed_state(small_naca, amp=-0.64)
    cfg1 = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=5, cfl=1.0)
    with pytest.raises(PositivityError) as e1:
        solve(cfg1, small_naca, small_naca_conn, initial_state=bad, instrument=False)
    with pytest.raises(PositivityError) as e2:
        solve(cfg1, small_naca, small_naca_conn, initial_state=bad, devices=[0, 0])
    assert str(e1.value) == str(e2.value) and list(e1.value.indices) == list(e2.value.indices)


@pytest.mark.parametrize("gamma", [5.0 / 3.0, 1.3])
def test_group_peer_other_gammas(gpu, gamma, small_naca, small_naca_conn):
    """The gamma-specialised flux / boundary kernels (GK=2 at 5/3, the
    generic GK=0 at 1.3) under the peer transport: bitwise one domain."""
    init = perturbed_state(small_naca, gamma=gamma)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=8, gamma=gamma)
    ref = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
    hist, prims, _, _ = solve_group(cfg, small_naca, small_naca_conn, 3, initial_state=init, scheme="sectors",
                                    transport="peer")
    assert np.array_equal(hist, ref.residue_history)
    assert np.array_equal(prims, ref.primitives.as_array())
