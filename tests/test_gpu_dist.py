"""Partitioned device solve (2 and 3 ranks on one GPU through the group
runner) reproduces the single-domain solve bit for bit."""

import numpy as np
import pytest

from conftest import perturbed_state
from paper_2108_07031_b200 import SolverConfig, solve
from paper_2108_07031_b200.dist import solve_group

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nranks", [2, 3])
def test_group_solve_bitwise(gpu, nranks, small_naca, small_naca_conn):
    init = perturbed_state(small_naca)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=6)
    ref = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
    hist, prims, U, conv = solve_group(cfg, small_naca, small_naca_conn, nranks, initial_state=init)
    assert np.array_equal(hist, ref.residue_history)
    assert np.array_equal(prims, ref.primitives.as_array())
    assert np.array_equal(U, ref.conserved)


def test_group_solve_default_init_transonic(gpu, small_naca, small_naca_conn):
    cfg = SolverConfig(mach=0.85, aoa_deg=1.0, n_outer=20)
    ref = solve(cfg, small_naca, small_naca_conn, instrument=False)
    hist, prims, _, _ = solve_group(cfg, small_naca, small_naca_conn, 2)
    assert np.array_equal(hist, ref.residue_history)
    assert np.array_equal(prims, ref.primitives.as_array())


def test_group_solve_convergence_stop(gpu, small_naca, small_naca_conn):
    from paper_2108_07031_b200 import free_stream

    init = free_stream(0.63, 2.0, n=small_naca.n_points)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=30, convergence_tol=1e-6)
    hist, _, _, conv = solve_group(cfg, small_naca, small_naca_conn, 2, initial_state=init)
    assert conv and hist.shape == (1,)


def test_group_solve_positivity(gpu, small_naca, small_naca_conn):
    from paper_2108_07031_b200 import PositivityError

    init = perturbed_state(small_naca, amp=-0.64)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=5, cfl=1.0)
    with pytest.raises(PositivityError) as exc:
        solve_group(cfg, small_naca, small_naca_conn, 2, initial_state=init)
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
