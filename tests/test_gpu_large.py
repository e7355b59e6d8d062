"""Full-size parity (BASELINE config 3: NACA 0012 2.5M points, M 0.85,
AoA 1): the device path against the CPU oracle on the whole cloud.

Sizes where the oracle still finishes in seconds: q-gradients (first order
+ 3 sweeps) bitwise on the initial state, and three whole outer iterations
(residue history <= 1e-10 relative, final primitives rtol 1e-10 / atol
1e-12).  The connectivity comes from the native builder (bit-exact with the
reference builder, tests/test_builder.py).
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2108_07031_b200 import (
    SolverConfig,
    build_stencils,
    compute_q_derivatives,
    free_stream,
    generate_naca_cloud,
    initial_primitives,
    primitives_to_q,
    solve,
)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    cloud = generate_naca_cloud(3160, 790, 1.00734, 20.0)
    conn = build_stencils(cloud)
    cfg = SolverConfig(mach=0.85, aoa_deg=1.0, n_outer=3)
    import os

    O.set_threads(os.cpu_count() or 1)
    return cloud, conn, cfg, initial_primitives(cfg, cloud), O.Packed(conn)


def test_c3_q_gradients_bitwise(gpu, c3):
    cloud, conn, cfg, init, pk = c3
    q = primitives_to_q(init)
    g = compute_q_derivatives(q, conn, 3)
    qx, qy, res = O.q_derivatives(pk, q, 3)
    assert np.array_equal(g.qx, qx) and np.array_equal(g.qy, qy)


def test_c3_three_iterations_match_oracle(gpu, c3):
    cloud, conn, cfg, init, pk = c3
    res = solve(cfg, cloud, conn, initial_state=init, instrument=False)
    fs = free_stream(cfg.mach, cfg.aoa_deg)
    hist, prims, _, _, _ = O.solve(pk, init.as_array(), [fs.rho[0], fs.u1[0], fs.u2[0], fs.p[0]], cfg.n_outer)
    assert res.iterations == 3
    rel = np.abs(res.residue_history - hist) / hist
    assert rel.max() <= 1e-10, rel
    assert np.allclose(res.primitives.as_array(), prims, rtol=1e-10, atol=1e-12)


def test_c3_fused_equals_split4_bitwise(gpu, c3):
    """At 2.5M points the HBM-streaming kernel variants are active (index
    staging, flux prefetch + lean arithmetic); split4 must still equal fused."""
    cloud, conn, cfg, init, _ = c3
    a = solve(SolverConfig(mach=0.85, aoa_deg=1.0, n_outer=2, mode="fused"), cloud, conn, initial_state=init,
              instrument=False)
    b = solve(SolverConfig(mach=0.85, aoa_deg=1.0, n_outer=2, mode="split4"), cloud, conn, initial_state=init,
              instrument=False)
    assert np.array_equal(a.residue_history, b.residue_history)
    assert np.array_equal(a.primitives.as_array(), b.primitives.as_array())


def test_c3_partitioned_solve_bitwise(gpu, c3):
    """Two partitions of the 2.5M cloud (1.25M owned points each: the
    HBM-streaming kernel variants, on partitioned contexts) reproduce the
    single-domain history and state bit for bit."""
    from paper_2108_07031_b200.dist import solve_group

    cloud, conn, cfg, init, _ = c3
    two = SolverConfig(mach=0.85, aoa_deg=1.0, n_outer=2)
    ref = solve(two, cloud, conn, initial_state=init, instrument=False)
    hist, prims, U, _ = solve_group(two, cloud, conn, 2, initial_state=init)
    assert np.array_equal(hist, ref.residue_history)
    assert np.array_equal(prims, ref.primitives.as_array())



_GOLDEN = __import__("pathlib").Path(__file__).parent / "golden"


def _needs(name):
    return pytest.mark.skipif(not (_GOLDEN / f"{name}.json").exists(),
                              reason=f"tests/golden/{name} not generated (tools/make_golden.py {name})")


@_needs("c2p5m")
def test_c3_two_iterations_match_reference(gpu, c3):
    """Config 3 against the reference package itself (tests/golden/c2p5m,
    written by the reference's own builder and solver): residue history of
    the first two iterations <= 1e-10 relative, 4096-point state sample."""
    from conftest import golden

    A, meta = golden("c2p5m")
    cloud, conn, cfg, init, _ = c3
    assert meta["params"][:3] == [3160, 790, 1.00734] and (meta["mach"], meta["aoa"]) == (0.85, 1.0)
    res = solve(SolverConfig(mach=0.85, aoa_deg=1.0, n_outer=meta["iters"]), cloud, conn, initial_state=init,
                instrument=False)
    rel = np.abs(res.residue_history - A["history"]) / A["history"]
    assert rel.max() <= 1e-10, rel
    idx = A["sample_idx"]
    assert np.allclose(res.primitives.as_array()[:, idx], A["prims_sample"], rtol=1e-10, atol=1e-12)

# --------------------------------------------------------------- 40M (opt-in)
# The bench's default configuration (BASELINE configs[4]): one whole outer
# iteration of the device path against the oracle on all 39,992,976 points,
# plus fused == split4 bitwise.  ~4 min and ~70 GB of host memory, so it runs
# only with KMF_FULL_SIZE_TESTS=1 (results: profiles/r1_full_size_parity.txt).

full_size = pytest.mark.skipif(not __import__("os").environ.get("KMF_FULL_SIZE_TESTS"),
                               reason="set KMF_FULL_SIZE_TESTS=1 (40M points, ~4 min, ~70 GB host memory)")


@pytest.fixture(scope="module")
def c5():
    cloud = generate_naca_cloud(12648, 3162, 1.001821, 20.0)
    conn = build_stencils(cloud)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=1)
    return cloud, conn, cfg, initial_primitives(cfg, cloud)


@full_size
def test_c5_one_iteration_matches_oracle(gpu, c5):
    import os
    import time

    cloud, conn, cfg, init = c5
    t = time.perf_counter()
    res = solve(cfg, cloud, conn, initial_state=init, instrument=False)
    t_gpu = time.perf_counter() - t
    O.set_threads(os.cpu_count() or 1)
    pk = O.Packed(conn)
    fs = free_stream(cfg.mach, cfg.aoa_deg)
    t = time.perf_counter()
    hist, prims, _, _, _ = O.solve(pk, init.as_array(), [fs.rho[0], fs.u1[0], fs.u2[0], fs.p[0]], 1)
    t_cpu = time.perf_counter() - t
    rel = abs(res.residue_history[0] - hist[0]) / hist[0]
    err = np.abs(res.primitives.as_array() - prims) / (1e-12 + 1e-10 * np.abs(prims))
    print(f"c5 one iteration: residue rel diff {rel:.3e}, max scaled state error {err.max():.3e}; "
          f"device solve {t_gpu:.1f} s (incl. context), oracle {t_cpu:.1f} s")
    assert rel <= 1e-10
    assert np.allclose(res.primitives.as_array(), prims, rtol=1e-10, atol=1e-12)


@full_size
def test_c5_fused_equals_split4_bitwise(gpu, c5):
    cloud, conn, cfg, init = c5
    a = solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=2, mode="fused"), cloud, conn, initial_state=init,
              instrument=False)
    b = solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=2, mode="split4"), cloud, conn, initial_state=init,
              instrument=False)
    assert np.array_equal(a.residue_history, b.residue_history)
    assert np.array_equal(a.primitives.as_array(), b.primitives.as_array())


@full_size
def test_c2_thousand_iterations_match_oracle(gpu):
    """BASELINE configs[1] (160K points, M 0.63, AoA 2) for the paper's 1000
    iterations: residue history within 1e-10 relative per iteration and
    final primitives within rtol 1e-10 / atol 1e-12 of the oracle."""
    import os

    cloud = generate_naca_cloud(800, 200, 1.03, 20.0)
    conn = build_stencils(cloud)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=1000)
    init = initial_primitives(cfg, cloud)
    res = solve(cfg, cloud, conn, initial_state=init, instrument=False)
    O.set_threads(os.cpu_count() or 1)
    fs = free_stream(cfg.mach, cfg.aoa_deg)
    hist, prims, _, its, _ = O.solve(O.Packed(conn), init.as_array(), [fs.rho[0], fs.u1[0], fs.u2[0], fs.p[0]], 1000)
    assert res.iterations == its == 1000
    rel = np.abs(res.residue_history - hist) / hist
    err = np.abs(res.primitives.as_array() - prims) / (1e-12 + 1e-10 * np.abs(prims))
    print(f"c2 1000 iterations: max residue rel diff {rel.max():.3e} (at iteration {int(rel.argmax()) + 1}), "
          f"max scaled state error {err.max():.3e}; residue {hist[0]:.6e} -> {hist[-1]:.6e}")
    assert rel.max() <= 1e-10
    assert np.allclose(res.primitives.as_array(), prims, rtol=1e-10, atol=1e-12)


# ------------------------------------------ against the reference itself
# Fixtures written by the reference package (tools/make_golden.py, run in the
# build container): BASELINE configs[0] and [1] on the native builder's
# connectivity (bit-exact with the reference builder, digests checked in
# tests/test_geometry_parity.py).


def test_c160k_twenty_iterations_match_reference(gpu):
    """Config 2 (160K points, M 0.63, AoA 2): the reference's own 20-iteration
    residue history (<= 1e-10 relative) and a 4096-point state sample."""
    from conftest import golden

    A, meta = golden("c160k")
    m, L, gr, ff = meta["params"]
    cloud = generate_naca_cloud(m, L, gr, ff)
    cfg = SolverConfig(mach=meta["mach"], aoa_deg=meta["aoa"], n_outer=meta["iters"])
    res = solve(cfg, cloud, build_stencils(cloud), instrument=False)
    rel = np.abs(res.residue_history - A["history"]) / A["history"]
    assert rel.max() <= 1e-10, rel.max()
    idx = A["sample_idx"]
    assert np.allclose(res.primitives.as_array()[:, idx], A["prims_sample"], rtol=1e-10, atol=1e-12)


@_needs("c40k")
def test_c40k_reference_breakdown_reproduced(gpu):
    """Config 1 (40K points, M 0.63, AoA 2, 1000 iterations) breaks down in
    the reference: a flux_residual positivity failure part-way through.  The
    device path reproduces the history up to it (<= 1e-10 relative), the
    state before it, and the failure itself: same iteration, same stage
    operator, same offending points."""
    from conftest import golden

    from paper_2108_07031_b200 import PositivityError

    A, meta = golden("c40k")
    fail = meta.get("failure")
    m, L, gr, ff = meta["params"]
    cloud = generate_naca_cloud(m, L, gr, ff)
    conn = build_stencils(cloud)
    before = SolverConfig(mach=meta["mach"], aoa_deg=meta["aoa"], n_outer=meta["iters"])
    res = solve(before, cloud, conn, instrument=False)
    rel = np.abs(res.residue_history - A["history"]) / A["history"]
    assert res.iterations == meta["iters"]
    assert rel.max() <= 1e-10, rel.max()
    assert np.allclose(res.primitives.as_array(), A["prims"], rtol=1e-10, atol=1e-12)
    if fail is None:
        return
    with pytest.raises(PositivityError) as exc:
        solve(SolverConfig(mach=meta["mach"], aoa_deg=meta["aoa"], n_outer=1000), cloud, conn, instrument=False)
    # message: "iteration N: flux_residual[kind]: ... on K edge(s)"; indices:
    # positions in that 4096-point block's family edge list (solver.py:162-168)
    assert str(exc.value) == fail["message"]
    assert [int(i) for i in exc.value.indices] == fail["indices"]


def test_c1_first_order_thousand_iterations_match_oracle(gpu):
    """BASELINE configs[0]: 40K points, M 0.63, AoA 2, first order, 1000
    iterations (the reference's solve() is second order only; the oracle's
    first-order loop is pinned to the reference's operators in
    tests/test_oracle_golden.py)."""
    import os

    cloud = generate_naca_cloud(400, 100, 1.06, 20.0)
    conn = build_stencils(cloud)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=1000, order=1)
    init = initial_primitives(cfg, cloud)
    res = solve(cfg, cloud, conn, initial_state=init, instrument=False)
    O.set_threads(os.cpu_count() or 1)
    fs = free_stream(cfg.mach, cfg.aoa_deg)
    hist, prims, _, its, _ = O.solve(O.Packed(conn), init.as_array(), [fs.rho[0], fs.u1[0], fs.u2[0], fs.p[0]], 1000,
                                     n_inner=0)
    assert res.iterations == its == 1000
    assert np.max(np.abs(res.residue_history - hist) / hist) <= 1e-10
    assert np.allclose(res.primitives.as_array(), prims, rtol=1e-10, atol=1e-12)
