"""CUDA path vs the oracle and the reference's golden vectors (B200 only).

Bitwise: timestep, q-gradients (first order + Jacobi sweeps), state update,
decode, residue, fused == split4.  Tolerance: q variables
<= 4 ulp; flux_residual + boundary |dR| <= 1e-11 * max(max|R_row|, 1) per
conserved row; residue history <= 1e-10 relative per iteration; final
primitives rtol 1e-10 / atol 1e-12.
"""

import numpy as np
import pytest

from conftest import channel_cloud, fs_vec, golden, perturbed_state
from oracle import oracle as O
from paper_2108_07031_b200 import (
    FlowState,
    PositivityError,
    Primitives,
    SolverConfig,
    apply_boundary,
    build_stencils,
    compute_q_derivatives,
    conserved_to_primitives,
    first_order_q_gradients,
    flux_residual,
    free_stream,
    local_timestep,
    primitives_to_conserved,
    primitives_to_q,
    residue_norm,
    solve,
    state_update_rk,
)

pytestmark = pytest.mark.gpu
PREFIXES = ("pert", "init")


def flux_tol(ref):
    return 1e-11 * np.maximum(np.abs(ref).max(axis=1, keepdims=True), 1.0)


def flow(G, pre):
    return FlowState(prims=Primitives.from_array(G[f"{pre}.prims"]), q=G[f"{pre}.q"], qx=G[f"{pre}.qx3"],
                     qy=G[f"{pre}.qy3"])


@pytest.mark.parametrize("pre", PREFIXES)
def test_timestep_bitwise(gpu, pre, small_golden, small_naca_conn):
    G, _ = small_golden
    dt = local_timestep(Primitives.from_array(G[f"{pre}.prims"]), small_naca_conn, 0.2)
    assert np.array_equal(dt, G[f"{pre}.dt"])


@pytest.mark.parametrize("pre", PREFIXES)
def test_q_variables_within_4ulp(gpu, pre, small_golden):
    G, _ = small_golden
    q = primitives_to_q(Primitives.from_array(G[f"{pre}.prims"]))
    ref = G[f"{pre}.q"]
    assert np.all(np.abs(q - ref) <= 4 * np.spacing(np.abs(ref)))


@pytest.mark.parametrize("pre", PREFIXES)
def test_q_gradients_bitwise(gpu, pre, small_golden, small_naca_conn):
    G, _ = small_golden
    q = G[f"{pre}.q"]
    fo = first_order_q_gradients(q, small_naca_conn)
    assert np.array_equal(fo.qx, G[f"{pre}.qx0"]) and np.array_equal(fo.qy, G[f"{pre}.qy0"])
    for n_inner in (1, 3):
        g = compute_q_derivatives(q, small_naca_conn, n_inner)
        assert np.array_equal(g.qx, G[f"{pre}.qx{n_inner}"])
        assert np.array_equal(g.qy, G[f"{pre}.qy{n_inner}"])
        assert np.array_equal(np.asarray(g.inner_residuals), G[f"{pre}.inner_res{n_inner}"])


def test_q_gradients_bitwise_random_state(gpu, small_naca_conn, oracle_small):
    rng = np.random.default_rng(3)
    q = rng.normal(size=(4, small_naca_conn.cloud.n_points))
    g = compute_q_derivatives(q, small_naca_conn, 5)
    qx, qy, res = O.q_derivatives(oracle_small, q, 5)
    assert np.array_equal(g.qx, qx) and np.array_equal(g.qy, qy)
    assert np.array_equal(np.asarray(g.inner_residuals), res)


@pytest.mark.parametrize("pre", PREFIXES)
@pytest.mark.parametrize("mode", ["fused", "split4"])
def test_flux_residual_tolerance(gpu, pre, mode, small_golden, small_naca_conn, oracle_small):
    G, _ = small_golden
    R = flux_residual(flow(G, pre), small_naca_conn, mode)
    ref = G[f"{pre}.R_int"]
    assert np.all(np.abs(R - ref) <= flux_tol(ref))
    orc = O.flux_residual(oracle_small, G[f"{pre}.q"], G[f"{pre}.qx3"], G[f"{pre}.qy3"])
    assert np.all(np.abs(R - orc) <= flux_tol(orc))
    assert np.all(R[:, small_naca_conn.cloud.flag != 0] == 0.0)


@pytest.mark.parametrize("pre", PREFIXES)
def test_fused_equals_split4_bitwise(gpu, pre, small_golden, small_naca_conn):
    G, _ = small_golden
    a = flux_residual(flow(G, pre), small_naca_conn, "fused")
    b = flux_residual(flow(G, pre), small_naca_conn, "split4")
    assert np.array_equal(a, b)


def _stored_offset_twin(conn):
    """The same Connectivity with one interior point's coordinates nudged by
    an ulp after the stencils were built: full.dx/dy no longer equal
    x[j] - x[i] bitwise there, so the device stores the ELL offsets and runs
    its stored-offset kernels (k_first_order / k_sweep / k_flux <XY = false>)
    on exactly the reference's offsets."""
    import copy

    twin = copy.copy(conn)
    cl = copy.copy(conn.cloud)
    cl.x = conn.cloud.x.copy()
    i = int(np.flatnonzero(cl.flag == 0)[len(cl.x) // 3])
    cl.x[i] = np.nextafter(cl.x[i], np.inf)
    twin.cloud = cl
    return twin


def test_stored_offset_kernels_bitwise(gpu, small_golden, small_naca, small_naca_conn):
    """Stored-offset kernel path == coordinate path, bit for bit: q-gradients,
    fused and split4 flux, and a 3-iteration solve."""
    twin = _stored_offset_twin(small_naca_conn)
    G, _ = small_golden
    for pre in PREFIXES:
        q = G[f"{pre}.q"]
        a, b = compute_q_derivatives(q, small_naca_conn, 3), compute_q_derivatives(q, twin, 3)
        assert np.array_equal(a.qx, b.qx) and np.array_equal(a.qy, b.qy)
        for mode in ("fused", "split4"):
            assert np.array_equal(flux_residual(flow(G, pre), small_naca_conn, mode),
                                  flux_residual(flow(G, pre), twin, mode))
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=3)
    init = Primitives.from_array(G["pert.prims"])
    ra = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
    rb = solve(cfg, twin.cloud, twin, initial_state=init, instrument=False)
    assert np.array_equal(ra.residue_history, rb.residue_history)
    assert np.array_equal(ra.conserved, rb.conserved)


@pytest.mark.parametrize("pre", PREFIXES)
def test_boundary_closure_tolerance(gpu, pre, small_golden, small_naca_conn):
    G, _ = small_golden
    R = G[f"{pre}.R_int"].copy()
    out = apply_boundary(flow(G, pre), R, small_naca_conn, free_stream(0.63, 2.0))
    assert out is R
    ref = G[f"{pre}.R"]
    assert np.all(np.abs(R - ref) <= flux_tol(ref))


@pytest.mark.parametrize("pre", PREFIXES)
def test_update_decode_residue_bitwise(gpu, pre, small_golden):
    G, _ = small_golden
    U = G[f"{pre}.U"]
    assert np.array_equal(primitives_to_conserved(Primitives.from_array(G[f"{pre}.prims"])), U)
    U1 = state_update_rk(U, U, 1, G[f"{pre}.dt"], G[f"{pre}.R"])
    assert np.array_equal(U1, G[f"{pre}.U1"])
    U3 = state_update_rk(U, G[f"{pre}.U1"], 3, G[f"{pre}.dt"], G[f"{pre}.R"])
    assert np.array_equal(U3, G[f"{pre}.U3"])
    p1 = conserved_to_primitives(G[f"{pre}.U1"])
    assert np.array_equal(p1.as_array(), G[f"{pre}.prims1"])
    assert residue_norm(G[f"{pre}.U1"], U) == G[f"{pre}.residue1"][0]


def test_stage_arithmetic_matches_coefficients(gpu):
    """Reference tests/test_solver.py:124-133 on the device operator."""
    U0, dt, R = np.array([[1.0]]), np.array([0.1]), np.array([[2.0]])
    assert state_update_rk(U0, np.array([[0.7]]), 1, dt, R)[0, 0] == pytest.approx(0.6)
    assert state_update_rk(U0, np.array([[0.7]]), 4, dt, R)[0, 0] == pytest.approx(0.6)
    expected = 2.0 / 3.0 + 0.7 / 3.0 - 0.1 / 6.0 * 2.0
    assert state_update_rk(U0, np.array([[0.7]]), 3, dt, R)[0, 0] == pytest.approx(expected)
    with pytest.raises(ValueError, match="stage"):
        state_update_rk(U0, U0, 5, dt, R)


def test_integrator_is_third_order_on_linear_decay(gpu):
    """Reference tests/test_solver.py:136-151: y' = -y through the device
    stage operator (residual R = U), convergence order >= 2.9."""
    import math

    def decay(dt):
        U, d = np.array([[1.0], [0.0], [0.0], [0.0]]), np.array([dt])
        for _ in range(round(1.0 / dt)):
            Uo = U
            for stage in (1, 2, 3, 4):
                U = state_update_rk(Uo, U, stage, d, U)
        return float(U[0, 0])

    errs = [abs(decay(dt) - math.exp(-1.0)) for dt in (0.1, 0.05, 0.025)]
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert min(orders) >= 2.9, (errs, orders)


def test_residue_norm_values(gpu):
    """Reference tests/test_solver.py:197-209 on the device reduction."""
    old, new = np.zeros((4, 2)), np.zeros((4, 2))
    new[0] = [3.0, 4.0]
    assert residue_norm(new, old) == pytest.approx(np.sqrt(12.5), rel=1e-15)
    assert residue_norm(np.full((4, 1), 3.0), np.zeros((4, 1))) == 3.0
    new3 = np.zeros((4, 3))
    new3[1:] = 7.0
    assert residue_norm(new3, np.zeros((4, 3))) == 0.0


def test_inner_sweep_updates_shrink(gpu, small_naca, small_naca_conn):
    """Reference tests/test_lsq.py:107-117: on a smooth field each Jacobi
    sweep moves the iterate less than the one before; the device's
    inner residuals equal the oracle's bitwise."""
    x, y = small_naca.x, small_naca.y
    q = np.stack([np.sin(0.6 * x + 0.3 * y), np.cos(0.5 * x) * y, x * y, -np.exp(0.1 * x)])
    g = compute_q_derivatives(q, small_naca_conn, 6)
    r = g.inner_residuals
    assert len(r) == 6 and all(r[k + 1] < r[k] for k in range(5))
    qx, qy, ro = O.q_derivatives(O.Packed(small_naca_conn), q, 6)
    assert np.array_equal(g.qx, qx) and np.array_equal(g.qy, qy) and np.array_equal(np.asarray(r), ro)


def test_first_order_scheme_matches_reference(gpu, small_naca, small_naca_conn):
    """SolverConfig(order=1): the first-order scheme (qx = qy = 0, BASELINE
    config 1) against a loop of the reference's own stage operators
    (tests/golden/order1): history <= 1e-10 relative, state rtol 1e-10;
    fused == split4 bitwise."""
    A, _ = golden("order1")
    for tag, (mach, aoa, iters) in {"m63a2": (0.63, 2.0, 200), "m85a1": (0.85, 1.0, 100)}.items():
        res = solve(SolverConfig(mach=mach, aoa_deg=aoa, n_outer=iters, order=1), small_naca, small_naca_conn,
                    instrument=False)
        ref = A[f"{tag}.history"]
        assert np.max(np.abs(res.residue_history - ref) / ref) <= 1e-10
        assert np.allclose(res.primitives.as_array(), A[f"{tag}.prims"], rtol=1e-10, atol=1e-12)
    a = solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=20, order=1, mode="split4"), small_naca, small_naca_conn,
              instrument=False)
    b = solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=20, order=1), small_naca, small_naca_conn,
              instrument=False)
    assert np.array_equal(a.residue_history, b.residue_history)
    with pytest.raises(ValueError, match="order"):
        SolverConfig(mach=0.63, order=3)


def test_uniform_flow_residual_vanishes(gpu, small_naca, small_naca_conn):
    """Reference tests/test_solver.py:139-142."""
    prims = free_stream(0.63, 2.0, n=small_naca.n_points)
    q = primitives_to_q(prims)
    g = compute_q_derivatives(q, small_naca_conn, 3)
    st = FlowState(prims=prims, q=q, qx=g.qx, qy=g.qy)
    R = apply_boundary(st, flux_residual(st, small_naca_conn), small_naca_conn, free_stream(0.63, 2.0))
    assert np.max(np.abs(R)) <= 1e-12


def test_tangent_wall_flow_has_no_wall_residual(gpu):
    """Reference tests/test_solver.py:145-152 (channel with a flat wall)."""
    cloud = channel_cloud()
    conn = build_stencils(cloud, k=8)
    n = cloud.n_points
    prims = Primitives(np.ones(n), np.full(n, 0.5), np.zeros(n), np.full(n, 1.0 / 1.4))
    q = primitives_to_q(prims)
    g = compute_q_derivatives(q, conn, 3)
    st = FlowState(prims=prims, q=q, qx=g.qx, qy=g.qy)
    R = apply_boundary(st, flux_residual(st, conn), conn, free_stream(0.5, 0.0))
    assert np.max(np.abs(R[:, cloud.wall])) <= 1e-12
    L, _ = golden("lattice")
    ref = L["chan_k8.R_tangent"]
    assert np.all(np.abs(R - ref) <= flux_tol(ref))


# ----------------------------------------------------------------- solve


@pytest.mark.parametrize("mode", ["fused", "split4"])
def test_solve_short_history(gpu, mode, small_golden, small_naca, small_naca_conn):
    G, _ = small_golden
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, cfl=0.2, n_outer=5, mode=mode)
    res = solve(cfg, small_naca, small_naca_conn, initial_state=perturbed_state(small_naca), instrument=False)
    ref = G[f"solve_pert5.{mode}.history"]
    assert res.iterations == 5 and not res.converged
    assert np.all(np.abs(res.residue_history - ref) <= 1e-10 * ref)
    assert np.allclose(res.primitives.as_array(), G[f"solve_pert5.{mode}.prims"], rtol=1e-10, atol=1e-12)
    assert np.allclose(res.conserved, G[f"solve_pert5.{mode}.U"], rtol=1e-10, atol=1e-12)


def test_modes_and_repeats_bit_identical(gpu, small_naca, small_naca_conn):
    init = perturbed_state(small_naca)
    out = []
    for mode in ("fused", "split4", "fused"):
        cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=6, mode=mode, threads=8)
        r = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
        out.append((r.residue_history, r.conserved))
    for h, U in out[1:]:
        assert np.array_equal(h, out[0][0]) and np.array_equal(U, out[0][1])


def test_history_matches_reference_1000(gpu, small_naca, small_naca_conn):
    """Full 1000-iteration M0.63/AoA2 run on the 2.4k cloud vs the reference."""
    H, _ = golden("hist2k")
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, cfl=0.2, n_outer=1000)
    res = solve(cfg, small_naca, small_naca_conn, instrument=False)
    ref = H["m63a2.history"]
    rel = np.abs(res.residue_history - ref) / ref
    assert rel.max() <= 1e-10, rel.max()
    assert np.allclose(res.primitives.as_array(), H["m63a2.prims"], rtol=1e-10, atol=1e-12)


def test_transonic_history_matches_reference(gpu, small_naca, small_naca_conn):
    H, _ = golden("hist2k")
    cfg = SolverConfig(mach=0.85, aoa_deg=1.0, cfl=0.2, n_outer=300)
    res = solve(cfg, small_naca, small_naca_conn, instrument=False)
    ref = H["m85a1.history"]
    assert np.max(np.abs(res.residue_history - ref) / ref) <= 1e-10
    assert np.allclose(res.primitives.as_array(), H["m85a1.prims"], rtol=1e-10, atol=1e-12)


def test_free_stream_fixed_point_and_early_stop(gpu, small_naca, small_naca_conn):
    init = free_stream(0.63, 2.0, n=small_naca.n_points)
    res = solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=5), small_naca, small_naca_conn,
                initial_state=init, instrument=False)
    assert np.max(res.residue_history) <= 1e-12
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=50, convergence_tol=1e-6)
    res = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
    assert res.converged and res.iterations == 1 and res.residue_history.shape == (1,)


def test_aoa_zero_mirror_symmetry(gpu, small_golden, small_naca, small_naca_conn):
    """Reference tests/test_solver.py:273-281."""
    G, _ = small_golden
    pr = solve(SolverConfig(mach=0.63, aoa_deg=0.0, n_outer=10), small_naca, small_naca_conn).primitives
    m = 80
    mirror = np.concatenate([r * m + (m - np.arange(m)) % m for r in range(30)])
    assert np.abs(pr.rho - pr.rho[mirror]).max() <= 1e-13
    assert np.abs(pr.u1 - pr.u1[mirror]).max() <= 1e-13
    assert np.abs(pr.u2 + pr.u2[mirror]).max() <= 1e-13
    assert np.abs(pr.p - pr.p[mirror]).max() <= 1e-13
    assert np.allclose(pr.as_array(), G["solve_a0_10.prims"], rtol=1e-10, atol=1e-12)


def test_instrumented_solve_reports_stages(gpu, small_naca, small_naca_conn):
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=8)
    res = solve(cfg, small_naca, small_naca_conn, instrument=True, timing_skip=3)
    plain = solve(cfg, small_naca, small_naca_conn, instrument=False)
    assert np.array_equal(res.residue_history, plain.residue_history)
    assert res.timed_iterations == 5 and res.iterations == 8
    assert res.wall_seconds > 0.0
    assert res.stage_seconds["flux_residual"] > 0.0 and res.stage_seconds["q_derivatives"] > 0.0


@pytest.mark.parametrize("amp,ctx", [(-0.64, "density"), (-0.66, "pressure"), (-0.7, "flux_residual[x+]")])
@pytest.mark.parametrize("mode", ["fused", "split4"])
def test_positivity_error_in_solve(gpu, amp, ctx, mode, small_naca, small_naca_conn, oracle_small):
    """A deep density/pressure dip fails at the same iteration, stage, raise
    site, count and first index as the oracle (reference semantics)."""
    init = perturbed_state(small_naca, amp=amp)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=40, cfl=1.0, mode=mode)
    with pytest.raises(PositivityError) as exc:
        solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
    with pytest.raises(O.OracleError) as oexc:
        O.solve(oracle_small, init.as_array(), fs_vec(0.63, 2.0), 40, cfl=1.0, mode=mode)
    msg, o = str(exc.value), oexc.value
    assert msg.startswith(f"iteration {o.iteration}: ")
    assert ctx in msg and ctx.split("[")[0] in o.context
    assert exc.value.indices.size == o.count and exc.value.indices[0] == o.first


def test_initial_state_validation(gpu, small_naca, small_naca_conn):
    init = free_stream(0.63, 2.0, n=small_naca.n_points)
    init.rho[7] = -1.0
    with pytest.raises(PositivityError, match="initial state"):
        solve(SolverConfig(mach=0.63, n_outer=2), small_naca, small_naca_conn, initial_state=init)
