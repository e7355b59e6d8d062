"""Pin the CPU oracle (oracle/kmf_oracle.c) to the reference's own outputs.

The golden vectors come from running the reference package itself
(tools/make_golden.py).  Rational operators must match bitwise; operators
with log/exp/erf (glibc here vs numpy SIMD / scipy in the reference) within
the per-call flux tolerance of DESIGN.md.  CPU only.
"""

import numpy as np
import pytest

from conftest import fs_vec, golden
from oracle import oracle as O

PREFIXES = ("pert", "init")


def flux_tol(ref):
    # |dR| <= 1e-11 * max(max|R_row|, 1) per conserved row
    return 1e-11 * np.maximum(np.abs(ref).max(axis=1, keepdims=True), 1.0)


@pytest.mark.parametrize("pre", PREFIXES)
def test_timestep_bitwise(pre, small_golden, oracle_small):
    G, _ = small_golden
    assert np.array_equal(O.local_timestep(oracle_small, G[f"{pre}.prims"], 0.2), G[f"{pre}.dt"])


@pytest.mark.parametrize("pre", PREFIXES)
def test_q_variables(pre, small_golden):
    G, _ = small_golden
    q = O.primitives_to_q(G[f"{pre}.prims"])
    ref = G[f"{pre}.q"]
    assert np.all(np.abs(q - ref) <= 4 * np.spacing(np.abs(ref)))


@pytest.mark.parametrize("pre", PREFIXES)
def test_q_gradients_bitwise(pre, small_golden, oracle_small):
    G, _ = small_golden
    q = G[f"{pre}.q"]
    qx, qy = O.first_order(oracle_small, q)
    assert np.array_equal(qx, G[f"{pre}.qx0"]) and np.array_equal(qy, G[f"{pre}.qy0"])
    for n_inner in (1, 3):
        qx, qy, res = O.q_derivatives(oracle_small, q, n_inner)
        assert np.array_equal(qx, G[f"{pre}.qx{n_inner}"])
        assert np.array_equal(qy, G[f"{pre}.qy{n_inner}"])
        assert np.array_equal(res, G[f"{pre}.inner_res{n_inner}"])


@pytest.mark.parametrize("pre", PREFIXES)
@pytest.mark.parametrize("mode", ["fused", "split4"])
def test_flux_and_boundary(pre, mode, small_golden, oracle_small):
    G, _ = small_golden
    q, qx, qy = G[f"{pre}.q"], G[f"{pre}.qx3"], G[f"{pre}.qy3"]
    R = O.flux_residual(oracle_small, q, qx, qy, mode)
    assert np.all(np.abs(R - G[f"{pre}.R_int"]) <= flux_tol(G[f"{pre}.R_int"]))
    Rb = O.apply_boundary(oracle_small, q, qx, qy, fs_vec(0.63, 2.0), G[f"{pre}.R_int"])
    assert np.all(np.abs(Rb - G[f"{pre}.R"]) <= flux_tol(G[f"{pre}.R"]))


@pytest.mark.parametrize("pre", PREFIXES)
def test_update_decode_residue_bitwise(pre, small_golden):
    G, _ = small_golden
    U = G[f"{pre}.U"]
    assert np.array_equal(O.primitives_to_conserved(G[f"{pre}.prims"]), U)
    assert np.array_equal(O.state_update_rk(U, U, 1, G[f"{pre}.dt"], G[f"{pre}.R"]), G[f"{pre}.U1"])
    assert np.array_equal(O.state_update_rk(U, G[f"{pre}.U1"], 3, G[f"{pre}.dt"], G[f"{pre}.R"]), G[f"{pre}.U3"])
    assert np.array_equal(O.conserved_to_primitives(G[f"{pre}.U1"]), G[f"{pre}.prims1"])
    assert O.residue_norm(G[f"{pre}.U1"], U) == G[f"{pre}.residue1"][0]


def test_fsum_exact():
    import math

    rng = np.random.default_rng(0)
    for scale in (1e-300, 1e-20, 1.0, 1e200):
        v = rng.uniform(0, 1, 5000) ** 7 * scale
        assert O.fsum(v) == math.fsum(v.tolist())


def test_split_flux_against_reference():
    K, _ = golden("kinetics")
    pr = K["prims"]
    for axis in ("x", "y"):
        assert np.array_equal(O.full_flux(pr, axis), K[f"full_{axis}"])
        for sign in ("+", "-"):
            g = O.split_flux(pr, axis, sign)
            ref = K[f"split_{axis}{sign}"]
            assert np.all(np.abs(g - ref) <= 1e-14 * np.maximum(np.abs(ref), 1.0))


def test_state_transforms_against_reference():
    K, _ = golden("kinetics")
    pr = K["prims"]
    for g in (1.4, 5.0 / 3.0):
        tag = f"g{g:.4f}"
        assert np.array_equal(O.primitives_to_conserved(pr, g), K[f"U.{tag}"])
        assert np.array_equal(O.conserved_to_primitives(K[f"U.{tag}"], g), K[f"U2p.{tag}"])
        q = O.primitives_to_q(pr, g)
        assert np.all(np.abs(q - K[f"q.{tag}"]) <= 4 * np.spacing(np.abs(K[f"q.{tag}"])))
        back = O.q_to_primitives(K[f"q.{tag}"], g)
        assert np.allclose(back, K[f"q2p.{tag}"], rtol=1e-14, atol=0)


@pytest.mark.parametrize("mode", ["fused", "split4"])
def test_short_solve_history(mode, small_golden, oracle_small):
    G, _ = small_golden
    hist, prims, U, its, conv = O.solve(oracle_small, G["pert.prims"], fs_vec(0.63, 2.0), 5, mode=mode)
    ref = G[f"solve_pert5.{mode}.history"]
    assert its == 5
    assert np.all(np.abs(hist - ref) <= 1e-10 * ref)
    assert np.allclose(prims, G[f"solve_pert5.{mode}.prims"], rtol=1e-10, atol=1e-12)


def test_free_stream_fixed_point(small_golden, oracle_small, small_naca):
    G, _ = small_golden
    fs = fs_vec(0.63, 2.0)
    init = np.repeat(fs[:, None], small_naca.n_points, axis=1)
    hist, *_ = O.solve(oracle_small, init, fs, 5)
    assert np.max(hist) <= 1e-12
    assert np.max(G["solve_fs5.history"]) <= 1e-12


def test_long_history_2k(oracle_small):
    """First 120 iterations of the reference's 1000-iteration M0.63 run."""
    H, _ = golden("hist2k")
    S, _ = golden("small")
    O.set_threads(8)
    n = 120
    hist, *_ = O.solve(oracle_small, S["init.m63a2"], fs_vec(0.63, 2.0), n)
    ref = H["m63a2.history"][:n]
    assert np.all(np.abs(hist - ref) <= 1e-10 * ref)


def test_config2_history_against_reference():
    """BASELINE config 2 (160K points, M 0.63, AoA 2): the reference's own
    20-iteration residue history and a 4096-point sample of the final state
    (tests/golden/c160k, tools/make_golden.py) on the native builder's
    connectivity (its digests are checked in test_geometry_parity.py)."""
    from paper_2108_07031_b200 import SolverConfig, build_stencils, generate_naca_cloud, initial_primitives

    A, meta = golden("c160k")
    m, L, g, ff = meta["params"]
    cloud = generate_naca_cloud(m, L, g, ff)
    init = initial_primitives(SolverConfig(mach=meta["mach"], aoa_deg=meta["aoa"]), cloud)
    O.set_threads(8)
    hist, prims, *_ = O.solve(O.Packed(build_stencils(cloud)), init.as_array(), fs_vec(meta["mach"], meta["aoa"]),
                              meta["iters"])
    assert np.all(np.abs(hist - A["history"]) <= 1e-10 * A["history"])
    idx = A["sample_idx"]
    assert np.allclose(prims[:, idx], A["prims_sample"], rtol=1e-10, atol=1e-12)


def test_config1_history_against_reference():
    """BASELINE config 1 (40K points, M 0.63, AoA 2): the first 60 iterations
    of the reference's own run (tests/golden/c40k; the reference breaks down
    at iteration 407, which the device test reproduces in full)."""
    from paper_2108_07031_b200 import SolverConfig, build_stencils, generate_naca_cloud, initial_primitives

    A, meta = golden("c40k")
    m, L, g, ff = meta["params"]
    cloud = generate_naca_cloud(m, L, g, ff)
    init = initial_primitives(SolverConfig(mach=meta["mach"], aoa_deg=meta["aoa"]), cloud)
    O.set_threads(8)
    n = 60
    hist, *_ = O.solve(O.Packed(build_stencils(cloud)), init.as_array(), fs_vec(meta["mach"], meta["aoa"]), n)
    assert np.all(np.abs(hist - A["history"][:n]) <= 1e-10 * A["history"][:n])


def test_first_order_scheme_against_reference_operators(small_naca_conn):
    """The first-order scheme (qx = qy = 0; BASELINE config 1) of the oracle
    (n_inner = 0) against the same loop composed of the reference's own
    stage operators (tests/golden/order1, tools/make_golden.py order1)."""
    from paper_2108_07031_b200 import SolverConfig, generate_naca_cloud, initial_primitives

    A, _ = golden("order1")
    cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
    pk = O.Packed(small_naca_conn)
    O.set_threads(8)
    for tag, (mach, aoa, iters) in {"m63a2": (0.63, 2.0, 200), "m85a1": (0.85, 1.0, 100)}.items():
        init = initial_primitives(SolverConfig(mach=mach, aoa_deg=aoa), cloud)
        hist, prims, *_ = O.solve(pk, init.as_array(), fs_vec(mach, aoa), iters, n_inner=0)
        ref = A[f"{tag}.history"]
        assert np.all(np.abs(hist - ref) <= 1e-10 * ref)
        assert np.allclose(prims, A[f"{tag}.prims"], rtol=1e-10, atol=1e-12)


GAMMAS = (5.0 / 3.0, 1.3)


@pytest.mark.parametrize("gamma", GAMMAS)
def test_gamma_split_flux_and_q(gamma):
    """Split fluxes and entropy variables at gamma = 5/3 and 1.3 (the
    decode's 5/3 and generic evaluation paths) against the reference."""
    K, _ = golden("kinetics")
    A, _ = golden("gammas")
    tag = f"g{gamma:.4f}"
    q = O.primitives_to_q(K["prims"], gamma)
    assert np.all(np.abs(q - A[f"{tag}.q"]) <= 4 * np.spacing(np.abs(A[f"{tag}.q"])))
    for axis in ("x", "y"):
        for sign in ("+", "-"):
            ref = A[f"{tag}.split_{axis}{sign}"]
            got = O.split_flux(K["prims"], axis, sign, gamma)
            assert np.all(np.abs(got - ref) <= 1e-13 * np.maximum(np.abs(ref), 1.0))


@pytest.mark.parametrize("gamma", GAMMAS)
def test_gamma_residual_and_history(gamma, small_naca, oracle_small):
    A, _ = golden("gammas")
    tag = f"g{gamma:.4f}"
    q = O.primitives_to_q(A[f"{tag}.prims"], gamma)
    qx, qy, _ = O.q_derivatives(oracle_small, q, 3)
    R = O.flux_residual(oracle_small, q, qx, qy, "fused", gamma)
    assert np.all(np.abs(R - A[f"{tag}.R_int"]) <= flux_tol(A[f"{tag}.R_int"]))
    Rb = O.apply_boundary(oracle_small, q, qx, qy, fs_vec(0.63, 2.0, gamma), R, gamma)
    assert np.all(np.abs(Rb - A[f"{tag}.R"]) <= flux_tol(A[f"{tag}.R"]))
    from paper_2108_07031_b200 import SolverConfig, initial_primitives

    init = initial_primitives(SolverConfig(mach=0.63, aoa_deg=2.0, gamma=gamma), small_naca)
    hist, prims, *_ = O.solve(oracle_small, init.as_array(), fs_vec(0.63, 2.0, gamma), 20, gamma=gamma)
    assert np.max(np.abs(hist - A[f"{tag}.history"]) / A[f"{tag}.history"]) <= 1e-10
    assert np.allclose(prims, A[f"{tag}.final"], rtol=1e-10, atol=1e-12)
