"""The flux path's gamma-specialised code (B200 only).

The decode evaluates beta^(-1/(gamma-1)) three ways (kmf_flux.cuh fdecode,
kmf_b200.cu gamma_kind): GK=1 for gamma = 7/5, GK=2 for 5/3 and GK=0
(log/exp) for any other gamma.  Every GK path of the interior flux, the
boundary closure and the whole solve is checked against the reference's own
outputs (tests/golden/gammas, tools/make_golden.py gammas) and the oracle;
the flux kernel's edge-state device functions (fdecode + fsflux_m, the lean
table exp and the erf tail for |s| >= 1) are probed directly against the
reference's q_to_primitives and split_flux.
"""

import numpy as np
import pytest

from conftest import fs_vec, golden
from oracle import oracle as O
from paper_2108_07031_b200 import (
    FlowState,
    Primitives,
    SolverConfig,
    apply_boundary,
    compute_q_derivatives,
    flux_residual,
    free_stream,
    initial_primitives,
    solve,
    split_flux,
)
from paper_2108_07031_b200 import _lib

pytestmark = pytest.mark.gpu
GAMMAS = (5.0 / 3.0, 1.3)
FAMILIES = ("x+", "x-", "y+", "y-")


def flux_tol(ref):
    return 1e-11 * np.maximum(np.abs(ref).max(axis=1, keepdims=True), 1.0)


def probe_edge_state(q, gamma):
    q = np.ascontiguousarray(q, dtype=np.float64)
    n = q.shape[1]
    prims, flux = np.empty((4, n)), np.empty((16, n))
    _lib.check(_lib.lib().kmf_probe_edge_state(n, _lib.dptr(q), gamma, _lib.dptr(prims), _lib.dptr(flux)), "probe")
    return prims, flux.reshape(4, 4, n)


def _kinetics_case(gamma):
    K, _ = golden("kinetics")
    if gamma == 1.4:
        return K["prims"], K["q.g1.4000"], {f: K[f"split_{f}"] for f in FAMILIES}
    A, _ = golden("gammas")
    tag = f"g{gamma:.4f}"
    return K["prims"], A[f"{tag}.q"], {f: A[f"{tag}.split_{f}"] for f in FAMILIES}


@pytest.mark.parametrize("gamma", (1.4,) + GAMMAS)
def test_edge_state_device_functions(gpu, gamma):
    """fdecode<GK> + fsflux_m<4> (the interior kernel's edge body) on the
    reference's entropy variables: the decoded primitives and the four split
    fluxes against the reference's primitives and split_flux, including the
    supersonic |s| >= 1 states (erf tail) of the kinetics fixture."""
    prims, q, split = _kinetics_case(gamma)
    s_max = np.max(np.abs(prims[1:3]) * np.sqrt(prims[0] / (2 * prims[3])))
    assert s_max > 6.5  # the tail branches up to erf = +-1 are exercised
    got_p, got_f = probe_edge_state(q, gamma)
    assert np.all(np.abs(got_p - prims) <= 1e-13 * np.abs(prims) + 1e-15)
    for k, f in enumerate(FAMILIES):
        ref = split[f]
        assert np.all(np.abs(got_f[k] - ref) <= 1e-12 * np.maximum(np.abs(ref), 1.0)), f


@pytest.mark.parametrize("gamma", (1.4,) + GAMMAS)
def test_split_flux_operator_uses_the_kernel_function(gpu, gamma):
    """split_flux runs fsflux_m (the lean moment algebra of the kernel)."""
    prims, _, split = _kinetics_case(gamma)
    pr = Primitives.from_array(prims)
    for f in FAMILIES:
        ref = split[f]
        got = split_flux(pr, f[0], f[1], gamma)
        assert np.all(np.abs(got - ref) <= 1e-13 * np.maximum(np.abs(ref), 1.0)), f


@pytest.mark.parametrize("gamma", GAMMAS)
@pytest.mark.parametrize("mode", ["fused", "split4"])
def test_gamma_flux_and_boundary(gpu, gamma, mode, small_naca_conn, oracle_small):
    A, _ = golden("gammas")
    tag = f"g{gamma:.4f}"
    q = O.primitives_to_q(A[f"{tag}.prims"], gamma)
    g = compute_q_derivatives(q, small_naca_conn, 3)
    flow = FlowState(prims=Primitives.from_array(A[f"{tag}.prims"]), q=q, qx=g.qx, qy=g.qy)
    R = flux_residual(flow, small_naca_conn, mode, gamma)
    assert np.all(np.abs(R - A[f"{tag}.R_int"]) <= flux_tol(A[f"{tag}.R_int"]))
    orc = O.flux_residual(oracle_small, q, g.qx, g.qy, mode, gamma)
    assert np.all(np.abs(R - orc) <= flux_tol(orc))
    if mode == "split4":
        assert np.array_equal(R, flux_residual(flow, small_naca_conn, "fused", gamma))
    Rb = apply_boundary(flow, R.copy(), small_naca_conn, free_stream(0.63, 2.0, gamma), gamma)
    assert np.all(np.abs(Rb - A[f"{tag}.R"]) <= flux_tol(A[f"{tag}.R"]))


@pytest.mark.parametrize("gamma", GAMMAS)
def test_gamma_solve_twenty_iterations(gpu, gamma, small_naca, small_naca_conn, oracle_small):
    A, _ = golden("gammas")
    tag = f"g{gamma:.4f}"
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, gamma=gamma, n_outer=20)
    res = solve(cfg, small_naca, small_naca_conn, instrument=False)
    rel = np.abs(res.residue_history - A[f"{tag}.history"]) / A[f"{tag}.history"]
    assert rel.max() <= 1e-10, rel
    assert np.allclose(res.primitives.as_array(), A[f"{tag}.final"], rtol=1e-10, atol=1e-12)
    init = initial_primitives(cfg, small_naca)
    hist, prims, *_ = O.solve(oracle_small, init.as_array(), fs_vec(0.63, 2.0, gamma), 20, gamma=gamma)
    assert np.max(np.abs(res.residue_history - hist) / hist) <= 1e-10
    split = solve(SolverConfig(mach=0.63, aoa_deg=2.0, gamma=gamma, n_outer=20, mode="split4"), small_naca,
                  small_naca_conn, instrument=False)
    assert np.array_equal(split.residue_history, res.residue_history)
