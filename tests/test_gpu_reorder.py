"""The Hilbert device order is bitwise neutral (operators and the full loop)."""

import numpy as np
import pytest

from conftest import perturbed_state
from paper_2108_07031_b200 import SolverConfig, compute_q_derivatives, solve
from paper_2108_07031_b200 import _device

pytestmark = pytest.mark.gpu


@pytest.fixture
def hilbert():
    old = _device.point_order()
    _device.set_point_order("hilbert")
    yield
    _device.set_point_order(old)


def test_solve_bitwise_identical_in_hilbert_order(gpu, small_naca, small_naca_conn, hilbert):
    init = perturbed_state(small_naca)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=12)
    a = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
    _device.set_point_order("natural")
    b = solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
    assert np.array_equal(a.residue_history, b.residue_history)
    assert np.array_equal(a.conserved, b.conserved)
    assert np.array_equal(a.primitives.as_array(), b.primitives.as_array())


def test_q_derivatives_bitwise_in_hilbert_order(gpu, small_naca_conn, hilbert):
    rng = np.random.default_rng(4)
    q = rng.normal(size=(4, small_naca_conn.cloud.n_points))
    a = compute_q_derivatives(q, small_naca_conn, 3)
    _device.set_point_order("natural")
    b = compute_q_derivatives(q, small_naca_conn, 3)
    assert np.array_equal(a.qx, b.qx) and np.array_equal(a.qy, b.qy)
    assert a.inner_residuals == b.inner_residuals


def test_positivity_indices_in_caller_numbering(gpu, small_naca, small_naca_conn, hilbert):
    from paper_2108_07031_b200 import PositivityError

    init = perturbed_state(small_naca, amp=-0.64)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=5, cfl=1.0)
    with pytest.raises(PositivityError) as exc:
        solve(cfg, small_naca, small_naca_conn, initial_state=init, instrument=False)
    assert list(exc.value.indices) == [880]
