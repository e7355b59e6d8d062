"""Streaming cases (kmf_run_cases / solve_cases): each case equals its own
solve bit for bit, whatever the mix of configurations, failures and buffer
reuse -- the uploads and downloads overlapped with the neighbouring cases'
iterations must not change a single value."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import perturbed_state
from paper_2108_07031_b200 import PositivityError, SolverConfig, free_stream, solve, solve_cases
from paper_2108_07031_b200 import _lib
from paper_2108_07031_b200._device import device_for
from paper_2108_07031_b200.solver import _params
from paper_2108_07031_b200.state import prims_array

pytestmark = pytest.mark.gpu


def _same(res, ref):
    assert np.array_equal(res.residue_history, ref.residue_history)
    assert np.array_equal(prims_array(res.primitives), prims_array(ref.primitives))
    assert np.array_equal(res.conserved, ref.conserved)
    assert res.converged == ref.converged and res.iterations == ref.iterations


def test_cases_equal_single_solves(gpu, small_naca, small_naca_conn):
    n = small_naca.n_points
    inits = [perturbed_state(small_naca, amp=a) for a in (0.02, -0.05, 0.1)] + [free_stream(0.5, 1.0, n=n)]
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=25)
    out = solve_cases(cfg, small_naca, small_naca_conn, inits)
    assert len(out) == 4
    for res, init in zip(out, inits):
        _same(res, solve(cfg, small_naca, small_naca_conn, init, instrument=False))


def test_cases_mixed_configs_and_failure(gpu, small_naca, small_naca_conn):
    """Per-case parameters (free stream, mode, first/second order, cfl) --
    graphs re-captured between cases -- and a case failing positivity in the
    middle: it comes back as the reference's PositivityError, the others
    are untouched."""
    cfgs = [
        SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=12),
        SolverConfig(mach=0.8, aoa_deg=1.25, n_outer=12, mode="split4"),
        SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=12, cfl=1.0),
        SolverConfig(mach=0.5, aoa_deg=0.0, n_outer=12, order=1),
        SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=12, convergence_tol=1e-3),
    ]
    inits = [perturbed_state(small_naca, mach=c.mach, aoa=c.aoa_deg) for c in cfgs]
    inits[2] = perturbed_state(small_naca, amp=-0.64)
    out = solve_cases(cfgs, small_naca, small_naca_conn, inits)
    with pytest.raises(PositivityError) as exc:
        solve(cfgs[2], small_naca, small_naca_conn, inits[2], instrument=False)
    assert isinstance(out[2], PositivityError)
    assert str(out[2]) == str(exc.value) and list(out[2].indices) == list(exc.value.indices)
    for k in (0, 1, 3, 4):
        _same(out[k], solve(cfgs[k], small_naca, small_naca_conn, inits[k], instrument=False))
    assert out[4].converged and out[4].iterations < 12


def test_run_cases_pinned_one_iteration(gpu, small_naca, small_naca_conn):
    """The bench's end-to-end pattern: pinned buffers, one iteration per
    case, outputs alternating between two host buffers, many cases."""
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=1)
    init = prims_array(perturbed_state(small_naca))
    dev = device_for(small_naca_conn)
    n = small_naca.n_points
    hin = _lib.pinned((4, n))
    hin[...] = init
    outs = [_lib.pinned((4, n)) for _ in range(2)]
    m = 9
    finals, hist, done, conv, status = dev.run_cases([_params(cfg)] * m, [hin] * m, 1,
                                                     outs=[outs[k % 2] for k in range(m)])
    # the context keeps the last case's state: a continuation matches
    h2, k2, _ = dev.run(_params(cfg), 1)
    ref = solve(cfg, small_naca, small_naca_conn, perturbed_state(small_naca), instrument=False)
    assert status == [0] * m and done == [1] * m
    assert np.all(hist[:, 0] == ref.residue_history[0])
    for o in outs:
        assert np.array_equal(o, prims_array(ref.primitives))
    ref2 = solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=2), small_naca, small_naca_conn,
                 perturbed_state(small_naca), instrument=False)
    assert k2 == 1 and h2[0] == ref2.residue_history[1]


def test_run_cases_validation(gpu, small_naca, small_naca_conn):
    dev = device_for(small_naca_conn)
    p = _params(SolverConfig(mach=0.63, n_outer=1))
    with pytest.raises(ValueError):
        dev.run_cases([p], [np.zeros((4, 3))], 1)
    bad = _params(SolverConfig(mach=0.63, n_outer=1))
    bad.cfl = -1.0
    with pytest.raises(ValueError, match="invalid parameters"):
        dev.run_cases([bad], [prims_array(free_stream(0.63, 2.0, n=small_naca.n_points))], 1)
