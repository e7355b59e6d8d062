"""The drop-in boundary accepts the reference's OWN objects.

The reference ``kmf.state.Primitives`` (state.py:46-88) has no ``as_array``
and ``kmf.solver.SolverConfig`` (solver.py:69-112) has no ``order``; the
INTEGRATION.md shim forwards both straight into this package.  The stand-in
classes below mirror those two reference types field for field (no extra
methods), so the CPU tests run everywhere; ``test_real_reference_objects``
imports the live reference when /root/reference is present (build
container only) and packs a reference-built Connectivity.  The GPU test
runs ``solve`` on the stand-ins and requires bitwise the same result as with
this package's own types.
"""

from __future__ import annotations

import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import pytest

from conftest import perturbed_state
from paper_2108_07031_b200 import SolverConfig, solve
from paper_2108_07031_b200._device import pack
from paper_2108_07031_b200.solver import MODES, _params, config_order
from paper_2108_07031_b200.state import prims_array

REF_SRC = Path("/root/reference/pkg/src")


def _f64(a):
    return np.atleast_1d(np.asarray(a, dtype=np.float64))


@dataclass
class RefPrimitives:
    """Field-for-field stand-in of reference state.py:46-88 (no as_array)."""

    rho: np.ndarray
    u1: np.ndarray
    u2: np.ndarray
    p: np.ndarray

    def __post_init__(self):
        self.rho, self.u1, self.u2, self.p = (_f64(v) for v in (self.rho, self.u1, self.u2, self.p))

    def copy(self):
        return RefPrimitives(self.rho.copy(), self.u1.copy(), self.u2.copy(), self.p.copy())

    def validate(self, context: str = "state") -> None:
        if (~((self.rho > 0.0) & (self.p > 0.0))).any():
            raise ValueError(context)


@dataclass
class RefSolverConfig:
    """Field-for-field stand-in of reference solver.py:69-99 (no `order`)."""

    mach: float
    aoa_deg: float = 0.0
    gamma: float = 1.4
    cfl: float = 0.2
    n_outer: int = 1000
    n_inner: int = 3
    mode: str = "fused"
    threads: int = 1
    convergence_tol: float | None = None


def test_reference_config_has_no_order_and_maps_to_second_order():
    cfg = RefSolverConfig(mach=0.63, aoa_deg=2.0, n_inner=3, mode="split4")
    assert not hasattr(cfg, "order")
    assert config_order(cfg) == 2
    p = _params(cfg)
    assert p.n_inner == 3 and p.mode == MODES.index("split4") and p.gamma == 1.4 and p.cfl == 0.2
    # identical to this package's own config
    q = _params(SolverConfig(mach=0.63, aoa_deg=2.0, n_inner=3, mode="split4"))
    for f, _ in p._fields_:
        a, b = getattr(p, f), getattr(q, f)
        assert (list(a) == list(b)) if f == "fs" else (a == b), f


def test_reference_primitives_pack_to_the_abi_layout(small_naca):
    ours = perturbed_state(small_naca)
    ref = RefPrimitives(ours.rho, ours.u1, ours.u2, ours.p)
    assert not hasattr(ref, "as_array")
    a = prims_array(ref)
    assert a.flags.c_contiguous and a.dtype == np.float64 and a.shape == (4, small_naca.n_points)
    assert np.array_equal(a, ours.as_array())
    # scalars promote like the reference's _as_f64 (state.py:40-42)
    assert prims_array(RefPrimitives(1.0, 0.5, 0.0, 0.7)).shape == (4, 1)


@pytest.mark.skipif(not REF_SRC.is_dir(), reason="reference package not present (GPU box)")
def test_real_reference_objects(small_naca):
    """The live reference's SolverConfig / Primitives / Connectivity go
    through _params, prims_array and the device packing unchanged."""
    sys.path.insert(0, str(REF_SRC))
    try:
        import kmf  # noqa: F401
        from kmf.geometry import build_stencils as ref_build
        from kmf.geometry import generate_naca_cloud as ref_gen
        from kmf.solver import SolverConfig as RefCfg
        from kmf.solver import _initial_primitives as ref_init
    finally:
        sys.path.remove(str(REF_SRC))
    cfg = RefCfg(mach=0.63, aoa_deg=2.0)
    assert _params(cfg).n_inner == 3
    cloud = ref_gen(80, 30, 1.15, 20.0)
    conn = ref_build(cloud)
    init = ref_init(cfg, cloud)
    a = prims_array(init)
    assert a.shape == (4, cloud.n_points) and a.flags.c_contiguous
    g, keep = pack(conn)
    assert g.n == cloud.n_points and g.full.n_edges == conn.full.idx.shape[0]
    assert g.has_wall == 1 and g.has_outer == 1
    assert keep


@pytest.mark.gpu
def test_solve_with_reference_types_is_bitwise(gpu, small_naca, small_naca_conn):
    ours = perturbed_state(small_naca)
    ref = RefPrimitives(ours.rho, ours.u1, ours.u2, ours.p)
    a = solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=5), small_naca, small_naca_conn, initial_state=ours,
              instrument=False)
    b = solve(RefSolverConfig(mach=0.63, aoa_deg=2.0, n_outer=5), small_naca, small_naca_conn, initial_state=ref,
              instrument=False)
    assert np.array_equal(a.residue_history, b.residue_history)
    assert np.array_equal(a.primitives.as_array(), prims_array(b.primitives))
    assert np.array_equal(a.conserved, b.conserved)
