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
