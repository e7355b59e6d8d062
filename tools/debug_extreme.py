"""Stage-by-stage GPU vs oracle on the amp=-0.64 bump state (debug aid)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

from conftest import fs_vec, perturbed_state  # noqa: E402
from oracle import oracle as O  # noqa: E402
import paper_2108_07031_b200 as K  # noqa: E402

c = K.generate_naca_cloud(80, 30, 1.15, 20.0)
conn = K.build_stencils(c)
pk = O.Packed(conn)
amp = float(sys.argv[1]) if len(sys.argv) > 1 else -0.64
init = perturbed_state(c, amp=amp).as_array()
fs = fs_vec(0.63, 2.0)
dt = O.local_timestep(pk, init, 1.0)
dtg = K.local_timestep(K.Primitives.from_array(init), conn, 1.0)
print("dt equal", np.array_equal(dt, dtg))
U0 = O.primitives_to_conserved(init)
prims, U = init, U0
for stage in (1, 2):
    q = O.primitives_to_q(prims)
    qg = K.primitives_to_q(K.Primitives.from_array(prims))
    print(stage, "q maxdiff", np.abs(q - qg).max())
    qx, qy, _ = O.q_derivatives(pk, q, 3)
    g = K.compute_q_derivatives(q, conn, 3)
    print(stage, "qgrad bitwise", np.array_equal(qx, g.qx), np.array_equal(qy, g.qy))
    R = O.flux_residual(pk, q, qx, qy)
    st = K.FlowState(prims=K.Primitives.from_array(prims), q=q, qx=qx, qy=qy)
    Rg = K.flux_residual(st, conn)
    d = np.abs(R - Rg)
    print(stage, "R_int maxdiff per row", d.max(axis=1), "scale", np.abs(R).max(axis=1), "argmax", d.argmax(axis=1))
    Rb = O.apply_boundary(pk, q, qx, qy, fs, R)
    Rbg = K.apply_boundary(st, R.copy(), conn, K.free_stream(0.63, 2.0))
    print(stage, "R_bnd maxdiff", np.abs(Rb - Rbg).max())
    U = O.state_update_rk(U0, U, stage, dt, Rb)
    prims = O.conserved_to_primitives(U) if U[0].min() > 0 else None
    if prims is None:
        print("oracle density fails at stage", stage)
        break
cfg = K.SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=1, cfl=1.0)
for n_outer in (1,):
    try:
        r = K.solve(cfg, c, conn, initial_state=K.Primitives.from_array(init), instrument=False)
        print("solve 1 iteration ok", r.residue_history)
    except K.PositivityError as e:
        print("solve error", e, e.indices[:10])
