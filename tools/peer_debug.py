"""Peer transport debugging aid: a 2-rank linked group on one GPU, short
deadline, counters of every rank after the run."""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
os.environ.setdefault("KMF_PEER_TIMEOUT_S", "3")
import numpy as np  # noqa: E402

from conftest import perturbed_state  # noqa: E402
from paper_2108_07031_b200 import SolverConfig, _lib, build_stencils, generate_naca_cloud  # noqa: E402
from paper_2108_07031_b200.dist import RankPart  # noqa: E402
from paper_2108_07031_b200.solver import _params  # noqa: E402

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
conn = build_stencils(cloud)
init = perturbed_state(cloud)
if os.environ.get("SOLVE_FIRST"):
    from paper_2108_07031_b200 import solve

    solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=n_iter), cloud, conn, initial_state=init, instrument=False)
ranks = [RankPart(conn, r, nr, n_inner=3, scheme=os.environ.get("SCHEME", "bands")) for r in range(nr)]
for rp in ranks:
    rp.set_state(init.as_array())
    print("rank", rp.part.rank, "send", {k: v.size for k, v in rp.part.send.items()},
          "recv", {k: v.size for k, v in rp.part.recv.items()})
h = (C.c_void_p * nr)(*[rp.dev.handle.value for rp in ranks])
_lib.check(_lib.lib().kmf_peer_link(h, nr), "link")
runs = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [n_iter]
for n_iter in runs:
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=n_iter)
    hist = np.zeros(n_iter)
    done, conv = C.c_int(0), C.c_int(0)
    rc = _lib.lib().kmf_run_linked(h, nr, C.byref(_params(cfg)), n_iter, _lib.dptr(hist), C.byref(done),
                                   C.byref(conv))
    print("rc", rc, _lib.lib().kmf_strerror().decode(), "done", done.value, hist)
    for rp in ranks:
        out = (C.c_uint64 * (3 + 3 * nr))()
        _lib.lib().kmf_peer_counters(rp.dev.handle, out)
        v = list(out)
        print("rank", rp.part.rank, "pushes/bands/iters", v[:3], "data", v[3:3 + nr], "read", v[3 + nr:3 + 2 * nr],
              "limb", v[3 + 2 * nr:])
