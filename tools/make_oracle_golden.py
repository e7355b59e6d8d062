"""Long-horizon fixtures from the CPU oracle (test infrastructure).

The reference package (numpy) needs ~2 min per iteration at 2.5M points,
so long horizons at the HBM-streaming sizes are pinned through the oracle
(oracle/kmf_oracle.c), itself pinned to the reference's own outputs by
tests/test_oracle_golden.py.  Writes tests/golden/<name>.{npz,json}:
residue history, a deterministic 4096-point sample of the final primitives
and their sha256 over the full state.

    python tools/make_oracle_golden.py c2o1000 c3o50
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2108_07031_b200 import (  # noqa: E402
    SolverConfig,
    build_stencils,
    free_stream,
    generate_naca_cloud,
    initial_primitives,
)

OUT = ROOT / "tests" / "golden"

CASES = {
    # name: ((m, L, g), mach, aoa, iterations)
    "c2o1000": ((800, 200, 1.03), 0.63, 2.0, 1000),        # BASELINE configs[1], the paper's 1000 iterations
    "c3o50": ((3160, 790, 1.00734), 0.85, 1.0, 50),        # BASELINE configs[2], transonic
}


def make(name):
    (m, L, g), mach, aoa, iters = CASES[name]
    O.set_threads(os.cpu_count() or 1)
    t0 = time.perf_counter()
    cloud = generate_naca_cloud(m, L, g, 20.0)
    conn = build_stencils(cloud)
    cfg = SolverConfig(mach=mach, aoa_deg=aoa, n_outer=iters)
    init = initial_primitives(cfg, cloud)
    fs = free_stream(mach, aoa)
    t1 = time.perf_counter()
    hist, prims, _, its, _ = O.solve(O.Packed(conn), init.as_array(), [fs.rho[0], fs.u1[0], fs.u2[0], fs.p[0]], iters)
    t2 = time.perf_counter()
    assert its == iters
    idx = np.linspace(0, cloud.n_points - 1, 4096).astype(np.int64)
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", history=hist, sample_idx=idx, prims_sample=prims[:, idx])
    meta = {"generated_by": f"tools/make_oracle_golden.py {name}", "oracle": "oracle/kmf_oracle.c",
            "params": [m, L, g, 20.0], "mach": mach, "aoa": aoa, "iters": iters, "n_points": int(cloud.n_points),
            "final_prims_sha256": hashlib.sha256(np.ascontiguousarray(prims).tobytes()).hexdigest(),
            "setup_seconds": t1 - t0, "oracle_seconds": t2 - t1, "threads": os.cpu_count()}
    (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(f"wrote {name}: n={cloud.n_points} iters={iters} oracle {t2 - t1:.0f} s", flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        make(name)
