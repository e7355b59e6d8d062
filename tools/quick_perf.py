"""Quick device timing of the solve loop (development aid, not the bench).

    python tools/quick_perf.py [m L g] [iters]
"""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_2108_07031_b200 import SolverConfig, build_stencils, generate_naca_cloud, initial_primitives  # noqa: E402
import os  # noqa: E402

from paper_2108_07031_b200 import reorder  # noqa: E402
from paper_2108_07031_b200._device import DeviceConnectivity  # noqa: E402
from paper_2108_07031_b200.solver import _params  # noqa: E402


def main():
    args = sys.argv[1:]
    m, L, g = (int(args[0]), int(args[1]), float(args[2])) if len(args) >= 3 else (800, 200, 1.03)
    iters = int(args[3]) if len(args) >= 4 else 50
    t = time.perf_counter()
    cloud = generate_naca_cloud(m, L, g, 20.0)
    conn = build_stencils(cloud)
    print(f"n={cloud.n_points} edges={conn.full.idx.size} build {time.perf_counter() - t:.1f}s", flush=True)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=iters)
    init = initial_primitives(cfg, cloud)
    t = time.perf_counter()
    dev = DeviceConnectivity(conn, perm=reorder.permutation(cloud, os.environ.get("KMF_ORDER", "natural")))
    print(f"context {time.perf_counter() - t:.2f}s", flush=True)
    for instrument in (False, True):
        dev.set_state(init.as_array())
        p = _params(cfg, instrument=instrument)
        dev.run(p, 3)  # warm-up (graph capture)
        t = time.perf_counter()
        h, k, _ = dev.run(p, iters)
        dt = time.perf_counter() - t
        print(f"instrument={instrument}: {iters} its in {dt:.4f}s -> {cloud.n_points * iters / dt:.3e} pt-it/s, "
              f"rdp {dt / (iters * cloud.n_points):.3e}; last residue {h[-1]:.6e}", flush=True)
        if instrument:
            print("stage seconds per iteration:", np.round(dev.stage_seconds() / iters * 1e6, 1), "us", flush=True)


if __name__ == "__main__":
    main()
