"""Native builder vs the scipy restatement of the reference builder, bit for
bit on every Connectivity array, at BASELINE sizes (one-off, CPU only; the
10M case needs ~40 GB and ~25 min for the scipy side).

    python tools/builder_parity.py c3 c4      # 2.5M and 10M
"""

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from oracle.builder_ref import build_stencils_ref  # noqa: E402
from paper_2108_07031_b200 import build_stencils, generate_naca_cloud  # noqa: E402

SIZES = {"c1": (400, 100, 1.06), "c2": (800, 200, 1.03), "c3": (3160, 790, 1.00734), "c4": (6324, 1581, 1.003647)}
F = ("ptr", "idx", "dx", "dy", "sxx", "sxy", "syy", "det")


def diff(a, b):
    bad = [f"full.{k}" for k in F if not np.array_equal(getattr(a.full, k), getattr(b.full, k))]
    for kind in a.split:
        bad += [f"{kind}.{k}" for k in F if not np.array_equal(getattr(a.split[kind], k), getattr(b.split[kind], k))]
        bad += [f"det_safe{kind}"] if not np.array_equal(a.det_safe[kind], b.det_safe[kind]) else []
    bad += [k for k in ("d_min", "d_mean") if not np.array_equal(getattr(a, k), getattr(b, k))]
    for fr in ("wall_frame", "outer_frame"):
        fa, fb = getattr(a, fr), getattr(b, fr)
        for st in ("tplus", "tminus", "normal"):
            bad += [f"{fr}.{st}.{k}" for k in F if not np.array_equal(getattr(getattr(fa, st), k),
                                                                     getattr(getattr(fb, st), k))]
        bad += [f"{fr}.fallback"] if fa.fallback != fb.fallback else []
    return bad


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c3"]:
        cloud = generate_naca_cloud(*SIZES[name], 20.0)
        t = time.perf_counter()
        nat = build_stencils(cloud)
        tn = time.perf_counter() - t
        t = time.perf_counter()
        ref = build_stencils_ref(cloud)
        ts = time.perf_counter() - t
        print(f"{name}: n={cloud.n_points} edges={nat.full.idx.size} native {tn:.1f} s, scipy {ts:.1f} s, "
              f"mismatching arrays: {diff(nat, ref) or 'none'}", flush=True)
        del nat, ref
