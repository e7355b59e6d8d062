"""Per-kernel device times of one outer iteration (development aid, not the
bench): kmf_bench_steps' event-node pass on a BASELINE configuration.

    python tools/kperf.py [c3|c5|...] [steps]
"""

import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2108_07031_b200 import _lib  # noqa: E402
from paper_2108_07031_b200._device import DeviceConnectivity  # noqa: E402
from paper_2108_07031_b200.solver import _params  # noqa: E402


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    cloud, conn, cfg, init = bench.build_config(cfg_name)
    dev = DeviceConnectivity(conn)
    dev.set_state(init.as_array())
    L = _lib.lib()
    p = _params(cfg)
    step = np.zeros(steps)
    kern = np.zeros((steps, _lib.BENCH_KERNELS))
    lps = C.c_int(0)
    for rep in range(2):  # the first pass warms up (graph capture)
        _lib.check(L.kmf_bench_steps(dev.handle, C.byref(p), steps, bench.L2_FLUSH_BYTES, _lib.dptr(step),
                                     _lib.dptr(kern), C.byref(lps)), "bench")
    k = kern.mean(axis=0)
    ni = cfg.n_inner if cfg.order == 2 else 0
    print(f"{cfg_name}: step {np.median(step):.3f} ms | flux {k[0] / 4:.3f} ms/launch | first order "
          f"{k[1] / 4 if ni else 0:.3f} | sweep {k[2] / (4 * ni) if ni else 0:.3f} | other "
          f"{np.median(step) - k.sum():.3f} ms/step", flush=True)


if __name__ == "__main__":
    main()
