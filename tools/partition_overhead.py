"""Cost of the partitioned schedule on ONE GPU: N peer-linked ranks of one
cloud run concurrently on the same device (kmf_run_linked) against the
single-domain solve of the same cloud (kmf_run), same iterations, wall
clock around synchronous runs after a warm-up run.  On one device the ranks
share the SMs, so the ideal ratio is 1.0: the shortfall is the schedule's
own cost (extra halo work, per-stage waits, launch count), not NVLink.

    python tools/partition_overhead.py [config] [iterations] [ranks,...]
"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # ranks x 2 spinning streams on one device
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2108_07031_b200 import _lib  # noqa: E402
from paper_2108_07031_b200._device import DeviceConnectivity  # noqa: E402
from paper_2108_07031_b200.dist import RankPart  # noqa: E402
from paper_2108_07031_b200.partition import owner_map  # noqa: E402
from paper_2108_07031_b200.solver import _params  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ranks = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "2,4,8").split(",")]
cloud, conn, cfg, init = bench.build_config(cfg_name)
L = _lib.lib()
p = _params(cfg)
g = init.as_array()

dev = DeviceConnectivity(conn)
dev.set_state(g)
dev.run(p, 8)
dev.set_state(g)
t = time.perf_counter()
h1, _, _ = dev.run(p, iters)
single = time.perf_counter() - t
dev.close()
print(f"{cfg_name}: single domain {1e3 * single / iters:.3f} ms/iteration", flush=True)
for nr in ranks:
    owner = owner_map(cloud, nr, "sectors")
    parts = [RankPart(conn, r, nr, cfg.n_inner, scheme="sectors", owner=owner) for r in range(nr)]
    h = (C.c_void_p * nr)(*[rp.dev.handle.value for rp in parts])
    _lib.check(L.kmf_peer_link(h, nr), "link")
    hist = np.zeros(iters)
    done, conv = C.c_int(0), C.c_int(0)
    for rp in parts:
        rp.set_state(g)
    _lib.check(L.kmf_run_linked(h, nr, C.byref(p), 8, _lib.dptr(hist), C.byref(done), C.byref(conv)), "warm")
    for rp in parts:
        rp.set_state(g)
    t = time.perf_counter()
    _lib.check(L.kmf_run_linked(h, nr, C.byref(p), iters, _lib.dptr(hist), C.byref(done), C.byref(conv)), "run")
    el = time.perf_counter() - t
    halo = sum(rp.part.global_ids.size - rp.part.n_owned for rp in parts)
    print(f"{cfg_name}: {nr} peer-linked ranks on one GPU {1e3 * el / iters:.3f} ms/iteration, "
          f"throughput ratio {single / el:.3f}, bitwise {np.array_equal(hist, h1)}, "
          f"halo points {halo} ({halo / cloud.n_points:.2%} of the cloud)", flush=True)
    del parts
