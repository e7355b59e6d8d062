"""Try the NCCL rank path with two processes on ONE GPU (dev aid): NCCL may
refuse duplicate devices; if it accepts, compare with the single domain."""
import faulthandler
import os
import socket
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402


def worker(rank, world, port, q):
    faulthandler.dump_traceback_later(240, exit=True)
    import torch.distributed as dist

    from conftest import perturbed_state
    from paper_2108_07031_b200 import SolverConfig, build_stencils, generate_naca_cloud
    from paper_2108_07031_b200.dist import RankSolver
    from paper_2108_07031_b200.state import prims_array

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if os.environ.get("FAKE_HOSTS"):
        # each rank reports its own host: NCCL skips its same-host duplicate-
        # device check and connects the ranks through its socket transport
        os.environ["NCCL_HOSTID"] = f"kmf-fake-host-{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        os.environ.setdefault("NCCL_IB_DISABLE", "1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
        conn = build_stencils(cloud)
        cfg = SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=6)
        rs = RankSolver(conn, dist, n_inner=3, device=0, scheme=sys.argv[1] if len(sys.argv) > 1 else "sectors")
        hist, conv = rs.run(cfg, prims_array(perturbed_state(cloud)), cfg.n_outer)
        gid, prims, _ = rs.rp.owned_state()
        q.put((rank, hist, gid, prims, None))
    except Exception as e:  # report, do not hang
        q.put((rank, None, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    from conftest import perturbed_state
    from paper_2108_07031_b200 import SolverConfig, build_stencils, generate_naca_cloud, solve
    from paper_2108_07031_b200.state import prims_array

    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=150) for _ in range(2)]
    for p in procs:
        p.join(timeout=30)
    cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
    conn = build_stencils(cloud)
    ref = solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=6), cloud, conn, initial_state=perturbed_state(cloud),
                instrument=False)
    for rank, hist, gid, prims, err in out:
        if err:
            print(f"rank {rank}: error {err}")
            continue
        print(f"rank {rank}: history equal {np.array_equal(hist, ref.residue_history)}, state equal "
              f"{np.array_equal(prims, prims_array(ref.primitives)[:, gid])}")
