#!/usr/bin/env python
"""Benchmark: q-LSKUM outer iterations on B200 (driver contract, one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5]

With --gpus N > 1 and no torchrun environment, bench.py launches itself
under torchrun with N ranks on this node (one GPU per rank); under torchrun
WORLD_SIZE must equal N.

A step is one outer iteration of the solver (local time step + 4 SSP-RK
stages of q-variables, q-derivatives with 3 inner sweeps, flux residual with
wall/outer closures, state update + exact residue) over the whole synthetic
NACA 0012 cloud.  The default workload is BASELINE.json configs[4], the
configuration the metric's 1/2/4/8-B200 sweep and the paper's best
published RDP (3.41e-8 s, C++ on V100) are quoted on:
39,992,976 points, M 0.63, AoA 2 deg, second order, n_inner 3, fused; it
fits one B200 (~24 GB).  --config c1..c4 select the other BASELINE configs
(c1 = configs[0] in the reference's own second-order scheme; c1o1 the same
cloud in the first-order scheme configs[0] names, SolverConfig(order=1)).

Reported (ours):
  value          point-iterations/s with the state resident in HBM, each step
                 one CUDA-graph launch timed by CUDA events on the solver
                 stream, L2 flushed (256 MiB memset) between timed steps
                 (the 40M state is also far larger than L2);
  e2e            the same metric through the C ABI with host buffers: per
                 step the pinned H2D of the initial primitives, one outer
                 iteration and the D2H of the final primitives + residue
                 (kmf_run_cases: step k+1's upload and step k-1's download
                 overlap step k's iteration); e2e.serial the same three
                 transfers/calls one after another (kmf_set_state + kmf_run
                 + kmf_get_state), checked bitwise equal;
  roofline       flux_residual interior kernel (the dominant kernel) against
                 HBM (MEASURED_PEAKS.json) -- it is FP64-bound, so
                 roofline_fp64 reports executed DP-pipe instructions against
                 the FP64 peak measured in the same run (DFMA probe);
                 roofline_qgrad the first-order and sweep kernels against HBM;
  cpu_baseline   the reference package itself (kmf, numpy, installed under
                 baseline/_ref; its thread pool over all host cores) on a
                 bounded sample of the same workload: one outer iteration per
                 step of a geometric slab of the cloud (~100K points with its
                 deep halo, the reference's own types and solve);
                 cpu_baseline_port the C/OpenMP restatement (oracle/) on the
                 same kind of sample for context.
``--impl reference`` times the reference package alone on that sample (the
oracle port when baseline/_ref is missing).
Under torchrun (N > 1) rank 0 builds the connectivity once and shares it
with the other ranks through a memory-mapped store in /dev/shm.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (chord_points, layers, growth, mach, aoa, description)
    "c1": (400, 100, 1.06, 0.63, 2.0, "NACA0012 40K (400x100, g=1.06) M0.63 AoA2 second order n_inner=3"),
    "c1o1": (400, 100, 1.06, 0.63, 2.0, "NACA0012 40K (400x100, g=1.06) M0.63 AoA2 first order (qx = qy = 0)"),
    "c2": (800, 200, 1.03, 0.63, 2.0, "NACA0012 160K (800x200, g=1.03) M0.63 AoA2 second order n_inner=3"),
    "c3": (3160, 790, 1.00734, 0.85, 1.0, "NACA0012 2.5M (3160x790, g=1.00734) M0.85 AoA1 second order"),
    "c4": (6324, 1581, 1.003647, 0.63, 2.0, "NACA0012 10M (6324x1581, g=1.003647) M0.63 AoA2 second order"),
    "c5": (12648, 3162, 1.001821, 0.63, 2.0, "NACA0012 40M (12648x3162, g=1.001821) M0.63 AoA2 second order"),
}
# BASELINE configs[0] names the first-order scheme; the reference's solve()
# has none, so c1 runs the reference's second-order scheme
# and c1o1 the first-order extension (SolverConfig.order = 1)
ORDER = {"c1o1": 1}
# best published RDP for this metric, C++ optimised on V100,
# NACA 0012 40M points -> point-iterations/s
PUBLISHED = {"c5": 1.0 / 3.41e-8}
# configs above this size time the CPU oracle on a slab of this many owned points
CPU_SLAB_POINTS = int(os.environ.get("KMF_CPU_SLAB", 1_250_000))
METRIC = "point-iterations/sec (RDP = 1/value s/point/iter), NACA0012 q-LSKUM"
UNIT = "point-iterations/s"
# algorithmic bytes per point of one launch of the interior
# flux, first-order q-gradient and Jacobi sweep kernels
FLUX_BYTES_PER_POINT = 337
FO_BYTES_PER_POINT = 208
SWEEP_BYTES_PER_POINT = 272
# algorithmic bytes / DP ops of one whole point-iteration
# (timestep, 4 x [q, first order, 3 sweeps, flux, update], residue)
ITER_BYTES_PER_POINT = 6440
# first-order scheme: no q-gradient kernels (4 x (208 + 3 x 272) B fewer)
ITER_BYTES_PER_POINT_O1 = ITER_BYTES_PER_POINT - 4 * (208 + 3 * 272)
L2_FLUSH_BYTES = 256 << 20


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def self_launch(args) -> int:
    """--gpus N > 1 outside torchrun: relaunch this script under torchrun
    with N ranks on this node (127.0.0.1 rendezvous); rank 0 prints the
    JSON line.  NCCL's INFO log (communicator size and transport per rank)
    goes to stderr so stdout keeps the one JSON line."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return subprocess.call(cmd, env=env)


def dist_init(ws):
    if ws <= 1:
        return None
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    return dist


def allreduce_max(dist, v: float) -> float:
    if dist is None:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def build_config(name):
    from paper_2108_07031_b200 import SolverConfig, build_stencils, generate_naca_cloud, initial_primitives

    m, L, g, mach, aoa, _ = CONFIGS[name]
    t = time.perf_counter()
    cloud = generate_naca_cloud(m, L, g, 20.0)
    conn = build_stencils(cloud)  # native builder (libkmf_build.so), bit-exact with the reference's
    t1 = time.perf_counter()
    cfg = SolverConfig(mach=mach, aoa_deg=aoa, cfl=0.2, n_inner=3, mode="fused", order=ORDER.get(name, 2))
    init = initial_primitives(cfg, cloud)
    print(f"[bench] setup {name}: {cloud.n_points} points, {conn.full.idx.size} edges; generator+builder "
          f"{t1 - t:.1f} s, initial state {time.perf_counter() - t1:.1f} s", file=sys.stderr, flush=True)
    return cloud, conn, cfg, init


def setup(name, dist=None, rank=0):
    """(cloud, conn, cfg, initial primitives).  Multi-rank: rank 0 builds
    and stores to /dev/shm, every rank maps the same pages (store.py)."""
    if dist is None:
        return build_config(name)
    from paper_2108_07031_b200 import Primitives, SolverConfig, store

    box = [None]
    if rank == 0:
        import shutil

        from paper_2108_07031_b200 import builder

        # the other ranks wait: this one may use every core (torchrun sets
        # OMP_NUM_THREADS=1 per rank, which made the 40M build take 318 s)
        builder.lib().kmfb_set_threads(0)
        cloud, conn, cfg, init = build_config(name)
        need = 1.2 * (conn.full.idx.nbytes * 3 + conn.cloud.n_points * 8 * 40)  # idx, dx, dy + per-point arrays
        shm = Path("/dev/shm")
        if not shm.is_dir() or shutil.disk_usage(shm).free < need:
            shm = Path(tempfile.gettempdir())  # small /dev/shm: disk-backed, still one page-cache copy
        box[0] = tempfile.mkdtemp(prefix=f"kmf_{name}_", dir=shm)
        store.save(conn, box[0], extra={"init": init.as_array()})
        del cloud, conn, init
    dist.broadcast_object_list(box, src=0)
    conn, extra = store.load(box[0])
    barrier(dist)
    if rank == 0:
        import shutil

        shutil.rmtree(box[0], ignore_errors=True)  # mappings stay valid until the ranks exit
    _, _, _, mach, aoa, _ = CONFIGS[name]
    cfg = SolverConfig(mach=mach, aoa_deg=aoa, cfl=0.2, n_inner=3, mode="fused", order=ORDER.get(name, 2))
    return conn.cloud, conn, cfg, Primitives.from_array(np.asarray(extra["init"]))


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return None
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        busy = [s for s in sm if s > 400] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def oracle_sample(conn, init4n, cfg):
    """(Packed oracle connectivity, its initial state, points advanced per
    iteration, description) of a bounded CPU sample of the workload: the
    whole cloud up to CPU_SLAB_POINTS x 2, else the first geometric slab of
    ~CPU_SLAB_POINTS owned points with its deep halo (partition.py), flux
    and residue on the owned rows only (oracle n_act)."""
    from oracle import oracle as O
    from paper_2108_07031_b200.partition import build_part

    n = conn.cloud.n_points
    if n <= 2 * CPU_SLAB_POINTS:
        return O.Packed(conn), init4n, n, f"the whole {n}-point cloud"
    nslab = max(2, round(n / CPU_SLAB_POINTS))
    part = build_part(conn, 0, nslab, cfg.n_inner + 2)
    pk = O.Packed(part.conn)
    pk.c.n_act = part.n_owned
    desc = (f"geometric slab 1/{nslab} of the {n}-point cloud: {part.n_owned} owned points (counted) + "
            f"{part.global_ids.size - part.n_owned} deep-halo points (q-gradients only)")
    return pk, np.ascontiguousarray(np.asarray(init4n)[:, part.global_ids]), part.n_owned, desc


REF_SAMPLE_POINTS = int(os.environ.get("KMF_REF_SAMPLE", 64_000))
# point counts of the configuration clouds (m * L)
CONFIG_POINTS = {k: v[0] * v[1] for k, v in CONFIGS.items()}


def reference_package():
    """The reference package (kmf) from its offline install baseline/_ref, or None."""
    root = ROOT / "baseline" / "_ref"
    if not (root / "kmf" / "__init__.py").exists():
        return None
    sys.path.insert(0, str(root))
    try:
        import importlib

        kmf = importlib.import_module("kmf")
        for sub in ("geometry", "solver", "state"):
            importlib.import_module(f"kmf.{sub}")
        return kmf
    finally:
        sys.path.remove(str(root))


def reference_patch(kmf, name, target=REF_SAMPLE_POINTS):
    """A bounded sample of configuration `name` built ENTIRELY by the
    reference package (no code of this repo): the reference's generator
    makes the configuration's cloud, the `target` points nearest to the
    leading-edge wall point form a compact patch (wall points included, with
    their wall closures), the patch's outermost 3 % become an artificial
    far-field boundary (outer points, radial normals), and the reference's
    own builder and initial state set it up.  Returns (reference
    Connectivity, reference Primitives, points, description)."""
    m, L, g, mach, aoa, _ = CONFIGS[name]
    G = kmf.geometry
    cloud = G.generate_naca_cloud(m, L, g, 20.0)
    cfg = kmf.solver.SolverConfig(mach=mach, aoa_deg=aoa, n_outer=1)
    if cloud.n_points <= 1.5 * target:  # small configurations: the whole cloud
        rconn = G.build_stencils(cloud)
        desc = (f"the whole {cloud.n_points}-point configuration cloud, generated, built and initialised by the "
                f"reference package itself")
        return rconn, kmf.solver._initial_primitives(cfg, cloud), cloud.n_points, desc
    w = np.flatnonzero(cloud.flag == 1)
    c0 = int(w[np.argmin(cloud.x[w])])
    xc, yc = float(cloud.x[c0]), float(cloud.y[c0])
    d = np.hypot(cloud.x - xc, cloud.y - yc)
    near = np.sort(np.argpartition(d, target)[:target])
    dd = d[near]
    x, y = cloud.x[near], cloud.y[near]
    flag, nx, ny = cloud.flag[near].copy(), cloud.nx[near].copy(), cloud.ny[near].copy()
    rim = (dd > 0.97 * dd.max()) & (flag == 0)
    flag[rim] = 2
    nx[rim], ny[rim] = (x[rim] - xc) / dd[rim], (y[rim] - yc) / dd[rim]
    sub = G.PointCloud(x, y, flag, nx, ny)
    rconn = G.build_stencils(sub)
    prims = kmf.solver._initial_primitives(cfg, sub)
    desc = (f"a {target}-point patch of the {cloud.n_points}-point configuration cloud around the leading edge "
            f"({int((flag == 1).sum())} wall points, {int(rim.sum())} rim points as far field), generated, built "
            f"and initialised by the reference package itself")
    return rconn, prims, target, desc


def time_reference(kmf, rconn, prims, cfg, steps, warmup):
    """Seconds per step of the reference's own solve (solver.py:477-573),
    one outer iteration per step from the sample's initial state, its
    thread pool over every host core."""
    threads = os.cpu_count() or 1
    rc = kmf.solver.SolverConfig(mach=cfg.mach, aoa_deg=cfg.aoa_deg, gamma=cfg.gamma, cfl=cfg.cfl, n_outer=1,
                                 n_inner=cfg.n_inner, mode=cfg.mode, threads=threads)
    for _ in range(warmup):
        kmf.solver.solve(rc, rconn.cloud, rconn, initial_state=prims, instrument=False)
    t = []
    for _ in range(steps):
        t0 = time.perf_counter()
        kmf.solver.solve(rc, rconn.cloud, rconn, initial_state=prims, instrument=False)
        t.append(time.perf_counter() - t0)
    return t, threads


def cpu_baseline_reference(name, cfg, steps=3):
    kmf = reference_package()
    if kmf is None or cfg.order != 2:
        return None
    rconn, prims, counted, desc = reference_patch(kmf, name)
    t, threads = time_reference(kmf, rconn, prims, cfg, steps, 1)
    sec = float(np.median(t))
    return {"value": counted / sec, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"reference package kmf (numpy, baseline/_ref) solve(), one outer iteration per step, median of "
                      f"{steps} after 1 warm-up ({sec:.2f} s each) on {desc}; threads={threads}"}


def cpu_baseline(conn, cfg, init, target_s=12.0):
    """Oracle (CPU restatement of the reference) on a bounded sample of
    ~target_s seconds of whole outer iterations (oracle_sample)."""
    from oracle import oracle as O
    from paper_2108_07031_b200 import free_stream

    threads = os.cpu_count() or 1
    O.set_threads(threads)
    pk, init4n, npts, desc = oracle_sample(conn, init.as_array(), cfg)
    fs = free_stream(cfg.mach, cfg.aoa_deg, cfg.gamma)
    fsv = [fs.rho[0], fs.u1[0], fs.u2[0], fs.p[0]]
    t = time.perf_counter()
    O.solve(pk, init4n, fsv, 1, gamma=cfg.gamma, cfl=cfg.cfl, n_inner=cfg.n_inner if cfg.order == 2 else 0)
    one = time.perf_counter() - t
    if one > 0.5 * target_s:  # the first whole iteration is the sample
        iters, sec = 1, one
    else:
        iters = int(min(200, max(2, target_s / max(one, 1e-3))))
        t = time.perf_counter()
        O.solve(pk, init4n, fsv, iters, gamma=cfg.gamma, cfl=cfg.cfl, n_inner=cfg.n_inner if cfg.order == 2 else 0)
        sec = time.perf_counter() - t
    return {"value": npts * iters / sec, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{iters} outer iterations ({sec:.1f} s) on {desc}; oracle/kmf_oracle.c (C restatement of "
                      f"the reference) with OpenMP over {threads} threads"}


def qgrad_roofline(n_fo, n_sweep, fo_s, sweep_s, peak, peak_kind, share):
    """First-order and sweep kernels against HBM: SURVEY 8(d)'s algorithmic
    bytes per point (208 / 272) x the points one launch covers, divided by
    the launch's average duration (event nodes on its stream)."""
    fo = FO_BYTES_PER_POINT * n_fo / fo_s / 1e9
    sw = SWEEP_BYTES_PER_POINT * n_sweep / sweep_s / 1e9
    return {"bound": "hbm", "unit": "GB/s", "peak": peak, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
            "first_order": {"kernel": "k_first_order", "bytes_per_point": FO_BYTES_PER_POINT, "launch_us": fo_s * 1e6,
                            "achieved": fo, "frac": fo / peak},
            "sweep": {"kernel": "k_sweep", "bytes_per_point": SWEEP_BYTES_PER_POINT, "launch_us": sweep_s * 1e6,
                      "achieved": sw, "frac": sw / peak},
            "share_of_step": share}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0}, "fallback"


def roofline_fp64(counts, n_cloud, n_flux, launch_s, dfma_rate, probe_tflops):
    """The binding roofline of the flux kernel: executed DP-pipe thread
    instructions (DFMA + DMUL + DADD, ncu count of this build, per point of
    the cloud) per second against the DFMA instruction peak measured in the
    same run.  (SURVEY 8(d)'s 13,214 "DP ops"/point weighs each libdevice
    transcendental by its instruction count -- exp 18, erf 25, log 28,
    div/sqrt 10 -- which this kernel does not execute: its lean
    exp/erf/rcp/rsqrt and shared per-state constants take 4.7K DP-pipe
    instructions per point, so that count is not a rate against the pipe.)"""
    out = {"bound": "fp64", "unit": "T DP-pipe thread-inst/s", "peak": dfma_rate,
           "peak_source": f"DFMA probe in this run: {probe_tflops:.2f} TFLOP/s = {dfma_rate:.2f} T DFMA/s"}
    if counts:
        dp_pt = counts["dp_thread_inst_per_launch"] / n_cloud  # counted single-GPU over the whole cloud
        ach = dp_pt * n_flux / launch_s / 1e12
        out.update({"achieved": ach, "frac": ach / dfma_rate, "executed_dp_inst_per_point": dp_pt,
                    "ncu_fp64_pipe_active_pct": counts.get("fp64_pipe_active_pct"),
                    "counts_source": f"profiles/flux_counts_{counts['config']}.json (ncu, {counts['kernel'][:40]})"})
    else:
        out.update({"achieved": None, "frac": None, "counts_source": "no ncu count for this config"})
    return out


def rank_solver_checked(args, conn, cfg, init, dist, rank, local):
    """The N-rank solver on args.transport, checked before it is timed: its
    first `args.check_iters` residues must equal, bit for bit, a single-GPU
    solve of the whole cloud on rank 0 (the partitioned arithmetic is the
    single-GPU one).  A peer transport that fails the check (error, deadline
    or mismatch on any rank) is replaced by NCCL, and the line says so."""
    import dataclasses

    from paper_2108_07031_b200 import _lib
    from paper_2108_07031_b200._device import DeviceConnectivity
    from paper_2108_07031_b200.dist import RankSolver
    from paper_2108_07031_b200.solver import _params

    k = max(args.check_iters, 0)
    ref = None
    if k and rank == 0:
        t = time.perf_counter()
        full = DeviceConnectivity(conn, device=local)
        full.set_state(init.as_array())
        ref, _, _ = full.run(_params(dataclasses.replace(cfg, n_outer=k)), k)
        full.close()
        print(f"[bench] single-GPU reference residues ({k} iterations) {time.perf_counter() - t:.1f} s",
              file=sys.stderr, flush=True)
    transport, fallback = args.transport, None
    while True:
        err, same = None, True
        try:
            rs = RankSolver(conn, dist, n_inner=cfg.n_inner, device=local, scheme=args.partition, transport=transport)
            if k:
                hist, _ = rs.run(dataclasses.replace(cfg, n_outer=k), init.as_array(), k)
                same = rank != 0 or bool(np.array_equal(hist, ref))
        except (_lib.DeviceError, ValueError) as e:
            err, same, rs = str(e).splitlines()[0][:200], False, None
        flags = [None] * dist.get_world_size()
        dist.all_gather_object(flags, (same, err))
        ok = all(f[0] for f in flags)
        if ok or transport == "nccl":
            if not ok:
                raise SystemExit(f"bench: the {transport} transport failed its check: {flags}")
            break
        fallback = {"from": transport, "why": [f[1] or ("residues differ from the single-GPU solve" if not f[0]
                                                        else None) for f in flags]}
        print(f"[bench] {transport} transport failed its check, falling back to NCCL: {fallback}", file=sys.stderr,
              flush=True)
        transport, rs = "nccl", None
        import gc

        gc.collect()
    info = {"name": transport, "fallback": fallback,
            "check": {"iterations": k, "bitwise_vs_single_gpu": bool(k)} if k else None}
    part = rs.rp.part
    print(f"[bench] rank {rank}/{dist.get_world_size()} on cuda:{local}: {transport} transport, sends "
          f"{ {p: int(v.size) for p, v in part.send.items()} } halo points to / receives "
          f"{ {p: int(v.size) for p, v in part.recv.items()} } from its peers per stage; first {k} residues "
          f"bitwise equal to the single-GPU solve", file=sys.stderr, flush=True)
    return rs, info


def run_ours(args):
    ws, rank, local = dist_env()
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    dist = dist_init(ws)
    from paper_2108_07031_b200 import _lib
    from paper_2108_07031_b200._device import DeviceConnectivity
    from paper_2108_07031_b200.solver import _params
    import ctypes as C

    L = _lib.lib()
    _lib.require_device()
    from paper_2108_07031_b200 import reorder

    shared_gpu = ws > 1 and os.environ.get("KMF_SHARE_GPU") == "1"
    if shared_gpu:
        # functional run of the N-rank path on fewer GPUs (tests / one-GPU
        # boxes): ranks share devices and NCCL connects them over its socket
        # transport (one fake host per rank).  Timings are NOT scaling data;
        # the JSON line says so ("shared_gpu": true).
        local = local % L.kmf_device_count()
        os.environ["NCCL_HOSTID"] = f"kmf-bench-host-{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        os.environ.setdefault("NCCL_IB_DISABLE", "1")

    cloud, conn, cfg, init = setup(args.config, dist, rank)
    n = cloud.n_points
    transport_info = None
    if ws > 1:
        # geometric partition over the ranks; the halo exchange and residue
        # reduction inside the iteration graph over the chosen transport
        # (paper_2108_07031_b200/dist.py), validated before timing
        rs, transport_info = rank_solver_checked(args, conn, cfg, init, dist, rank, local)
        dev = rs.dev
        part = rs.rp.part
        print(f"[bench] rank {rank}: {part.n_owned} owned + {part.global_ids.size - part.n_owned} halo points "
              f"({args.partition}), interior pass {part.interior_end[-1]} points", file=sys.stderr, flush=True)
        local_init = np.ascontiguousarray(init.as_array()[:, rs.rp.part.global_ids])
    else:
        t = time.perf_counter()
        dev = DeviceConnectivity(conn, device=local, perm=reorder.permutation(cloud, args.order))
        print(f"[bench] device context {time.perf_counter() - t:.1f} s", file=sys.stderr, flush=True)
        local_init = init.as_array()
    n_local = local_init.shape[1]
    part_stats = None
    if ws > 1:
        # per-rank partition shape (rank 0 reports all ranks): owned and halo
        # points, the interior pass (owned points deep enough to run before
        # the stage's halo exchange lands) and the exchange volume
        mine = {"owned": part.n_owned, "halo": int(part.global_ids.size - part.n_owned),
                "interior_flux": int(part.interior_end[min(cfg.n_inner + 3, part.depth + 1)]),
                "recv_points": int(sum(v.size for v in part.recv.values())), "peers": len(part.recv)}
        every = [None] * ws
        dist.all_gather_object(every, mine)
        part_stats = {"scheme": args.partition, "depth": part.depth, "ranks": every,
                      "interior_flux_fraction_min": min(r["interior_flux"] / r["owned"] for r in every),
                      "halo_fraction_max": max(r["halo"] / r["owned"] for r in every)}
    params = _params(cfg)
    peak_fp64 = C.c_double(0.0)
    _lib.check(L.kmf_fp64_peak(C.byref(peak_fp64)), "kmf_fp64_peak")

    # ---- device-resident value --------------------------------------------
    dev.set_state(local_init)
    W, K = max(args.warmup, 0), args.steps
    step_ms = np.zeros(max(K, W, 1))
    kern_ms = np.zeros((step_ms.size, _lib.BENCH_KERNELS))  # interior flux, first order, sweeps
    lps = C.c_int(0)
    if W:
        _lib.check(L.kmf_bench_steps(dev.handle, C.byref(params), W, L2_FLUSH_BYTES, _lib.dptr(step_ms),
                                     _lib.dptr(kern_ms), C.byref(lps)), "warm-up")
    barrier(dist)
    with Clocks(local) as clk:
        _lib.check(L.kmf_bench_steps(dev.handle, C.byref(params), K, L2_FLUSH_BYTES, _lib.dptr(step_ms),
                                     _lib.dptr(kern_ms), C.byref(lps)), "timed steps")
    barrier(dist)
    total_s = allreduce_max(dist, float(step_ms[:K].sum()) * 1e-3)
    value = n * K / total_s  # every step advances all n points once (strong scaling over ranks)
    kern_s = kern_ms[:K].sum(axis=0) * 1e-3
    n_sweeps = cfg.n_inner if cfg.order == 2 else 0
    flux_launch_s = float(kern_s[0]) / (4 * K)
    fo_launch_s = float(kern_s[1]) / (4 * K) if n_sweeps else 0.0
    sweep_launch_s = float(kern_s[2]) / (4 * n_sweeps * K) if n_sweeps else 0.0
    stage_share = float(kern_s[0] / (step_ms[:K].sum() * 1e-3))

    # ---- end to end through the C ABI with pinned host buffers ------------
    # (1) kmf_run_cases: every step is one case -- upload of its initial
    # state, one outer iteration, download of its final state and residue --
    # with step k+1's upload and step k-1's download on the copy engines
    # while step k iterates; (2) the same three calls serialised per step
    # (kmf_set_state + kmf_run + kmf_get_state).
    host_in = _lib.pinned((4, n_local))
    host_out = [_lib.pinned((4, n_local)) for _ in range(2)]
    host_in[...] = local_init
    hist = np.zeros(1)
    done, conv = C.c_int(0), C.c_int(0)
    e2e_params = _params(cfg)

    def cases(m):
        parr = (_lib.Params * m)(*([e2e_params] * m))
        pin = (C.c_void_p * m)(*([host_in.ctypes.data] * m))
        pout = (C.c_void_p * m)(*[host_out[k % 2].ctypes.data for k in range(m)])
        hist_c = np.zeros(m)
        _lib.check(L.kmf_run_cases(dev.handle, parr, 1, m, pin, pout, None, _lib.dptr(hist_c), None, None, None),
                   "run_cases")
        return hist_c

    def serial_step():
        _lib.check(L.kmf_set_state(dev.handle, _lib.dptr(host_in)), "set_state")
        _lib.check(L.kmf_run(dev.handle, C.byref(e2e_params), 1, _lib.dptr(hist), C.byref(done), C.byref(conv)),
                   "run")
        _lib.check(L.kmf_get_state(dev.handle, _lib.dptr(host_out[0]), None), "get_state")

    cases(max(W, 2))
    barrier(dist)
    t0 = time.perf_counter()
    e2e_hist = cases(K)
    e2e_s = allreduce_max(dist, time.perf_counter() - t0)
    streamed = host_out[(K - 1) % 2].copy()
    for _ in range(max(W, 1)):
        serial_step()
    barrier(dist)
    t0 = time.perf_counter()
    for _ in range(K):
        serial_step()
    ser_s = allreduce_max(dist, time.perf_counter() - t0)
    if not (np.all(e2e_hist == hist[0]) and np.array_equal(streamed, host_out[0])):
        raise SystemExit("bench: streamed and serial end-to-end steps disagree")
    e2e = {"value": n * K / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 4 * n_local * 8,
           "d2h_bytes_per_step": 4 * n_local * 8 + 8, "ms_per_step": 1e3 * e2e_s / K,
           "path": "kmf_run_cases (pinned host in/out per step, copies overlapped with the previous/next step)",
           "serial": {"value": n * K / ser_s, "ms_per_step": 1e3 * ser_s / K,
                      "path": "kmf_set_state(pinned) + kmf_run(1 iteration) + kmf_get_state(pinned) per step"}}

    if rank != 0:
        return
    peaks, peak_kind = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # points the timed launches cover: the whole cloud on one GPU; under a
    # partition the timed (event-marked) launches are the interior pass's
    # (partition.stage_ranges), the band pass runs unmarked on its own stream
    n_fo = n_sweep = n_flux = n
    if ws > 1:
        from paper_2108_07031_b200.partition import stage_ranges

        ranges = {name: iv for name, iv, _ in stage_ranges(rs.rp.part, cfg.n_inner if n_sweeps else 0)}
        n_flux = ranges["flux"][1]
        if n_sweeps:
            n_fo = ranges["first_order"][1]
            n_sweep = sum(ranges[f"sweep{s}"][1] for s in range(1, n_sweeps + 1)) / n_sweeps
    achieved_gbs = FLUX_BYTES_PER_POINT * n_flux / flux_launch_s / 1e9
    dfma_rate = peak_fp64.value / 2.0  # DP-pipe instructions/s (TFLOP/s / 2)
    # executed DP-pipe instructions and DRAM traffic of one flux launch,
    # measured once per kernel build by ncu (tools/flux_counts.sh)
    traffic, counts = None, None
    tf = ROOT / "profiles" / f"flux_counts_{args.config}.json"
    if tf.exists():
        counts = json.loads(tf.read_text())
        traffic = counts.get("dram_bytes_per_launch")
    iter_bytes = ITER_BYTES_PER_POINT_O1 if cfg.order == 1 else ITER_BYTES_PER_POINT
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": K,
        "warmup": W,
        "ms_per_step": 1e3 * total_s / K,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": value / PUBLISHED[args.config] if args.config in PUBLISHED else None,
        "vs_baseline_source": ("BASELINE.md: paper's best published RDP 3.41e-8 s (C++ optimised, V100, NACA 0012 "
                               "40M points)") if args.config in PUBLISHED else None,
        "dtype": "f64",
        "data": "synthetic (procedurally generated NACA 0012 O-cloud, reference generator restated bit-exactly)",
        "config": {"workload": CONFIGS[args.config][5], "config_key": args.config, "n_points": n,
                   "n_edges": int(conn.full.idx.size), "n_inner": cfg.n_inner, "order": cfg.order, "mode": cfg.mode,
                   "l2": "flushed between timed steps (256 MiB memset on the solver stream)",
                   "parallelism": (f"partition x{ws} ({args.partition}, deep halo, {transport_info['name']} halo "
                                   "exchange overlapped with the interior pass)") if ws > 1 else "single GPU",
                   "point_order": args.order},
        "rdp_s_per_point_iter": 1.0 / value,
        "e2e": e2e,
        "gpu_launches": int(lps.value) * K,
        "roofline": {"bound": "hbm", "kernel": "k_flux<fused> (flux_residual interior)",
                     "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": achieved_gbs / hbm_peak,
                     "traffic": traffic, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "bytes_per_point": FLUX_BYTES_PER_POINT, "launch_us": flux_launch_s * 1e6,
                     "share_of_step": stage_share,
                     "note": "the flux kernel is FP64-pipe bound (SURVEY.md 8(d)); see roofline_fp64"},
        "roofline_iteration": {
            "bound": "hbm", "bytes_per_point_iter": iter_bytes,
            "achieved": iter_bytes * value / ws / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": iter_bytes * value / ws / 1e9 / hbm_peak,
            "note": "whole outer iteration against the HBM roofline implied by SURVEY 8(d)'s 6.44 KB per "
                    "point-iteration (north star), per GPU"},
        "roofline_fp64": roofline_fp64(counts, n, n_flux, flux_launch_s, dfma_rate, peak_fp64.value),
        "roofline_qgrad": qgrad_roofline(n_fo, n_sweep, fo_launch_s, sweep_launch_s, hbm_peak, peak_kind, float(
            kern_s[1] + kern_s[2]) / (step_ms[:K].sum() * 1e-3)) if n_sweeps else None,
        "clocks": clk.summary(),
        "partition": part_stats,
        "transport": transport_info,
        **({"shared_gpu": True, "note": "KMF_SHARE_GPU: ranks share GPUs (NCCL over sockets / IPC on one device); "
                                        "not scaling data"} if shared_gpu else {}),
    }
    if not args.no_cpu_baseline and ws == 1:
        port = cpu_baseline(conn, cfg, init)
        ref = cpu_baseline_reference(args.config, cfg)
        line["cpu_baseline"] = ref or port
        if ref:
            line["cpu_baseline_port"] = port
    print(json.dumps(line), flush=True)


def run_reference(args):
    """The reference arm: the reference package's own solve (kmf from
    baseline/_ref, numpy, all host threads) on a bounded sample of the
    configuration that the reference package itself generates, builds and
    initialises (reference_patch: no code of this repo runs or is loaded),
    one outer iteration per step; the oracle port (C/OpenMP restatement)
    when the package is not installed or for the first-order scheme."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    W, K = max(args.warmup, 0), args.steps
    kmf = reference_package()
    order = 1 if args.config in ORDER else 2
    if kmf is not None and order == 2:
        rconn, prims, npts, desc = reference_patch(kmf, args.config)
        _, _, _, mach, aoa, _ = CONFIGS[args.config]
        cfg = type("Cfg", (), dict(mach=mach, aoa_deg=aoa, gamma=1.4, cfl=0.2, n_inner=3, mode="fused"))()
        t, threads = time_reference(kmf, rconn, prims, cfg, K, W)
        sec = float(sum(t))
        kind = "reference"
        sample = (f"each step one outer iteration of the reference package kmf (numpy, baseline/_ref) solve() "
                  f"({K} timed after {W} warm-up) on {desc}; threads={threads}")
        n = None
    else:
        from oracle import oracle as O
        from paper_2108_07031_b200 import free_stream

        cloud, conn, cfg, init = setup(args.config)
        n = cloud.n_points
        threads = os.cpu_count() or 1
        O.set_threads(threads)
        pk, prims, npts, desc = oracle_sample(conn, init.as_array(), cfg)
        fs = free_stream(cfg.mach, cfg.aoa_deg, cfg.gamma)
        fsv = [fs.rho[0], fs.u1[0], fs.u2[0], fs.p[0]]
        n_inner = cfg.n_inner if cfg.order == 2 else 0
        if W:
            _, prims, _, _, _ = O.solve(pk, prims, fsv, W, gamma=cfg.gamma, cfl=cfg.cfl, n_inner=n_inner)
        t0 = time.perf_counter()
        O.solve(pk, prims, fsv, K, gamma=cfg.gamma, cfl=cfg.cfl, n_inner=n_inner)
        sec = time.perf_counter() - t0
        kind = "port"
        sample = (f"each step one outer iteration ({K} timed after {W} warm-up) on {desc}; the C restatement "
                  f"oracle/kmf_oracle.c (OpenMP, {threads} threads)"
                  + ("" if kmf is None else "; the reference's solve() has no first-order scheme"))
    value = npts * K / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": K,
        "warmup": W, "ms_per_step": 1e3 * sec / K, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": value / PUBLISHED[args.config] if args.config in PUBLISHED else None,
        "dtype": "f64", "data": "synthetic (procedurally generated NACA 0012 O-cloud)",
        "config": {"workload": CONFIGS[args.config][5], "config_key": args.config,
                   "n_points": n if n is not None else CONFIG_POINTS.get(args.config)},
        "rdp_s_per_point_iter": 1.0 / value,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="c5",
                    help="c5 (default): 40M points, BASELINE configs[4]; c2: 160K, configs[1]")
    ap.add_argument("--partition", choices=("sectors", "bands"), default="sectors",
                    help="ownership scheme of the multi-GPU partition (partition.py)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", choices=("peer", "nccl"), default="peer",
                    help="N > 1: halo / residue transport (peer: the update kernels push the halo into the peers' "
                         "memory; nccl: NCCL send/recv + all-reduce); either inside the iteration graph")
    ap.add_argument("--check-iters", type=int, default=2,
                    help="N > 1: residues checked bitwise against a single-GPU solve before timing (0: skip)")
    ap.add_argument("--order", choices=("natural", "hilbert", "ringtile2", "ringtile4", "ringtile8"),
                    default=os.environ.get("KMF_ORDER", "natural"),
                    help="device point order (bitwise neutral, locality only)")
    args = ap.parse_args()
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1 and args.impl == "ours":
        sys.exit(self_launch(args))
    if ws is not None and int(ws) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws} (launch N ranks for --gpus N)")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
