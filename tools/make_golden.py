"""Generate the golden fixtures under tests/golden/ by running the reference.

This script is the ONLY place that imports the reference package
(`/root/reference/pkg/src/kmf`, read-only).  It runs in the build container
(numpy/scipy CPU); the fixtures it writes are committed so the GPU box, which
has no `/root/reference`, can check the oracle and the CUDA path against the
reference's own outputs.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tools/make_golden.py <case> [<case> ...]

Cases
-----
small      2,400-pt `small_naca` cloud (reference tests/conftest.py:31-38):
           connectivity digests, per-stage operator outputs on the perturbed
           state (tests/test_solver.py:98) and on the solver's initial state,
           and short solve histories (fused/split4, AoA 0 mirror run).
hist2k     1000-iteration M0.63/AoA2 history + final state on small_naca, and
           300 iterations of the transonic M0.85/AoA1 case.
kinetics   split_flux / full_flux / state transforms on seeded random states.
lattice    lattice / jittered / channel clouds (tests/conftest.py:7-28,
           tests/test_solver.py:74-95): connectivity digests and the
           uniform-flow and wall-tangent residuals.
c40k       config 1 (bench.py:37 POINT_LEVELS["40k"]): digests + 1000-iter
           history + final state (long: ~35 min on 8 threads).
c160k      config 2 (800, 200, 1.03): digests + 20-iter history.
c2p5m      config 3 (3160, 790, 1.00734), M0.85 AoA1: digests + 2 iterations.
gammas     gamma = 5/3 and 1.3 (the decode's other two evaluation paths): split
           fluxes and entropy variables of the kinetics states, flux_residual +
           apply_boundary on small_naca, and a 20-iteration solve.

Every digest is sha256 over the little-endian C-contiguous bytes of the array
cast to int64 (integer arrays) or float64 (real arrays).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

import kmf  # noqa: F401  (the reference; PYTHONPATH must point at it)
from kmf.geometry import (
    INTERIOR,
    OUTER,
    WALL,
    PointCloud,
    build_stencils,
    generate_naca_cloud,
)
from kmf.kinetics import full_flux, split_flux
from kmf.lsq import compute_q_derivatives, first_order_q_gradients
from kmf.solver import (
    SolverConfig,
    _initial_primitives,
    apply_boundary,
    flux_residual,
    local_timestep,
    residue_norm,
    solve,
    state_update_rk,
)
from kmf.state import (
    FlowState,
    PositivityError,
    Primitives,
    conserved_to_primitives,
    free_stream,
    primitives_to_conserved,
    primitives_to_q,
    q_to_primitives,
)

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def digest(a) -> str:
    a = np.asarray(a)
    if a.dtype.kind in "biu":
        a = a.astype("<i8")
    else:
        a = a.astype("<f8")
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _stencil_digests(prefix, s, out):
    for name in ("ptr", "idx", "dx", "dy", "sxx", "sxy", "syy", "det"):
        out[f"{prefix}.{name}"] = digest(getattr(s, name))


def conn_digests(cloud: PointCloud, conn) -> dict:
    out = {}
    for name in ("x", "y", "flag", "nx", "ny"):
        out[f"cloud.{name}"] = digest(getattr(cloud, name))
    _stencil_digests("full", conn.full, out)
    for kind, s in conn.split.items():
        _stencil_digests(f"split[{kind}]", s, out)
        out[f"det_safe[{kind}]"] = digest(conn.det_safe[kind])
    out["d_min"] = digest(conn.d_min)
    out["d_mean"] = digest(conn.d_mean)
    for fname in ("wall_frame", "outer_frame"):
        fr = getattr(conn, fname)
        if fr is None:
            out[fname] = None
            continue
        for name in ("points", "tx", "ty", "nx", "ny"):
            out[f"{fname}.{name}"] = digest(getattr(fr, name))
        for sname in ("tplus", "tminus", "normal"):
            _stencil_digests(f"{fname}.{sname}", getattr(fr, sname), out)
        out[f"{fname}.fallback"] = sorted([int(k), v] for k, v in fr.fallback.items())
    out["n_points"] = int(cloud.n_points)
    out["n_edges"] = int(conn.full.idx.size)
    return out


def perturbed_state(cloud, mach=0.63, aoa=2.0, gamma=1.4, amp=0.02):
    # restated from reference tests/test_solver.py:98-102
    fs = free_stream(mach, aoa, gamma, n=cloud.n_points)
    bump = amp * np.exp(-((cloud.x - 1.8) ** 2 + cloud.y ** 2) / 0.16)
    return Primitives(fs.rho * (1.0 + bump), fs.u1, fs.u2, fs.p * (1.0 + gamma * bump))


def prims_arr(p: Primitives) -> np.ndarray:
    return np.stack([p.rho, p.u1, p.u2, p.p])


def stage_ops(prefix, cloud, conn, prims, mach, aoa, out):
    """Every hot-path operator once, on one state (solver.py:154-421)."""
    gamma = 1.4
    out[f"{prefix}.prims"] = prims_arr(prims)
    out[f"{prefix}.dt"] = local_timestep(prims, conn, 0.2, gamma)
    q = primitives_to_q(prims, gamma)
    out[f"{prefix}.q"] = q
    fo = first_order_q_gradients(q, conn)
    out[f"{prefix}.qx0"] = fo.qx
    out[f"{prefix}.qy0"] = fo.qy
    for n_inner in (1, 3):
        g = compute_q_derivatives(q, conn, n_inner)
        out[f"{prefix}.qx{n_inner}"] = g.qx
        out[f"{prefix}.qy{n_inner}"] = g.qy
        out[f"{prefix}.inner_res{n_inner}"] = np.asarray(g.inner_residuals)
    g = compute_q_derivatives(q, conn, 3)
    flow = FlowState(prims=prims, q=q, qx=g.qx, qy=g.qy)
    R_int = flux_residual(flow, conn, "fused", gamma)
    out[f"{prefix}.R_int"] = R_int
    R_s4 = flux_residual(flow, conn, "split4", gamma)
    assert np.array_equal(R_int, R_s4)
    fs = free_stream(mach, aoa, gamma)
    R = apply_boundary(flow, R_int.copy(), conn, fs, gamma)
    out[f"{prefix}.R"] = R
    U = primitives_to_conserved(prims, gamma)
    out[f"{prefix}.U"] = U
    dt = out[f"{prefix}.dt"]
    U1 = state_update_rk(U, U, 1, dt, R)
    U3 = state_update_rk(U, U1, 3, dt, R)
    out[f"{prefix}.U1"] = U1
    out[f"{prefix}.U3"] = U3
    out[f"{prefix}.prims1"] = prims_arr(conserved_to_primitives(U1, gamma))
    out[f"{prefix}.residue1"] = np.array([residue_norm(U1, U)])


def save(name, arrays: dict, meta: dict):
    OUT.mkdir(parents=True, exist_ok=True)
    if arrays:
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
    meta = dict(meta)
    meta["generated_by"] = "tools/make_golden.py " + name
    meta["host"] = {
        "numpy": np.__version__,
        "cpus": os.cpu_count(),
        "note": "transcendentals (log/exp/erf) are host-ISA dependent at the ulp level",
    }
    (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(f"wrote {name}: {len(arrays)} arrays", flush=True)


def case_small():
    cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
    conn = build_stencils(cloud)
    meta = {"digests": conn_digests(cloud, conn), "params": [80, 30, 1.15, 20.0]}
    arrays = {}
    # initial states the solver would seed (solver.py:424-458)
    for tag, (mach, aoa) in {"m63a2": (0.63, 2.0), "m63a0": (0.63, 0.0), "m85a1": (0.85, 1.0)}.items():
        init = _initial_primitives(SolverConfig(mach=mach, aoa_deg=aoa), cloud)
        arrays[f"init.{tag}"] = prims_arr(init)
        meta["digests"][f"init.{tag}"] = digest(prims_arr(init))
    stage_ops("pert", cloud, conn, perturbed_state(cloud), 0.63, 2.0, arrays)
    init = _initial_primitives(SolverConfig(mach=0.63, aoa_deg=2.0), cloud)
    stage_ops("init", cloud, conn, init, 0.63, 2.0, arrays)
    # short solves: perturbed fused/split4 5 iterations (test_solver.py:214-221)
    for mode in ("fused", "split4"):
        cfg = SolverConfig(mach=0.63, aoa_deg=2.0, cfl=0.2, n_outer=5, mode=mode)
        res = solve(cfg, cloud, conn, initial_state=perturbed_state(cloud), instrument=False)
        arrays[f"solve_pert5.{mode}.history"] = res.residue_history
        arrays[f"solve_pert5.{mode}.prims"] = prims_arr(res.primitives)
        arrays[f"solve_pert5.{mode}.U"] = res.conserved
    # AoA 0 mirror run (test_solver.py:273-281)
    cfg = SolverConfig(mach=0.63, aoa_deg=0.0, cfl=0.2, n_outer=10)
    res = solve(cfg, cloud, conn, instrument=False)
    arrays["solve_a0_10.history"] = res.residue_history
    arrays["solve_a0_10.prims"] = prims_arr(res.primitives)
    # free stream fixed point (test_solver.py:155-159)
    cfg = SolverConfig(mach=0.63, aoa_deg=2.0, cfl=0.2, n_outer=5)
    init = free_stream(0.63, 2.0, 1.4, n=cloud.n_points)
    res = solve(cfg, cloud, conn, initial_state=init, instrument=False)
    arrays["solve_fs5.history"] = res.residue_history
    save("small", arrays, meta)


def case_hist2k():
    cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
    conn = build_stencils(cloud)
    arrays = {}
    meta = {"params": [80, 30, 1.15, 20.0]}
    for tag, (mach, aoa, iters) in {"m63a2": (0.63, 2.0, 1000), "m85a1": (0.85, 1.0, 300)}.items():
        cfg = SolverConfig(mach=mach, aoa_deg=aoa, cfl=0.2, n_outer=iters, threads=8)
        t0 = time.perf_counter()
        res = solve(cfg, cloud, conn, instrument=False)
        meta[f"{tag}.seconds"] = time.perf_counter() - t0
        arrays[f"{tag}.history"] = res.residue_history
        arrays[f"{tag}.prims"] = prims_arr(res.primitives)
        arrays[f"{tag}.U"] = res.conserved
    save("hist2k", arrays, meta)


def case_kinetics():
    rng = np.random.default_rng(2108)
    n = 256
    pr = Primitives(
        rng.uniform(0.2, 3.0, n), rng.uniform(-2.5, 2.5, n),
        rng.uniform(-2.5, 2.5, n), rng.uniform(0.2, 3.0, n),
    )
    # tidy states of reference tests/test_kinetics.py:311-319 appended
    extra = [(2.0, s, 0.3, 1.0) for s in (0.0, 0.5, -0.5, 2.0, -2.0, 8.0, -8.0)]
    extra += [(0.37, -0.81, 1.21, 2.6), (3.1, 0.05, -0.4, 0.09), (1.0, 0.0, 0.0, 1.0)]
    ex = np.array(extra).T
    pr = Primitives(*(np.concatenate([a, e]) for a, e in zip(prims_arr(pr), ex)))
    arrays = {"prims": prims_arr(pr)}
    for axis in ("x", "y"):
        arrays[f"full_{axis}"] = full_flux(pr, axis)
        for sign in ("+", "-"):
            arrays[f"split_{axis}{sign}"] = split_flux(pr, axis, sign)
    for g in (1.4, 5.0 / 3.0):
        arrays[f"q.g{g:.4f}"] = primitives_to_q(pr, g)
        arrays[f"U.g{g:.4f}"] = primitives_to_conserved(pr, g)
        back = q_to_primitives(arrays[f"q.g{g:.4f}"], g)
        arrays[f"q2p.g{g:.4f}"] = prims_arr(back)
        arrays[f"U2p.g{g:.4f}"] = prims_arr(conserved_to_primitives(arrays[f"U.g{g:.4f}"], g))
    save("kinetics", arrays, {"n": int(pr.n_points)})


def case_gammas():
    K = dict(np.load(OUT / "kinetics.npz"))
    pr = Primitives(*K["prims"])
    cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
    conn = build_stencils(cloud)
    arrays, meta = {}, {"gammas": [5.0 / 3.0, 1.3], "params": [80, 30, 1.15, 20.0]}
    for g in (5.0 / 3.0, 1.3):
        tag = f"g{g:.4f}"
        arrays[f"{tag}.q"] = primitives_to_q(pr, g)
        for axis in ("x", "y"):
            for sign in ("+", "-"):
                arrays[f"{tag}.split_{axis}{sign}"] = split_flux(pr, axis, sign, g)
        # one residual evaluation on the perturbed state of this gamma
        prims = perturbed_state(cloud, gamma=g)
        q = primitives_to_q(prims, g)
        grads = compute_q_derivatives(q, conn, 3)
        flow = FlowState(prims=prims, q=q, qx=grads.qx, qy=grads.qy)
        R_int = flux_residual(flow, conn, "fused", g)
        arrays[f"{tag}.prims"] = prims_arr(prims)
        arrays[f"{tag}.R_int"] = R_int
        arrays[f"{tag}.R"] = apply_boundary(flow, R_int.copy(), conn, free_stream(0.63, 2.0, g), g)
        cfg = SolverConfig(mach=0.63, aoa_deg=2.0, gamma=g, cfl=0.2, n_outer=20, threads=8)
        res = solve(cfg, cloud, conn, instrument=False)
        arrays[f"{tag}.history"] = res.residue_history
        arrays[f"{tag}.final"] = prims_arr(res.primitives)
    save("gammas", arrays, meta)


def lattice_cloud(n=5, h=1.0, classify_boundary=False):
    # restated from reference tests/conftest.py:7-28
    xs, ys = np.meshgrid(np.arange(n) * h, np.arange(n) * h, indexing="ij")
    x, y = xs.ravel(), ys.ravel()
    flag = np.full(x.size, INTERIOR, dtype=np.int64)
    nx = np.zeros(x.size)
    ny = np.zeros(x.size)
    if classify_boundary:
        lim = (n - 1) * h
        rim = (x == 0.0) | (y == 0.0) | (x == lim) | (y == lim)
        flag[rim] = OUTER
        nx[x == 0.0] -= 1.0
        nx[x == lim] += 1.0
        ny[y == 0.0] -= 1.0
        ny[y == lim] += 1.0
        norm = np.hypot(nx, ny)
        good = norm > 0
        nx[good] /= norm[good]
        ny[good] /= norm[good]
    return PointCloud(x, y, flag, nx, ny)


def channel_cloud(nx=9, ny=6, h=0.1):
    # restated from reference tests/test_solver.py:74-95
    gx, gy = np.meshgrid(np.arange(nx) * h, np.arange(ny) * h, indexing="ij")
    x, y = gx.ravel(), gy.ravel()
    flag = np.zeros(x.size, dtype=np.int64)
    nrm_x = np.zeros(x.size)
    nrm_y = np.zeros(x.size)
    bottom = y < 0.5 * h
    top = y > (ny - 1.5) * h
    left = x < 0.5 * h
    right = x > (nx - 1.5) * h
    flag[bottom] = WALL
    nrm_y[bottom] = 1.0
    for side, (sx, sy) in ((top, (0.0, 1.0)), (left, (-1.0, 0.0)), (right, (1.0, 0.0))):
        sel = side & ~bottom
        flag[sel] = OUTER
        nrm_x[sel], nrm_y[sel] = sx, sy
    corner = (left | right) & top
    nrm = np.hypot(np.where(left, -1.0, 1.0), 1.0)
    nrm_x[corner] = np.where(left, -1.0, 1.0)[corner] / nrm[corner]
    nrm_y[corner] = 1.0 / nrm[corner]
    return PointCloud(x, y, flag, nrm_x, nrm_y)


def case_lattice():
    meta = {"digests": {}}
    arrays = {}
    cases = {
        "lat5_k8": (lattice_cloud(5, 0.01, True), 8),
        "lat7_k15": (lattice_cloud(7, 1.0, True), None),
        "chan_k8": (channel_cloud(), 8),
    }
    for tag, (cloud, k) in cases.items():
        conn = build_stencils(cloud, k=k)
        meta["digests"][tag] = conn_digests(cloud, conn)
        arrays[f"{tag}.cloud"] = np.stack([cloud.x, cloud.y, cloud.flag.astype(float), cloud.nx, cloud.ny])
    # channel: tangent flow residual (test_solver.py:145-152)
    cloud, k = cases["chan_k8"]
    conn = build_stencils(cloud, k=8)
    n = cloud.n_points
    prims = Primitives(np.ones(n), np.full(n, 0.5), np.zeros(n), np.full(n, 1.0 / 1.4))
    q = primitives_to_q(prims, 1.4)
    g = compute_q_derivatives(q, conn, 3)
    flow = FlowState(prims=prims, q=q, qx=g.qx, qy=g.qy)
    R = apply_boundary(flow, flux_residual(flow, conn, "fused", 1.4), conn, free_stream(0.5, 0.0), 1.4)
    arrays["chan_k8.R_tangent"] = R
    save("lattice", arrays, meta)


def _big(name, params, mach, aoa, iters, store_final=True):
    m, L, g = params
    t0 = time.perf_counter()
    cloud = generate_naca_cloud(m, L, g, 20.0)
    conn = build_stencils(cloud)
    t_build = time.perf_counter() - t0
    meta = {"digests": conn_digests(cloud, conn), "params": [m, L, g, 20.0],
            "mach": mach, "aoa": aoa, "iters": iters, "build_seconds": t_build}
    cfg = SolverConfig(mach=mach, aoa_deg=aoa, cfl=0.2, n_outer=iters, threads=8)
    init = _initial_primitives(cfg, cloud)
    meta["digests"]["init"] = digest(prims_arr(init))
    print(f"{name}: n={cloud.n_points} built in {t_build:.1f}s", flush=True)
    t0 = time.perf_counter()
    try:
        res = solve(cfg, cloud, conn, instrument=False)
    except PositivityError as exc:
        # the reference itself breaks down (config 1 does at iteration 407):
        # record the failure, then the state just before it
        meta["failure"] = {"message": str(exc), "indices": [int(i) for i in exc.indices]}
        it = int(str(exc).split(":")[0].split()[1])
        meta["iters"] = it - 1
        cfg = SolverConfig(mach=mach, aoa_deg=aoa, cfl=0.2, n_outer=it - 1, threads=8)
        res = solve(cfg, cloud, conn, instrument=False)
    meta["solve_seconds"] = time.perf_counter() - t0
    arrays = {"history": res.residue_history}
    fin = prims_arr(res.primitives)
    meta["digests"]["final_prims"] = digest(fin)
    meta["final_prims_absmax"] = np.abs(fin).max(axis=1).tolist()
    if store_final:
        arrays["prims"] = fin
    else:
        # a deterministic 4096-point sample keeps the fixture small
        idx = np.linspace(0, cloud.n_points - 1, 4096).astype(np.int64)
        arrays["sample_idx"] = idx
        arrays["prims_sample"] = fin[:, idx]
    save(name, arrays, meta)


def _first_order_loop(cloud, conn, mach, aoa, iters):
    """The first-order scheme (qx = qy = 0; BASELINE config 1 "first-order",
    SURVEY.md 8(d)) composed from the reference's own stage operators in the
    order of its solve loop (solver.py:515-559): the reference solve() has no
    order switch, so this loop is the oracle for the device's order=1 mode."""
    cfg = SolverConfig(mach=mach, aoa_deg=aoa, cfl=0.2, n_outer=iters)
    gamma = cfg.gamma
    fs = free_stream(mach, aoa, gamma)
    prims = _initial_primitives(cfg, cloud)
    U = primitives_to_conserved(prims, gamma)
    zero = np.zeros((4, cloud.n_points))
    hist = []
    for _ in range(iters):
        dt = local_timestep(prims, conn, cfg.cfl, gamma)
        U_outer = U
        for stage in range(1, 5):
            q = primitives_to_q(prims, gamma)
            flow = FlowState(prims=prims, q=q, qx=zero, qy=zero)
            R = apply_boundary(flow, flux_residual(flow, conn, "fused", gamma), conn, fs, gamma)
            U = state_update_rk(U_outer, U, stage, dt, R)
            prims = conserved_to_primitives(U, gamma)
        hist.append(residue_norm(U, U_outer))
    return np.array(hist), prims_arr(prims)


def case_order1():
    cloud = generate_naca_cloud(80, 30, 1.15, 20.0)
    conn = build_stencils(cloud)
    arrays, meta = {}, {"params": [80, 30, 1.15, 20.0], "note": "first-order loop of reference operators"}
    for tag, (mach, aoa, iters) in {"m63a2": (0.63, 2.0, 200), "m85a1": (0.85, 1.0, 100)}.items():
        t0 = time.perf_counter()
        h, pr = _first_order_loop(cloud, conn, mach, aoa, iters)
        meta[f"{tag}.seconds"] = time.perf_counter() - t0
        meta[f"{tag}.iters"] = iters
        arrays[f"{tag}.history"] = h
        arrays[f"{tag}.prims"] = pr
    save("order1", arrays, meta)


def main(argv):
    cases = {
        "small": case_small,
        "hist2k": case_hist2k,
        "kinetics": case_kinetics,
        "gammas": case_gammas,
        "lattice": case_lattice,
        "order1": case_order1,
        "c40k": lambda: _big("c40k", (400, 100, 1.06), 0.63, 2.0, 1000),
        "c160k": lambda: _big("c160k", (800, 200, 1.03), 0.63, 2.0, 20, store_final=False),
        "c2p5m": lambda: _big("c2p5m", (3160, 790, 1.00734), 0.85, 1.0, 2, store_final=False),
    }
    for name in argv or ["small", "kinetics", "lattice"]:
        cases[name]()


if __name__ == "__main__":
    main(sys.argv[1:])
