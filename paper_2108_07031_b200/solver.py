"""Solver API on the B200 -- drop-in for reference ``kmf.solver``.

``solve`` keeps the reference signature (solver.py:477-485) and result type
(solver.py:115-124).  The whole outer loop runs on the device: per
iteration one CUDA graph replays

    4 x [ k_first_order -> n_inner x k_sweep -> (k_flux || k_boundary) -> k_update ]
    -> k_finalize

where k_update fuses state_update_rk, conserved_to_primitives, the next
stage's primitives_to_q and (stage 4) local_timestep plus the exact residue
sum, so ``timestep`` and ``q_variables`` time is reported inside
``state_update``.  The host touches the device once per ``solve`` (state in,
history + state out).

The individual stage operators (local_timestep, flux_residual,
apply_boundary, state_update_rk, residue_norm) are exposed with the
reference signatures for operator-level use and parity tests; each is one
synchronous device call.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
from scipy.spatial import cKDTree

from . import _lib
from ._device import device_for
from .geometry import Connectivity, PointCloud, build_stencils
from .state import (
    FlowState,
    PositivityError,
    Primitives,
    conserved_to_primitives,
    prims_array,
    free_stream,
)

MODES = ("fused", "split4")
RK_STAGES = 4
STAGE_NAMES = ("timestep", "q_variables", "q_derivatives", "flux_residual", "state_update", "residue")
BLOCK = 4096  # reference point block (solver.py:64); only fixes error-report order here


@dataclass
class SolverConfig:
    """Run parameters, validated on construction (solver.py:69-112)."""

    mach: float
    aoa_deg: float = 0.0
    gamma: float = 1.4
    cfl: float = 0.2
    n_outer: int = 1000
    n_inner: int = 3
    mode: str = "fused"
    threads: int = 1
    convergence_tol: float | None = None
    # extension: 1 = first-order scheme (qx = qy = 0, BASELINE config 1
    # "first-order"); the reference's solve() is second order
    order: int = 2

    def __post_init__(self):
        if not self.mach > 0.0:
            raise ValueError("mach must be positive")
        if not 1.0 < self.gamma < 2.0:
            raise ValueError("gamma must lie in (1, 2)")
        if not 0.0 < self.cfl <= 1.0:
            raise ValueError("cfl must lie in (0, 1]")
        if self.n_outer < 1:
            raise ValueError("n_outer must be at least 1")
        if self.n_inner < 1:
            raise ValueError("n_inner must be at least 1")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        if self.threads < 1:
            raise ValueError("threads must be at least 1")
        if self.convergence_tol is not None and not self.convergence_tol > 0.0:
            raise ValueError("convergence_tol must be positive")
        if self.order not in (1, 2):
            raise ValueError("order must be 1 or 2")

    def to_dict(self) -> dict:
        """The reference's keys (solver.py:101-112); `order` only when it is
        not the reference's own second-order scheme, so reports and config
        echoes stay readable by the reference's tools."""
        d = {k: getattr(self, k) for k in ("mach", "aoa_deg", "gamma", "cfl", "n_outer", "n_inner", "mode",
                                            "threads", "convergence_tol")}
        if self.order != 2:
            d["order"] = self.order
        return d


@dataclass
class SolveResult:
    primitives: Primitives
    conserved: np.ndarray
    residue_history: np.ndarray
    stage_seconds: dict
    wall_seconds: float
    timed_iterations: int
    iterations: int
    converged: bool


def config_order(config) -> int:
    """Scheme order of a config: this package's extension field, or 2 for
    the reference's own SolverConfig (which is always second order)."""
    return int(getattr(config, "order", 2))


def _params(config: SolverConfig, instrument: bool = False, timing_skip: int = 0) -> _lib.Params:
    fs = free_stream(config.mach, config.aoa_deg, config.gamma)
    p = _lib.Params()
    p.gamma = config.gamma
    p.cfl = config.cfl
    for i, v in enumerate((fs.rho[0], fs.u1[0], fs.u2[0], fs.p[0])):
        p.fs[i] = float(v)
    # the reference's SolverConfig has no `order` (solver.py:69-112): second order
    p.n_inner = config.n_inner if config_order(config) == 2 else 0  # 0: first-order scheme on the device
    p.mode = MODES.index(config.mode)
    p.convergence_tol = config.convergence_tol if config.convergence_tol is not None else 0.0
    p.instrument = int(instrument)
    p.timing_skip = int(timing_skip)
    return p


# ------------------------------------------------------------ stage operators


def local_timestep(prims: Primitives, conn: Connectivity, cfl: float, gamma: float = 1.4) -> np.ndarray:
    """cfl * d_min / (|u| + a) per point on the device (solver.py:154-159), bitwise."""
    if not 0.0 < cfl <= 1.0:
        raise ValueError("cfl must lie in (0, 1]")
    dev = device_for(conn)
    pa = prims_array(prims)
    dt = np.empty(pa.shape[1])
    _lib.check(_lib.lib().kmf_op_timestep(dev.handle, _lib.dptr(pa), cfl, gamma, _lib.dptr(dt)), "local_timestep")
    return dt


def flux_residual(state: FlowState, conn: Connectivity, mode: str = "fused", gamma: float = 1.4,
                  blocks=None) -> np.ndarray:
    """Interior residual R (4, n) with boundary rows zero (solver.py:198-235).

    ``fused``: one kernel, all four split families per stencil pass;
    ``split4``: four kernels, one family each.  Bitwise equal.
    """
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    dev = device_for(conn)
    q, qx, qy = _lib.f64(state.q), _lib.f64(state.qx), _lib.f64(state.qy)
    R = np.empty_like(q)
    rc = _lib.lib().kmf_op_flux_residual(dev.handle, _lib.dptr(q), _lib.dptr(qx), _lib.dptr(qy), MODES.index(mode),
                                         gamma, _lib.dptr(R))
    if rc == _lib.KMF_EPOSITIVITY:
        dev.raise_positivity(_lib.CTX_FLUX_XP, 0, which=0, mode=MODES.index(mode), gamma=gamma)
    _lib.check(rc, "flux_residual")
    return R


def apply_boundary(state: FlowState, residual: np.ndarray, conn: Connectivity, free_stream_prims: Primitives,
                   gamma: float = 1.4) -> np.ndarray:
    """Wall / outer frame closures into ``residual`` in place (solver.py:336-373)."""
    dev = device_for(conn)
    q, qx, qy = _lib.f64(state.q), _lib.f64(state.qx), _lib.f64(state.qy)
    R = _lib.f64(residual).copy()
    fs = np.array([float(free_stream_prims.rho[0]), float(free_stream_prims.u1[0]),
                   float(free_stream_prims.u2[0]), float(free_stream_prims.p[0])])
    rc = _lib.lib().kmf_op_boundary(dev.handle, _lib.dptr(q), _lib.dptr(qx), _lib.dptr(qy), _lib.dptr(fs), gamma,
                                    _lib.dptr(R))
    if rc == _lib.KMF_EPOSITIVITY:
        dev.raise_positivity(_lib.CTX_WALL_TANGENT, 0, which=0, mode=0, gamma=gamma)
    _lib.check(rc, "apply_boundary")
    residual[...] = R
    return residual


def state_update_rk(U_outer: np.ndarray, U_stage: np.ndarray, stage: int, dt: np.ndarray, residual: np.ndarray,
                    gamma: float | None = None) -> np.ndarray:
    """One SSP(4,3) stage on the device (solver.py:385-409), bitwise."""
    if stage not in (1, 2, 3, 4):
        raise ValueError("stage must be 1..4")
    Us = _lib.f64(U_stage)
    shape = Us.shape
    n = shape[-1]
    Uo = np.broadcast_to(np.asarray(U_outer, dtype=np.float64), shape)
    R = np.broadcast_to(np.asarray(residual, dtype=np.float64), shape)
    d = np.broadcast_to(np.asarray(dt, dtype=np.float64), shape)
    if Us.ndim == 2 and shape[0] == 4:
        a, b, r, dd, m = _lib.f64(Uo), Us, _lib.f64(R), _lib.f64(d[0]), n
    else:
        # any other shape: the same elementwise kernel on one flattened row
        # (padded to the (4, m) layout with zero rows)
        m = Us.size
        z = np.zeros((3, m))
        a, b, r = (np.ascontiguousarray(np.vstack([np.ravel(x), z])) for x in (Uo, Us, R))
        dd = _lib.f64(np.ravel(d))
    out = np.empty((4, m))
    _lib.require_device()
    _lib.check(_lib.lib().kmf_op_state_update(m, _lib.dptr(a), _lib.dptr(b), stage, _lib.dptr(dd), _lib.dptr(r),
                                              _lib.dptr(out)), "state_update_rk")
    out = out if (Us.ndim == 2 and shape[0] == 4) else out[0].reshape(shape)
    if gamma is not None:
        conserved_to_primitives(out, gamma)
    return out


def residue_norm(U_new: np.ndarray, U_old: np.ndarray) -> float:
    """sqrt(sum(drho^2)/n) with an exact device sum (solver.py:412-421):
    bitwise equal to math.fsum, independent of point order."""
    a = np.ascontiguousarray(np.atleast_1d(np.asarray(U_new, dtype=np.float64)[0]))
    b = np.ascontiguousarray(np.atleast_1d(np.asarray(U_old, dtype=np.float64)[0]))
    out = np.zeros(1)
    _lib.require_device()
    _lib.check(_lib.lib().kmf_op_residue(a.shape[0], _lib.dptr(a), _lib.dptr(b), _lib.dptr(out)), "residue_norm")
    return float(out[0])


# ----------------------------------------------------------------- set-up


def initial_primitives(config: SolverConfig, cloud: PointCloud) -> Primitives:
    """Free stream with the windward wall-normal velocity removed near the
    wall under a Gaussian weight (solver.py:424-458).  Host set-up."""
    prims = free_stream(config.mach, config.aoa_deg, config.gamma, n=cloud.n_points)
    w = cloud.wall
    if w.size == 0:
        return prims
    wall_pts = np.column_stack([cloud.x[w], cloud.y[w]])
    tree = cKDTree(wall_pts)
    dist, near = tree.query(np.column_stack([cloud.x, cloud.y]), workers=-1)  # workers: same result, parallel
    if w.size > 1:
        sigma = 8.0 * float(np.mean(tree.query(wall_pts, k=2)[0][:, 1]))
    else:
        sigma = 8.0 * float(np.min(dist[dist > 0.0])) if (dist > 0.0).any() else 1.0
    nx, ny = cloud.nx[w][near], cloud.ny[w][near]
    weight = np.exp(-((dist / sigma) ** 2))
    speed = max(float(prims.speed[0]), 1e-300)
    weight = weight * np.clip(-(prims.u1 * nx + prims.u2 * ny) / speed, 0.0, 1.0)
    un = prims.u1 * nx + prims.u2 * ny
    prims.u1 -= weight * un * nx
    prims.u2 -= weight * un * ny
    return prims


_initial_primitives = initial_primitives  # reference-private name, kept for drop-in callers


# ------------------------------------------------------------------ solve


def solve(
    config: SolverConfig,
    cloud: PointCloud,
    conn: Connectivity | None = None,
    initial_state: Primitives | None = None,
    instrument: bool = True,
    timing_skip: int = 0,
    clock=time.perf_counter,
    devices=None,
) -> SolveResult:
    """Run ``config.n_outer`` outer iterations on the GPU (solver.py:477-573).

    Raises PositivityError (prefixed "iteration {it}: ") exactly where the
    reference would.  With ``instrument`` the iterations after
    ``timing_skip`` are timed per stage with CUDA events and by ``clock``.

    ``devices`` (extension; default: one GPU) -- a list of CUDA devices: the
    cloud is partitioned into angular sectors, one per entry, and the ranks
    run concurrently from this process over the peer transport
    (dist.solve_group); history and state are bitwise the one-GPU solve's.
    Per-stage seconds are not collected on that path (zeros); the wall time
    covers the whole run.
    """
    if conn is None:
        conn = build_stencils(cloud)
    prims = initial_state.copy() if initial_state is not None else initial_primitives(config, cloud)
    prims.validate("initial state")
    if devices is not None and len(devices) > 1:
        from .dist import solve_group

        t0 = clock()
        hist, p_out, U, conv = solve_group(config, cloud, conn, len(devices), initial_state=prims,
                                           devices=[int(d) for d in devices], scheme="sectors", transport="peer")
        wall = clock() - t0
        return SolveResult(
            primitives=Primitives.from_array(p_out),
            conserved=U,
            residue_history=np.asarray(hist),
            stage_seconds={name: 0.0 for name in STAGE_NAMES},
            wall_seconds=wall if instrument else 0.0,
            timed_iterations=len(hist),
            iterations=len(hist),
            converged=conv,
        )
    dev = device_for(conn)
    dev.set_state(prims_array(prims))

    n_outer = config.n_outer
    skip = min(max(timing_skip, 0), n_outer) if instrument else n_outer
    history = []
    converged = False
    wall = 0.0
    stage = np.zeros(6)
    done = 0

    def chunk(count, timed):
        nonlocal done, converged
        p = _params(config, instrument=timed, timing_skip=0)
        try:
            h, k, conv = dev.run(p, count)
        except PositivityError as exc:
            msg = str(exc)
            if done and msg.startswith("iteration "):
                head, _, rest = msg.partition(": ")
                msg = f"iteration {int(head.split()[1]) + done}: {rest}"
            raise PositivityError(msg, indices=exc.indices) from None
        history.extend(h.tolist())
        done += k
        converged = conv
        return conv

    stop = False
    if skip > 0:
        stop = chunk(skip, False)
    if not stop and done < n_outer:
        dev.prepare(_params(config, instrument=True, timing_skip=0))  # graph capture stays out of the clock
        t0 = clock()
        chunk(n_outer - done, True)
        wall = clock() - t0
        stage = dev.stage_seconds()
    p_out, U = dev.get_state()
    timing = {name: (float(stage[i]) if instrument else 0.0) for i, name in enumerate(STAGE_NAMES)}
    return SolveResult(
        primitives=Primitives.from_array(p_out),
        conserved=U,
        residue_history=np.asarray(history),
        stage_seconds=timing,
        wall_seconds=wall if instrument else 0.0,
        timed_iterations=max(done - timing_skip, 0),
        iterations=done,
        converged=converged,
    )


def solve_cases(
    configs,
    cloud: PointCloud,
    conn: Connectivity | None = None,
    initial_states=None,
) -> list:
    """Independent solves on one cloud, streamed through one device context.

    ``configs`` is a SolverConfig or one per case; ``initial_states`` a list of
    Primitives (default: ``initial_primitives`` of each config).  Case k gives
    ``solve(configs[k], cloud, conn, initial_states[k], instrument=False)``
    bit for bit in residue history, final primitives, final conserved state
    and convergence -- but
    case k+1's upload and case k-1's download overlap case k's iterations
    (kmf_run_cases), the batch the reference's harness runs one solve at a
    time (bench.py:174-215 ``sweep``).  A case that fails positivity is
    returned as its PositivityError instead of a SolveResult (the batch
    keeps going, as the reference's sweep records failed cells).
    """
    if conn is None:
        conn = build_stencils(cloud)
    if initial_states is None:
        cfgs = list(configs) if isinstance(configs, (list, tuple)) else [configs]
        initial_states = [initial_primitives(c, cloud) for c in cfgs]
    m = len(initial_states)
    cfgs = list(configs) if isinstance(configs, (list, tuple)) else [configs] * m
    if len(cfgs) != m:
        raise ValueError("one config per initial state")
    n_iter = cfgs[0].n_outer
    if any(c.n_outer != n_iter for c in cfgs):
        raise ValueError("every case runs the same n_outer")
    states = []
    for prims in initial_states:
        prims.validate("initial state")
        states.append(prims_array(prims))
    dev = device_for(conn)
    outs, hist, done, conv, status, Us = dev.run_cases([_params(c) for c in cfgs], states, n_iter, conserved=True)
    results = []
    for k in range(m):
        if status[k] == _lib.KMF_EPOSITIVITY:
            # replay the failing case alone for the reference's exact error
            try:
                solve(cfgs[k], cloud, conn, initial_states[k], instrument=False)
            except PositivityError as exc:
                results.append(exc)
                continue
            raise _lib.DeviceError(f"case {k}: positivity failure did not reproduce")
        prims = Primitives.from_array(outs[k])
        results.append(SolveResult(
            primitives=prims,
            conserved=Us[k],
            residue_history=hist[k, : done[k]].copy(),
            stage_seconds={name: 0.0 for name in STAGE_NAMES},
            wall_seconds=0.0,
            timed_iterations=done[k],
            iterations=done[k],
            converged=conv[k],
        ))
    return results
