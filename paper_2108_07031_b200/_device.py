"""Device context: packs a Connectivity into the C ABI and owns the kmf_ctx.

One context per Connectivity object (cached), bound to one GPU.  Also turns
device positivity flags back into the reference's PositivityError (message,
context and indices of solver.py:164-170, :260-265, state.py:110-128).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np

from . import _lib, reorder
from .geometry import SPLIT_KINDS, Connectivity
from .state import PositivityError, raise_decode_flags

BLOCK = 4096  # the reference's fixed point block (solver.py:64): fixes raise order


def _stencil_struct(s, keep) -> _lib.Stencil:
    arrs = {
        "ptr": _lib.i64(s.ptr), "idx": _lib.i64(s.idx),
        "dx": _lib.f64(s.dx), "dy": _lib.f64(s.dy),
        "sxx": _lib.f64(s.sxx), "sxy": _lib.f64(s.sxy), "syy": _lib.f64(s.syy), "det": _lib.f64(s.det),
    }
    keep.extend(arrs.values())
    st = _lib.Stencil()
    st.n_owners = arrs["ptr"].shape[0] - 1
    st.n_edges = arrs["idx"].shape[0]
    st.ptr, st.idx = _lib.i64ptr(arrs["ptr"]), _lib.i64ptr(arrs["idx"])
    for name in ("dx", "dy", "sxx", "sxy", "syy", "det"):
        setattr(st, name, _lib.dptr(arrs[name]))
    return st


def _frame_struct(fr, keep) -> _lib.Frame:
    out = _lib.Frame()
    pts = _lib.i64(fr.points)
    vec = {k: _lib.f64(getattr(fr, k)) for k in ("tx", "ty", "nx", "ny")}
    keep.append(pts)
    keep.extend(vec.values())
    out.b = pts.shape[0]
    out.points = _lib.i64ptr(pts)
    for k, v in vec.items():
        setattr(out, k, _lib.dptr(v))
    out.tplus = _stencil_struct(fr.tplus, keep)
    out.tminus = _stencil_struct(fr.tminus, keep)
    out.normal = _stencil_struct(fr.normal, keep)
    return out


def _check_split_layout(conn: Connectivity):
    """The device derives split membership from the signs of full.dx/dy
    (geometry.py:544-549); refuse connectivities built differently."""
    from .builder import SplitView

    if all(isinstance(conn.split[k], SplitView) for k in SPLIT_KINDS):
        return  # derived from the full stencil's signs by construction (builder.py)
    f = conn.full
    masks = {"x+": f.dx <= 0.0, "x-": f.dx >= 0.0, "y+": f.dy <= 0.0, "y-": f.dy >= 0.0}
    for kind, m in masks.items():
        s = conn.split[kind]
        if s.idx.shape[0] != int(m.sum()) or not np.array_equal(s.idx, f.idx[m]):
            raise ValueError(f"split stencil {kind} is not the sign subset of the full stencil")


def pack(conn: Connectivity, perm=None):
    """Geometry struct + the arrays it points into (keep them alive)."""
    _check_split_layout(conn)
    keep = []
    cl = conn.cloud
    g = _lib.Geometry()
    x, y, fl, dmin = _lib.f64(cl.x), _lib.f64(cl.y), _lib.i64(cl.flag), _lib.f64(conn.d_min)
    keep += [x, y, fl, dmin]
    g.n = x.shape[0]
    g.x, g.y, g.flag, g.d_min = _lib.dptr(x), _lib.dptr(y), _lib.i64ptr(fl), _lib.dptr(dmin)
    g.full = _stencil_struct(conn.full, keep)
    for f, kind in enumerate(SPLIT_KINDS):
        s = conn.split[kind]
        for attr, arr in (("split_sxx", s.sxx), ("split_sxy", s.sxy), ("split_syy", s.syy),
                          ("det_safe", conn.det_safe[kind])):
            a = _lib.f64(arr)
            keep.append(a)
            getattr(g, attr)[f] = _lib.dptr(a)
    g.has_wall = int(conn.wall_frame is not None)
    g.has_outer = int(conn.outer_frame is not None)
    if conn.wall_frame is not None:
        g.wall = _frame_struct(conn.wall_frame, keep)
    if conn.outer_frame is not None:
        g.outer = _frame_struct(conn.outer_frame, keep)
    if perm is not None:
        p = _lib.i64(perm)
        keep.append(p)
        g.perm = _lib.i64ptr(p)
    return g, keep


class DeviceConnectivity:
    """A kmf_ctx holding one Connectivity on one GPU."""

    def __init__(self, conn: Connectivity, device: int | None = None, perm=None):
        _lib.require_device()
        self.conn = conn
        self.n = conn.cloud.n_points
        self.n_edges = int(conn.full.idx.shape[0])
        g, keep = pack(conn, perm)
        h = C.c_void_p()
        _lib.check(_lib.lib().kmf_create(C.byref(h), C.byref(g), _lib.device_index() if device is None else device),
                   "kmf_create")
        self._h = h
        self._fin = weakref.finalize(self, _lib.lib().kmf_destroy, h)

    @property
    def handle(self):
        return self._h

    def close(self):
        self._fin()

    # ---------------------------------------------------------------- loop
    def set_state(self, prims4n: np.ndarray):
        a = _lib.f64(prims4n)
        _lib.check(_lib.lib().kmf_set_state(self._h, _lib.dptr(a)), "kmf_set_state")

    def run(self, params: _lib.Params, n_iter: int):
        hist = np.zeros(max(n_iter, 1))
        done = C.c_int(0)
        conv = C.c_int(0)
        rc = _lib.lib().kmf_run(self._h, C.byref(params), n_iter, _lib.dptr(hist), C.byref(done), C.byref(conv))
        if rc == _lib.KMF_EPOSITIVITY:
            info = _lib.ErrorInfo()
            _lib.lib().kmf_last_error(self._h, C.byref(info))
            self.raise_positivity(info.context, info.stage, which=_lib.DIAG_LAST_RUN, mode=params.mode,
                                  prefix=f"iteration {info.iteration}: ", gamma=params.gamma)
        _lib.check(rc, "kmf_run")
        return hist[: done.value].copy(), done.value, bool(conv.value)

    def run_cases(self, params, states, n_iter: int, outs=None, conserved: bool = False):
        """kmf_run_cases: one (params, initial (4, n) state) per case, uploads and
        downloads overlapped with the iterations (pinned buffers overlap; any
        array works).  Returns (finals, history (n_cases, n_iter), iters_done,
        converged, status[, conserved finals]) -- status KMF_OK /
        KMF_EPOSITIVITY per case; the conserved finals with conserved=True."""
        m = len(states)
        if len(params) != m or m < 1:
            raise ValueError("one Params per case and at least one case")
        ins = [_lib.f64(a) for a in states]
        for a in ins:
            if a.shape != (4, self.n):
                raise ValueError(f"initial state must be (4, {self.n})")
        if outs is None:
            outs = [np.empty((4, self.n)) for _ in range(m)]
        parr = (_lib.Params * m)(*params)
        pin = (C.c_void_p * m)(*[a.ctypes.data for a in ins])
        pout = (C.c_void_p * m)(*[a.ctypes.data for a in outs])
        Us = [np.empty((4, self.n)) for _ in range(m)] if conserved else None
        pU = (C.c_void_p * m)(*[a.ctypes.data for a in Us]) if conserved else None
        hist = np.zeros((m, n_iter))
        done = (C.c_int * m)()
        conv = (C.c_int * m)()
        st = (C.c_int * m)()
        rc = _lib.lib().kmf_run_cases(self._h, parr, n_iter, m, pin, pout, pU, _lib.dptr(hist), done, conv, st)
        if rc != _lib.KMF_EPOSITIVITY:
            _lib.check(rc, "kmf_run_cases")
        res = (outs, hist, list(done), [bool(v) for v in conv], list(st))
        return res + (Us,) if conserved else res

    def prepare(self, params: _lib.Params):
        """Capture the iteration graphs a run with `params` replays (not timed)."""
        _lib.check(_lib.lib().kmf_prepare(self._h, C.byref(params)), "kmf_prepare")

    def get_state(self):
        prims = np.empty((4, self.n))
        U = np.empty((4, self.n))
        _lib.check(_lib.lib().kmf_get_state(self._h, _lib.dptr(prims), _lib.dptr(U)), "kmf_get_state")
        return prims, U

    def stage_seconds(self) -> np.ndarray:
        out = np.zeros(6)
        _lib.check(_lib.lib().kmf_stage_seconds(self._h, _lib.dptr(out)), "kmf_stage_seconds")
        return out

    # ---------------------------------------------------------------- errors
    def raise_positivity(self, context: int, stage: int, which: int, mode: int, prefix: str = "",
                         gamma: float = 1.4):
        L = _lib.lib()
        if context in (_lib.CTX_FLUX_XP, _lib.CTX_FLUX_XM, _lib.CTX_FLUX_YP, _lib.CTX_FLUX_YM):
            flags = np.empty(self.n_edges, dtype=np.uint8)
            _lib.check(L.kmf_diag_flux(self._h, which, _lib.u8ptr(flags)), "kmf_diag_flux")
            self._raise_flux(flags, mode, prefix)
        if context in (_lib.CTX_WALL_TANGENT, _lib.CTX_WALL_NORMAL, _lib.CTX_OUTER_TANGENT, _lib.CTX_OUTER_NORMAL):
            self._raise_frame(which, prefix)
        if context in (_lib.CTX_C2P_DENSITY, _lib.CTX_C2P_PRESSURE):
            raise_decode_flags(self.stage_decode_flags(stage, gamma), prefix)
        raise PositivityError(f"{prefix}positivity failure (context {context})")

    def stage_decode_flags(self, stage: int, gamma: float, n_valid: int | None = None) -> np.ndarray:
        """state.py:110-128 flags (bit0 rho, bit1 p) of the state the failing
        update wrote, over the first ``n_valid`` slots (the owned points of a
        partition: halo slots are not updated and carry stale values)."""
        L = _lib.lib()
        U = np.empty((4, self.n))
        _lib.check(L.kmf_diag_stage_state(self._h, stage, _lib.dptr(U)), "kmf_diag_stage_state")
        fl = np.empty(self.n, dtype=np.uint8)
        out = np.empty((4, self.n))
        _lib.check(L.kmf_op_conserved_to_primitives(self.n, _lib.dptr(U), gamma, _lib.dptr(out), _lib.u8ptr(fl)),
                   "conserved_to_primitives")
        return fl if n_valid is None else fl[:n_valid]

    def _raise_flux(self, flags: np.ndarray, mode: int, prefix: str):
        """Reproduce the reference raise order: fused walks 4096-point
        blocks then kinds, split4 kinds then blocks (solver.py:218-229);
        indices are positions in that block's family edge list."""
        f = self.conn.full
        owner = np.repeat(np.arange(self.n), np.diff(f.ptr))
        fam_masks = (f.dx <= 0.0, f.dx >= 0.0, f.dy <= 0.0, f.dy >= 0.0)
        nblocks = (self.n + BLOCK - 1) // BLOCK
        per = []
        for m in fam_masks:
            edges = np.flatnonzero(m)
            blk = owner[edges] // BLOCK
            start = np.searchsorted(blk, np.arange(nblocks))
            per.append((edges, blk, start))
        order = ([(b, k) for b in range(nblocks) for k in range(4)] if mode == 0
                 else [(b, k) for k in range(4) for b in range(nblocks)])
        for b, k in order:
            edges, blk, start = per[k]
            lo = start[b]
            hi = start[b + 1] if b + 1 < nblocks else edges.shape[0]
            fl = flags[edges[lo:hi]]
            bad = np.flatnonzero(fl & 1)
            if bad.size:
                raise PositivityError(
                    f"{prefix}flux_residual[{SPLIT_KINDS[k]}]: perturbed entropy vector left the physical "
                    f"region on {bad.size} edge(s)",
                    indices=bad,
                )
            for bit in (2, 4):
                nan = np.flatnonzero(fl & bit)
                if nan.size:
                    raise PositivityError(
                        f"{prefix}q_to_primitives: q4 >= 0 at {nan.size} point(s), first index {nan[0]}",
                        indices=nan,
                    )

    def _raise_frame(self, which: int, prefix: str):
        L = _lib.lib()
        frames = [(fr, lbl) for fr, lbl in ((self.conn.wall_frame, "wall"), (self.conn.outer_frame, "outer"))
                  if fr is not None]
        fam_flags = []
        for fam in range(3):
            total = sum(int(getattr(fr, ("tplus", "tminus", "normal")[fam]).idx.shape[0]) for fr, _ in frames)
            fl = np.zeros(max(total, 1), dtype=np.uint8)
            _lib.check(L.kmf_diag_frame(self._h, which, fam, _lib.u8ptr(fl)), "kmf_diag_frame")
            fam_flags.append(fl)
        offs = [0, 0, 0]
        for fr, lbl in frames:
            for fam, name in enumerate(("tplus", "tminus", "normal")):
                s = getattr(fr, name)
                ne = int(s.idx.shape[0])
                fl = fam_flags[fam][offs[fam]:offs[fam] + ne]
                offs[fam] += ne
                bad = np.flatnonzero(fl)
                if bad.size:
                    own = np.repeat(fr.points, np.diff(s.ptr))
                    ctx = f"{lbl} {'normal' if fam == 2 else 'tangent'}"
                    raise PositivityError(f"{prefix}{ctx}: perturbed entropy vector left the physical region",
                                          indices=own[bad])


_cache: dict = {}
_cache_lock = threading.Lock()
_order = os.environ.get("KMF_ORDER", "natural")


def set_point_order(order: str) -> None:
    """Device slot order for contexts created from now on: "natural" (the
    caller's numbering) or "hilbert" (reorder.py).  Results are bitwise
    identical either way; only memory locality changes."""
    global _order
    if order not in reorder.ORDERS:
        raise ValueError(f"order must be one of {reorder.ORDERS}")
    _order = order


def point_order() -> str:
    return _order


def device_for(conn: Connectivity, order: str | None = None) -> DeviceConnectivity:
    """Cached device context for this Connectivity object in the given (or
    current default) point order."""
    order = order or _order
    key = (id(conn), order)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None:
            ref, dev = hit
            if ref() is conn:
                return dev
        dev = DeviceConnectivity(conn, perm=reorder.permutation(conn.cloud, order))
        _cache[key] = (weakref.ref(conn), dev)
        weakref.finalize(conn, _cache.pop, key, None)
        return dev
