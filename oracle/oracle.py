"""ctypes wrapper of the CPU oracle (oracle/kmf_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs as the checker and the
CPU baseline.  The product (paper_2108_07031_b200) never imports it.

Functions take and return numpy arrays in the reference layout and accept
any Connectivity-shaped object (the reference's or ours).
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libkmf_oracle.so"

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class OStencil(C.Structure):
    _fields_ = [("n_owners", C.c_int64), ("n_edges", C.c_int64), ("ptr", _i64p), ("idx", _i64p),
                ("dx", _dp), ("dy", _dp), ("sxx", _dp), ("sxy", _dp), ("syy", _dp), ("det", _dp)]


class OFrame(C.Structure):
    _fields_ = [("b", C.c_int64), ("points", _i64p), ("tx", _dp), ("ty", _dp), ("nx", _dp), ("ny", _dp),
                ("tplus", OStencil), ("tminus", OStencil), ("normal", OStencil)]


class OConn(C.Structure):
    _fields_ = [("n", C.c_int64), ("flag", _i64p), ("d_min", _dp), ("full", OStencil), ("split", OStencil * 4),
                ("det_safe", _dp * 4), ("has_wall", C.c_int), ("has_outer", C.c_int),
                ("wall", OFrame), ("outer", OFrame), ("n_act", C.c_int64)]


class OError(C.Structure):
    _fields_ = [("code", C.c_int), ("iteration", C.c_int), ("stage", C.c_int), ("context", C.c_int),
                ("count", C.c_int64), ("first", C.c_int64)]


class OParams(C.Structure):
    _fields_ = [("fs", C.c_double * 4), ("gamma", C.c_double), ("cfl", C.c_double), ("n_outer", C.c_int),
                ("n_inner", C.c_int), ("mode", C.c_int), ("convergence_tol", C.c_double)]


CONTEXTS = {
    1: "initial state", 2: "flux_residual[x+]", 3: "flux_residual[x-]", 4: "flux_residual[y+]",
    5: "flux_residual[y-]", 6: "wall tangent", 7: "wall normal", 8: "outer tangent", 9: "outer normal",
    10: "conserved_to_primitives density", 11: "conserved_to_primitives pressure", 12: "q_to_primitives",
    13: "primitives_to_q",
}


class OracleError(ValueError):
    def __init__(self, err: OError):
        self.context = CONTEXTS.get(err.context, str(err.context))
        self.iteration, self.stage, self.count, self.first = err.iteration, err.stage, err.count, err.first
        super().__init__(f"oracle positivity: iteration {err.iteration} stage {err.stage} {self.context} "
                         f"count {err.count} first {err.first}")


_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        vp = C.c_void_p
        P = C.POINTER
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        for name in ("orc_primitives_to_q", "orc_q_to_primitives", "orc_primitives_to_conserved",
                     "orc_conserved_to_primitives"):
            getattr(L, name).argtypes = [C.c_int64, _dp, C.c_double, _dp, P(OError)]
            getattr(L, name).restype = C.c_int
        L.orc_split_flux.argtypes = [C.c_int64, _dp, C.c_int, C.c_int, C.c_double, _dp]
        L.orc_full_flux.argtypes = [C.c_int64, _dp, C.c_int, C.c_double, _dp]
        L.orc_local_timestep.argtypes = [P(OConn), _dp, C.c_double, C.c_double, _dp]
        L.orc_first_order_q_gradients.argtypes = [P(OConn), _dp, _dp, _dp]
        L.orc_compute_q_derivatives.argtypes = [P(OConn), _dp, C.c_int, _dp, _dp, _dp]
        L.orc_flux_residual.argtypes = [P(OConn), _dp, _dp, _dp, C.c_int, C.c_double, _dp, P(OError)]
        L.orc_flux_residual.restype = C.c_int
        L.orc_apply_boundary.argtypes = [P(OConn), _dp, _dp, _dp, _dp, C.c_double, _dp, P(OError)]
        L.orc_apply_boundary.restype = C.c_int
        L.orc_state_update_rk.argtypes = [C.c_int64, _dp, _dp, C.c_int, _dp, _dp, _dp]
        L.orc_residue_norm.argtypes = [C.c_int64, _dp, _dp]
        L.orc_residue_norm.restype = C.c_double
        L.orc_fsum.argtypes = [C.c_int64, _dp]
        L.orc_fsum.restype = C.c_double
        L.orc_solve.argtypes = [P(OConn), P(OParams), _dp, _dp, _dp, P(C.c_int), P(C.c_int), P(OError)]
        L.orc_solve.restype = C.c_int
        del vp
        _lib = L
    return _lib


def set_threads(n: int):
    lib().orc_set_threads(int(n))


def _f(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _d(a):
    return a.ctypes.data_as(_dp)


class Packed:
    """orc_conn built from any Connectivity-shaped object; keeps arrays alive."""

    def __init__(self, conn):
        self.keep = []
        c = OConn()
        cl = conn.cloud
        c.n = cl.n_points
        fl = self._i(cl.flag)
        c.flag = fl.ctypes.data_as(_i64p)
        c.d_min = _d(self._f(conn.d_min))
        c.full = self._st(conn.full)
        for k, kind in enumerate(("x+", "x-", "y+", "y-")):
            c.split[k] = self._st(conn.split[kind])
            c.det_safe[k] = _d(self._f(conn.det_safe[kind]))
        c.has_wall = int(conn.wall_frame is not None)
        c.has_outer = int(conn.outer_frame is not None)
        if conn.wall_frame is not None:
            c.wall = self._fr(conn.wall_frame)
        if conn.outer_frame is not None:
            c.outer = self._fr(conn.outer_frame)
        self.c = c
        self.n = int(cl.n_points)

    def _f(self, a):
        a = _f(a)
        self.keep.append(a)
        return a

    def _i(self, a):
        a = _i(a)
        self.keep.append(a)
        return a

    def _st(self, s):
        o = OStencil()
        p, ix = self._i(s.ptr), self._i(s.idx)
        o.n_owners, o.n_edges = p.shape[0] - 1, ix.shape[0]
        o.ptr, o.idx = p.ctypes.data_as(_i64p), ix.ctypes.data_as(_i64p)
        for name in ("dx", "dy", "sxx", "sxy", "syy", "det"):
            setattr(o, name, _d(self._f(getattr(s, name))))
        return o

    def _fr(self, fr):
        o = OFrame()
        pts = self._i(fr.points)
        o.b, o.points = pts.shape[0], pts.ctypes.data_as(_i64p)
        for name in ("tx", "ty", "nx", "ny"):
            setattr(o, name, _d(self._f(getattr(fr, name))))
        o.tplus, o.tminus, o.normal = self._st(fr.tplus), self._st(fr.tminus), self._st(fr.normal)
        return o

    @property
    def ref(self):
        return C.byref(self.c)


def _raise(rc, err):
    if rc:
        raise OracleError(err)


def primitives_to_q(prims4n, gamma=1.4):
    p = _f(prims4n)
    q = np.empty_like(p)
    e = OError()
    _raise(lib().orc_primitives_to_q(p.shape[1], _d(p), gamma, _d(q), C.byref(e)), e)
    return q


def q_to_primitives(q4n, gamma=1.4):
    q = _f(q4n)
    p = np.empty_like(q)
    e = OError()
    _raise(lib().orc_q_to_primitives(q.shape[1], _d(q), gamma, _d(p), C.byref(e)), e)
    return p


def primitives_to_conserved(prims4n, gamma=1.4):
    p = _f(prims4n)
    U = np.empty_like(p)
    e = OError()
    _raise(lib().orc_primitives_to_conserved(p.shape[1], _d(p), gamma, _d(U), C.byref(e)), e)
    return U


def conserved_to_primitives(U4n, gamma=1.4):
    U = _f(U4n)
    p = np.empty_like(U)
    e = OError()
    _raise(lib().orc_conserved_to_primitives(U.shape[1], _d(U), gamma, _d(p), C.byref(e)), e)
    return p


def split_flux(prims4n, axis, sign, gamma=1.4):
    p = _f(prims4n)
    G = np.empty_like(p)
    lib().orc_split_flux(p.shape[1], _d(p), 0 if axis == "x" else 1, 1 if sign == "+" else -1, gamma, _d(G))
    return G


def full_flux(prims4n, axis, gamma=1.4):
    p = _f(prims4n)
    F = np.empty_like(p)
    lib().orc_full_flux(p.shape[1], _d(p), 0 if axis == "x" else 1, gamma, _d(F))
    return F


def local_timestep(pk: Packed, prims4n, cfl, gamma=1.4):
    p = _f(prims4n)
    dt = np.empty(pk.n)
    lib().orc_local_timestep(pk.ref, _d(p), cfl, gamma, _d(dt))
    return dt


def first_order(pk: Packed, q):
    q = _f(q)
    qx, qy = np.empty_like(q), np.empty_like(q)
    lib().orc_first_order_q_gradients(pk.ref, _d(q), _d(qx), _d(qy))
    return qx, qy


def q_derivatives(pk: Packed, q, n_inner=3):
    q = _f(q)
    qx, qy = np.empty_like(q), np.empty_like(q)
    res = np.zeros(n_inner)
    lib().orc_compute_q_derivatives(pk.ref, _d(q), n_inner, _d(qx), _d(qy), _d(res))
    return qx, qy, res


def flux_residual(pk: Packed, q, qx, qy, mode="fused", gamma=1.4):
    q, qx, qy = _f(q), _f(qx), _f(qy)
    R = np.empty_like(q)
    e = OError()
    _raise(lib().orc_flux_residual(pk.ref, _d(q), _d(qx), _d(qy), 0 if mode == "fused" else 1, gamma, _d(R),
                                   C.byref(e)), e)
    return R


def apply_boundary(pk: Packed, q, qx, qy, fs, R, gamma=1.4):
    q, qx, qy = _f(q), _f(qx), _f(qy)
    R = _f(R).copy()
    fsv = _f(fs)
    e = OError()
    _raise(lib().orc_apply_boundary(pk.ref, _d(q), _d(qx), _d(qy), _d(fsv), gamma, _d(R), C.byref(e)), e)
    return R


def state_update_rk(Uo, Us, stage, dt, R):
    Uo, Us, R, dt = _f(Uo), _f(Us), _f(R), _f(dt)
    out = np.empty_like(Us)
    lib().orc_state_update_rk(Us.shape[1], _d(Uo), _d(Us), stage, _d(dt), _d(R), _d(out))
    return out


def residue_norm(Un, Uo):
    a, b = _f(np.atleast_2d(Un)[0]), _f(np.atleast_2d(Uo)[0])
    return float(lib().orc_residue_norm(a.shape[0], _d(a), _d(b)))


def fsum(v):
    v = _f(v)
    return float(lib().orc_fsum(v.shape[0], _d(v)))


def solve(pk: Packed, prims4n, fs, n_outer, gamma=1.4, cfl=0.2, n_inner=3, mode="fused", tol=None):
    """(history, prims, U, iterations, converged) from the initial primitives."""
    p = OParams()
    for i in range(4):
        p.fs[i] = float(fs[i])
    p.gamma, p.cfl, p.n_outer, p.n_inner = gamma, cfl, n_outer, n_inner
    p.mode = 0 if mode == "fused" else 1
    p.convergence_tol = tol if tol else 0.0
    prims = _f(prims4n).copy()
    U = np.empty_like(prims)
    hist = np.zeros(n_outer)
    its, conv = C.c_int(0), C.c_int(0)
    e = OError()
    _raise(lib().orc_solve(pk.ref, C.byref(p), _d(prims), _d(U), _d(hist), C.byref(its), C.byref(conv),
                           C.byref(e)), e)
    return hist[: its.value], prims, U, its.value, bool(conv.value)
