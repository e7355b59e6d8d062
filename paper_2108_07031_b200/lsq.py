"""Least-squares q-gradients on the device -- drop-in for reference ``kmf.lsq``.

``first_order_q_gradients`` (lsq.py:164-175) and ``compute_q_derivatives``
(lsq.py:184-245) run the sm_100a kernels k_first_order / k_sweep: one thread
per point, neighbour slots in reference CSR order, every product rounded
before it is summed -- bitwise equal to the reference on the same q.
``block_map`` is accepted for signature compatibility and ignored: the
device result does not depend on any blocking (the reference's own
guarantee, tests/test_lsq.py:120-138).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib
from ._device import device_for
from .geometry import Connectivity


@dataclass
class QGradients:
    """Nodal q gradients, (4, n) each; ``inner_residuals`` = max |update|
    per Jacobi sweep (lsq.py:48-59)."""

    qx: np.ndarray
    qy: np.ndarray
    inner_residuals: tuple = ()


def first_order_q_gradients(q: np.ndarray, conn: Connectivity) -> QGradients:
    dev = device_for(conn)
    qa = _lib.f64(q)
    qx = np.empty_like(qa)
    qy = np.empty_like(qa)
    _lib.check(_lib.lib().kmf_op_first_order(dev.handle, _lib.dptr(qa), _lib.dptr(qx), _lib.dptr(qy)),
               "first_order_q_gradients")
    return QGradients(qx=qx, qy=qy)


def compute_q_derivatives(
    q: np.ndarray,
    conn: Connectivity,
    n_inner: int = 3,
    prev: QGradients | None = None,
    block_map: Callable | None = None,
) -> QGradients:
    """Cold-started (or ``prev``-started) Jacobi sweeps of the implicit
    defect-corrected gradient relation, double-buffered on the device."""
    if n_inner < 1:
        raise ValueError("n_inner must be at least 1")
    dev = device_for(conn)
    qa = _lib.f64(q)
    qx = np.empty_like(qa)
    qy = np.empty_like(qa)
    res = np.zeros(n_inner)
    if prev is not None:
        px, py = _lib.f64(prev.qx), _lib.f64(prev.qy)
        ppx, ppy = _lib.dptr(px), _lib.dptr(py)
    else:
        ppx = ppy = C.cast(None, C.POINTER(C.c_double))
    _lib.check(
        _lib.lib().kmf_op_q_derivatives(dev.handle, _lib.dptr(qa), n_inner, ppx, ppy, _lib.dptr(qx), _lib.dptr(qy),
                                        _lib.dptr(res)),
        "compute_q_derivatives",
    )
    return QGradients(qx=qx, qy=qy, inner_residuals=tuple(float(r) for r in res))
