"""Kinetic split fluxes on the device -- drop-in for reference ``kmf.kinetics``.

``split_flux`` runs the very device function the flux_residual and
boundary kernels use (kmf_flux.cuh ``fsflux_m``: lean table exp, branch-free
erf with the |s| >= 1 tail, per-state moment constants), so the operator
test certifies the solver's own arithmetic; ``kmf_probe_edge_state``
(tests/test_gpu_gamma.py) probes the kernel's decode + flux composition.  The Gauss-Legendre ``moment_oracle`` of the reference is a
test oracle and lives in the test suite, not here.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .state import GAMMA_DEFAULT, Primitives, prims_array

_AXES = ("x", "y")
_SIGNS = ("+", "-")


def internal_energy_scale(beta, gamma: float = GAMMA_DEFAULT):
    """I0 = (2-gamma)/(2 beta (gamma-1)) (kinetics.py:53-56)."""
    return (2.0 - gamma) / (2.0 * np.asarray(beta) * (gamma - 1.0))


def _check_axis(axis):
    if axis not in _AXES:
        raise ValueError(f"axis must be one of {_AXES}, got {axis!r}")


def split_flux(prim: Primitives, axis: str, sign: str, gamma: float = GAMMA_DEFAULT) -> np.ndarray:
    """Half-range Maxwellian flux G_axis^sign, shape (4, n) (kinetics.py:71-106)."""
    _check_axis(axis)
    if sign not in _SIGNS:
        raise ValueError(f"sign must be one of {_SIGNS}, got {sign!r}")
    _lib.require_device()
    pa = prims_array(prim)
    out = np.empty_like(pa)
    _lib.check(
        _lib.lib().kmf_op_split_flux(pa.shape[1], _lib.dptr(pa), _AXES.index(axis), 1 if sign == "+" else -1,
                                     gamma, _lib.dptr(out)),
        "split_flux",
    )
    return out


def full_flux(prim: Primitives, axis: str, gamma: float = GAMMA_DEFAULT) -> np.ndarray:
    """Euler flux along ``axis`` (kinetics.py:59-68), bitwise."""
    _check_axis(axis)
    _lib.require_device()
    pa = prims_array(prim)
    out = np.empty_like(pa)
    _lib.check(_lib.lib().kmf_op_full_flux(pa.shape[1], _lib.dptr(pa), _AXES.index(axis), gamma, _lib.dptr(out)),
               "full_flux")
    return out
