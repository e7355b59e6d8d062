"""Accuracy of the flux-path transcendentals (kmf_fastmath.cuh) against
100-digit decimal references: exp <= 1 ulp, erf <= 1 ulp of max(|erf|, 0.1),
reciprocal / rsqrt <= 1 ulp."""

from decimal import Decimal as D, getcontext

import numpy as np
import pytest

from paper_2108_07031_b200 import _lib

pytestmark = pytest.mark.gpu
getcontext().prec = 60


def probe(x, which):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _lib.check(_lib.lib().kmf_fastmath_probe(x.size, _lib.dptr(x), which, _lib.dptr(out)), "probe")
    return out


def erf_dec(x: float) -> float:
    xd = D(x)
    s, term, n, x2 = D(0), xd, 0, xd * xd
    while True:
        t = term / (2 * n + 1)
        s += t
        if abs(t) < D(10) ** -40 and n > 3:
            break
        n += 1
        term = -term * x2 / n
    pi = D("3.14159265358979323846264338327950288419716939937510582097494459")
    return float(2 / pi.sqrt() * s)


def ulps(a, ref, floor=0.0):
    scale = np.spacing(np.maximum(np.abs(ref), floor))
    return np.abs(a - ref) / scale


def test_exp(gpu):
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.uniform(-40, 40, 3000), rng.uniform(-1, 1, 1000), rng.uniform(-700, 700, 500),
                        [0.0, 1.0, -1.0, 0.5, -0.3465, 0.3466]])
    ref = np.array([float(D(v).exp()) for v in x])
    assert ulps(probe(x, 0), ref).max() <= 1.0


def test_exp_table(gpu):
    """fexp_tab (lean flux path): 64-entry hi/lo table + degree-5 expm1."""
    rng = np.random.default_rng(4)
    x = np.concatenate([rng.uniform(-40, 40, 3000), rng.uniform(-1, 1, 1000), rng.uniform(-700, 700, 500),
                        [0.0, 1.0, -1.0, 0.5, -0.3465, 0.3466, 0.0054, -0.0054]])
    ref = np.array([float(D(v).exp()) for v in x])
    assert ulps(probe(x, 4), ref).max() <= 1.0
    out = probe(np.array([-800.0, -746.0, 709.0]), 4)
    assert out[0] == 0.0 and out[1] == 0.0 and np.isfinite(out[2])


def test_exp_table_unclamped_nonpositive(gpu):
    """fexp_tab<false> (the Maxwellian exp(-s^2)): same accuracy on x <= 0,
    and arguments far below the underflow threshold still give 0."""
    rng = np.random.default_rng(5)
    x = -np.concatenate([rng.uniform(0, 40, 3000), rng.uniform(0, 700, 500), [0.0, 1e-300, 0.3466]])
    ref = np.array([float(D(v).exp()) for v in x])
    assert ulps(probe(x, 5), ref).max() <= 1.0
    assert np.all(probe(np.array([-746.0, -800.0, -1e5, -2e7]), 5) == 0.0)


def test_exp_underflow_and_nan(gpu):
    out = probe(np.array([-800.0, -746.0, 709.0, np.nan]), 0)
    assert out[0] == 0.0 and out[1] == 0.0 and np.isfinite(out[2]) and np.isnan(out[3])


def test_erf(gpu):
    rng = np.random.default_rng(2)
    x = np.concatenate([rng.uniform(-1, 1, 1500), rng.uniform(-7, 7, 1500), [0.0, 1.0, -1.0, 2.5, 4.5, 6.5, 8.0]])
    ref = np.array([erf_dec(v) for v in x])
    # absolute error judged against max(|erf|, 0.1): erf feeds A = (1 +- erf)/2
    assert ulps(probe(x, 1), ref, floor=0.1).max() <= 1.0


def test_rcp_rsqrt(gpu):
    rng = np.random.default_rng(3)
    x = np.exp(rng.uniform(-30, 30, 5000))
    assert ulps(probe(x, 2), 1.0 / x).max() <= 1.0
    ref = np.array([float(1 / D(v).sqrt()) for v in x])
    assert ulps(probe(x, 3), ref).max() <= 1.0
