"""Device split fluxes and state transforms (reference tests/test_kinetics.py,
tests/test_state.py) -- the device function under test is the one the
flux_residual kernel calls."""

import numpy as np
import pytest

from conftest import golden
from paper_2108_07031_b200 import (
    PositivityError,
    Primitives,
    conserved_to_primitives,
    full_flux,
    primitives_to_conserved,
    primitives_to_q,
    q_to_primitives,
    split_flux,
)

pytestmark = pytest.mark.gpu

STAGNANT_MASS_FLUX = 0.3989422804014327  # reference tests/test_kinetics.py:11-17


def test_stagnant_positive_mass_flux_frozen(gpu):
    g = split_flux(Primitives(1.0, 0.0, 0.0, 1.0), "x", "+")
    assert abs(float(g[0, 0]) - STAGNANT_MASS_FLUX) < 1e-15


@pytest.mark.parametrize("axis", ["x", "y"])
@pytest.mark.parametrize("sign", ["+", "-"])
def test_split_flux_matches_reference(gpu, axis, sign):
    K, _ = golden("kinetics")
    pr = Primitives.from_array(K["prims"])
    g = split_flux(pr, axis, sign)
    ref = K[f"split_{axis}{sign}"]
    assert np.all(np.abs(g - ref) <= 1e-13 * np.maximum(np.abs(ref), 1.0))


def test_full_flux_bitwise(gpu):
    K, _ = golden("kinetics")
    pr = Primitives.from_array(K["prims"])
    for axis in ("x", "y"):
        assert np.array_equal(full_flux(pr, axis), K[f"full_{axis}"])


def test_splitting_identity(gpu):
    rng = np.random.default_rng(11)
    pr = Primitives(rng.uniform(0.2, 3.0, 64), rng.uniform(-2.5, 2.5, 64), rng.uniform(-2.5, 2.5, 64),
                    rng.uniform(0.2, 3.0, 64))
    for axis in ("x", "y"):
        total = split_flux(pr, axis, "+") + split_flux(pr, axis, "-")
        ref = full_flux(pr, axis)
        assert np.max(np.abs(total - ref) / np.maximum(np.abs(ref), 1.0)) < 1e-13


def test_reflection_antisymmetry(gpu):
    rng = np.random.default_rng(5)
    pr = Primitives(rng.uniform(0.2, 3.0, 32), rng.uniform(-2.0, 2.0, 32), rng.uniform(-2.0, 2.0, 32),
                    rng.uniform(0.2, 3.0, 32))
    gp = split_flux(pr, "x", "+")
    gm = split_flux(Primitives(pr.rho, -pr.u1, pr.u2, pr.p), "x", "-")
    assert np.allclose(gp[0], -gm[0], rtol=1e-14, atol=1e-16)
    assert np.allclose(gp[1], gm[1], rtol=1e-14, atol=1e-16)
    assert np.allclose(gp[2], -gm[2], rtol=1e-14, atol=1e-16)
    assert np.allclose(gp[3], -gm[3], rtol=1e-14, atol=1e-16)


def test_supersonic_saturation(gpu):
    pr = Primitives(1.0, 8.0, 0.5, 0.5)
    assert np.allclose(split_flux(pr, "x", "+"), full_flux(pr, "x"), rtol=1e-13)
    assert np.max(np.abs(split_flux(pr, "x", "-"))) < 1e-12


def test_bad_axis_and_sign(gpu):
    pr = Primitives(1.0, 0.0, 0.0, 1.0)
    with pytest.raises(ValueError):
        split_flux(pr, "z", "+")
    with pytest.raises(ValueError):
        split_flux(pr, "x", "0")


@pytest.mark.parametrize("g", [1.4, 5.0 / 3.0])
def test_state_transforms_vs_reference(gpu, g):
    K, _ = golden("kinetics")
    tag = f"g{g:.4f}"
    pr = Primitives.from_array(K["prims"])
    assert np.array_equal(primitives_to_conserved(pr, g), K[f"U.{tag}"])
    assert np.array_equal(conserved_to_primitives(K[f"U.{tag}"], g).as_array(), K[f"U2p.{tag}"])
    q = primitives_to_q(pr, g)
    assert np.all(np.abs(q - K[f"q.{tag}"]) <= 4 * np.spacing(np.abs(K[f"q.{tag}"])))
    back = q_to_primitives(K[f"q.{tag}"], g).as_array()
    assert np.allclose(back, K[f"q2p.{tag}"], rtol=1e-14, atol=0)


def test_q_round_trip_thousand_states(gpu):
    rng = np.random.default_rng(12)
    pr = Primitives(rng.uniform(0.2, 3.0, 1000), rng.uniform(-2.5, 2.5, 1000), rng.uniform(-2.5, 2.5, 1000),
                    rng.uniform(0.2, 3.0, 1000))
    back = q_to_primitives(primitives_to_q(pr))
    for a, b in zip(pr.as_array(), back.as_array()):
        assert np.abs(a - b).max() < 1e-13


def test_examples(gpu):
    U = primitives_to_conserved(Primitives(2.0, 1.0, 0.0, 2.0))
    assert np.allclose(U[:, 0], [2.0, 2.0, 0.0, 6.0], rtol=1e-15)
    q = primitives_to_q(Primitives(1.0, 1.0, 0.0, 0.5))
    assert np.allclose(q[:, 0], [-1.0, 2.0, 0.0, -2.0], atol=1e-15)


def test_positivity_errors(gpu):
    U = primitives_to_conserved(Primitives([1.0, 1.0], [0.0, 0.0], [0.0, 0.0], [1.0, 1.0]))
    U[0, 1] = -0.5
    with pytest.raises(PositivityError) as exc:
        conserved_to_primitives(U)
    assert 1 in exc.value.indices and "density" in str(exc.value)
    U = primitives_to_conserved(Primitives(1.0, 1.0, 0.0, 1.0))
    U[3, 0] = 0.1
    with pytest.raises(PositivityError, match="pressure"):
        conserved_to_primitives(U)
    q = np.zeros((4, 1))
    q[3, 0] = 0.5
    with pytest.raises(PositivityError):
        q_to_primitives(q)
    with pytest.raises(PositivityError):
        primitives_to_q(Primitives(np.array([1.0, np.nan]), np.zeros(2), np.zeros(2), np.ones(2)))
