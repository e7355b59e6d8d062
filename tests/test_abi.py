"""The C-ABI library loads and exports every entry point include/kmf_b200.h
declares; without a GPU every product operation fails loudly (no CPU
fallback).  CPU only (no compute calls)."""

import ctypes
import re

import pytest

from conftest import ROOT
from paper_2108_07031_b200 import _lib


def declared_functions():
    text = (ROOT / "include" / "kmf_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kmf_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    declared = declared_functions()
    assert len(declared) >= 25
    assert set(declared) == set(_lib.EXPORTED)


def test_library_exports_every_symbol():
    so = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared_functions():
        assert hasattr(so, name), name


def test_abi_version():
    assert _lib.lib().kmf_abi_version() == 1


def test_structs_match_header_sizes():
    # kmf_stencil: 2 int64 + 8 pointers; kmf_frame: int64 + 5 pointers + 3 stencils
    assert ctypes.sizeof(_lib.Stencil) == 2 * 8 + 8 * 8
    assert ctypes.sizeof(_lib.Frame) == 8 + 5 * 8 + 3 * ctypes.sizeof(_lib.Stencil)


def _no_gpu():
    return _lib.lib().kmf_device_count() == 0


@pytest.mark.skipif(not _no_gpu(), reason="checks the no-GPU behaviour")
def test_no_silent_cpu_fallback(small_naca, small_naca_conn):
    from paper_2108_07031_b200 import primitives_to_q, free_stream, solve, SolverConfig

    prims = free_stream(0.63, 2.0, n=10)
    with pytest.raises(_lib.DeviceError):
        primitives_to_q(prims)
    with pytest.raises(_lib.DeviceError):
        solve(SolverConfig(mach=0.63, n_outer=1), small_naca, small_naca_conn)


def test_oracle_library_builds_and_is_separate():
    from oracle import oracle as O

    O.lib()
    # the product library must not depend on the oracle
    so = (ROOT / "paper_2108_07031_b200" / "libkmf_b200.so").read_bytes()
    assert b"orc_" not in so and b"kmf_oracle" not in so
    import paper_2108_07031_b200 as pkg

    for mod in ("solver", "lsq", "state", "kinetics", "geometry", "_device", "_lib"):
        src = (ROOT / "paper_2108_07031_b200" / f"{mod}.py").read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), mod
    assert pkg.__version__


def test_builder_library_exports_every_symbol():
    from paper_2108_07031_b200 import builder

    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "kmf_build.h").read_text(), flags=re.S)
    names = sorted(set(re.findall(r"\b(kmfb_[a-z0-9_]+)\s*\(", text)))
    assert names == ["kmfb_assemble", "kmfb_knn", "kmfb_radius", "kmfb_set_threads", "kmfb_threads", "kmfb_visibility"]
    so = ctypes.CDLL(str(builder.LIB_PATH))
    for name in names:
        assert hasattr(so, name), name
    assert builder.lib().kmfb_threads() >= 1
    # set-up code, not product compute: it must not depend on the oracle either
    for mod in ("builder", "store", "partition", "dist", "reorder", "integration"):
        src = (ROOT / "paper_2108_07031_b200" / f"{mod}.py").read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), mod


@pytest.mark.gpu
def test_plain_c_host(gpu, tmp_path):
    """tests/c/abi_smoke.c links libkmf_b200.so from C (no Python, no torch
    types) and calls three context-free operators; its hex-printed results
    equal the ctypes binding's bit for bit."""
    import shutil
    import subprocess

    import numpy as np

    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    exe = tmp_path / "abi_smoke"
    subprocess.run(["gcc", "-std=c11", "-O1", "-I", str(ROOT / "include"), str(ROOT / "tests" / "c" / "abi_smoke.c"),
                    "-L", str(_lib.LIB_PATH.parent), "-lkmf_b200", "-Wl,-rpath," + str(_lib.LIB_PATH.parent),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, (out.returncode, out.stderr)
    got = {}
    for line in out.stdout.split("\n"):
        if line:
            tag, v = line.split()
            got.setdefault(tag, []).append(float.fromhex(v))
    prims = np.array([1.0, 1.1, 0.9, 1.05, 0.97, 0.6, 0.62, 0.58, 0.0, -0.3,
                      0.02, 0.0, -0.05, 0.1, 0.2, 0.714, 0.8, 0.69, 0.7, 0.75]).reshape(4, 5)
    L = _lib.lib()
    q = np.empty((4, 5))
    fl = np.empty(5, np.uint8)
    assert L.kmf_op_primitives_to_q(5, _lib.dptr(prims), 1.4, _lib.dptr(q), fl.ctypes.data_as(_lib._u8p)) == 0
    G = np.empty((4, 5))
    assert L.kmf_op_split_flux(5, _lib.dptr(prims), 0, 1, 1.4, _lib.dptr(G)) == 0
    U1 = prims.copy()
    U1.flat[2] += 1e-3
    res = np.zeros(1)
    assert L.kmf_op_residue(5, _lib.dptr(U1), _lib.dptr(prims), _lib.dptr(res)) == 0
    assert np.array_equal(np.array(got["q"]), q.ravel())
    assert np.array_equal(np.array(got["G"]), G.ravel())
    assert got["res"][0] == res[0]
