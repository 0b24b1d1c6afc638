"""The C-ABI library and the host shim (CPU, no compute calls).

* libgk.so loads and exports every entry point include/gk.h declares, with the
  signatures _lib.py binds;
* the Python mirror raises the reference's ValueErrors before touching a device;
* the product package never imports the oracle (no CPU fallback).
"""
import ast
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2305_10553_b200 import _lib
from paper_2305_10553_b200.grid import GridShape
from paper_2305_10553_b200.kernels import (collision_kernel, field_kernel, nonlinear_kernel, run_kernel,
                                           shear_kernel, stream_kernel, time_kernel)
from paper_2305_10553_b200.spectral import bracket, to_real, to_spectrum

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "gk.h"


def header_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(gk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), "ctypes bindings must mirror include/gk.h"
    assert lib.gk_version() == _lib.ABI_VERSION


def test_error_reporting_without_device():
    lib = _lib.load()
    rc = lib.gk_field(None, None, None, 1, 1, 1, None)
    assert rc != 0
    assert b"null" in lib.gk_last_error()
    assert lib.gk_bracket_workspace_bytes(None, 1, 1) == -1


SMALL = GridShape(12, 4, 5, 3, 2, 2)


def test_validation_errors_raise_before_any_device_work():
    h = np.zeros(SMALL.dims, dtype=complex)
    m = SMALL.velocity_size
    with pytest.raises(ValueError):
        field_kernel(h, np.zeros((2, 2, 2)))
    with pytest.raises(ValueError):
        stream_kernel(h, (0.5, 0.5))
    with pytest.raises(ValueError):
        stream_kernel(h, tuple(range(7)))
    with pytest.raises(ValueError):
        stream_kernel(h, (1.0,), "fused")
    with pytest.raises(ValueError):
        shear_kernel(h, np.zeros(3, dtype=int))
    with pytest.raises(ValueError):
        shear_kernel(h, np.full(SMALL.n_toroidal, SMALL.n_radial + 1))
    with pytest.raises(ValueError):
        collision_kernel(h, np.zeros((SMALL.n_theta, m, m + 1)))
    with pytest.raises(ValueError):
        nonlinear_kernel(h, np.zeros((4, 4, 12), dtype=complex), (18, 12))
    with pytest.raises(ValueError):
        nonlinear_kernel(h, np.zeros(SMALL.field_dims, dtype=complex), (17, 12))  # x below 3/2 bound
    with pytest.raises(ValueError):
        run_kernel("advect", h, {})
    with pytest.raises(ValueError):
        run_kernel("field", h, {}, variant="fast")
    with pytest.raises(ValueError):
        time_kernel("field", "original", SMALL, reps=2, seed=1)
    f = np.zeros((4, 8), dtype=complex)
    with pytest.raises(ValueError):
        bracket(f, f, 11, 30)
    with pytest.raises(ValueError):
        bracket(f, f, 12, 9)
    with pytest.raises(ValueError):
        bracket(f, np.zeros((3, 8), dtype=complex), 16, 16)
    with pytest.raises(ValueError):
        to_real(np.zeros((3, 8), dtype=complex), 7, 12)
    with pytest.raises(ValueError):
        to_spectrum(np.zeros((6, 8)), 8, 5)


def test_product_package_never_imports_the_oracle():
    pkg = ROOT / "paper_2305_10553_b200"
    for py in pkg.rglob("*.py"):
        tree = ast.parse(py.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert not any(a.name.split(".")[0] == "oracle" for a in node.names), py
            if isinstance(node, ast.ImportFrom) and node.module:
                assert node.module.split(".")[0] != "oracle", py


def test_kernel_sources_target_sm100a_only():
    from paper_2305_10553_b200 import build
    assert build.ARCH == ["-gencode", "arch=compute_100a,code=sm_100a"]


def test_collision_mode_switch_without_device():
    lib = _lib.load()
    prev = lib.gk_collision_mode(-1)
    try:
        assert lib.gk_collision_mode(1) == prev
        assert lib.gk_collision_mode(-1) == 1
        assert lib.gk_collision_mode(7) == 1  # out of range: query only
        assert lib.gk_collision_mode(2) == 1 and lib.gk_collision_mode(-1) == 2
    finally:
        lib.gk_collision_mode(prev)
