"""Shared test configuration.

Tests marked ``gpu`` need a CUDA device (they run on the B200 box); everything
else runs on CPU.  Helpers: ``rel_err`` is the reference's max-abs relative
error (pkg/tests/test_kernels.py:32-36), ``golden`` loads the fixtures that
tests/golden/make_golden.py produced by running the reference itself.
"""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def rel_err(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    scale = np.max(np.abs(want)) if want.size else 0.0
    if scale == 0:
        return float(np.max(np.abs(got))) if got.size else 0.0
    return float(np.max(np.abs(got - want)) / scale)


def rel_l2(got, want):
    return float(np.linalg.norm(np.asarray(got) - np.asarray(want)) / np.linalg.norm(np.asarray(want)))


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN / "reference_outputs.npz")


@pytest.fixture(scope="session")
def tables():
    return json.loads((GOLDEN / "reference_tables.json").read_text())
