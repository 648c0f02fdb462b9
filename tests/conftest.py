"""Shared test helpers. `-m gpu` tests need a B200 (they call the CUDA library
through the C ABI); everything else runs on CPU."""
from __future__ import annotations

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def bits_equal(a, b) -> bool:
    """Bitwise equality of float64 arrays/scalars (treats +0/-0 as different)."""
    a = np.atleast_1d(np.asarray(a, dtype=np.float64))
    b = np.atleast_1d(np.asarray(b, dtype=np.float64))
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def max_rel(got, expect) -> float:
    """Reference metric max|a-b| / max|b| (tests/acceptance.cpp:40-50)."""
    got = np.asarray(got, dtype=np.float64)
    expect = np.asarray(expect, dtype=np.float64)
    scale = max(np.max(np.abs(expect)) if expect.size else 0.0, 1e-30)
    return float(np.max(np.abs(got - expect)) / scale) if got.size else 0.0


def golden_files(prefix: str):
    return sorted(glob.glob(os.path.join(GOLDEN, f"{prefix}_*.npz")))


def load(path: str) -> dict:
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def tup(a, cast=int):
    return tuple(cast(x) for x in np.asarray(a).ravel())


@pytest.fixture(scope="session")
def oracle():
    """The CPU checker: the compiled reference when present, else the C port."""
    from oracle.oracle import Oracle, available
    if not available("port") or (os.path.isdir("/root/reference/proj/src") and not available("ref")):
        from oracle.oracle import build
        build()
    return Oracle("ref") if available("ref") else Oracle("port")


@pytest.fixture(scope="module")
def P():
    import paper_1804_10541_b200 as P
    return P
