"""CPU: the C-ABI library builds, loads, exports every symbol include/mfreg_cuda.h
declares, and its host-side logic (grid construction, validation, error mapping)
matches the reference without touching a GPU."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mfreg_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mfreg_cu_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def pkg():
    import paper_1804_10541_b200 as P
    if not os.path.exists(P._LIB_PATH):
        P.build()
    return P


def test_library_exports_every_declared_symbol(pkg):
    lib = ctypes.CDLL(pkg._LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(pkg.exported_symbols())


def test_version_and_last_error(pkg):
    assert pkg.lib().mfreg_cu_version() == 1
    assert isinstance(pkg.lib().mfreg_cu_last_error(), bytes)


def test_deformation_grid_sizes(pkg):  # test_multilevel.cpp:49-55
    g = pkg.deformation_grid_for(pkg.make_image_grid((64, 64, 64)), 4)
    assert g.m == (17, 17, 17) and g.h == (4.0, 4.0, 4.0)
    g = pkg.deformation_grid_for(pkg.make_image_grid((512, 512, 900), (0.7, 0.7, 0.7)), 4)
    assert g.m == (129, 129, 226)
    assert g.h[0] == (512 * 0.7) / 128


def test_deform_grid_errors_match_reference(pkg):  # grid.hpp:131-146
    img = pkg.make_image_grid((8, 8, 8))
    with pytest.raises(ValueError, match="needs >= 2 points per axis"):
        pkg.make_deform_grid(img, (1, 4, 4))
    with pytest.raises(ValueError, match="finer than image grid"):
        pkg.make_deform_grid(img, (10, 4, 4))
    with pytest.raises(ValueError, match="ratio must be >= 1"):
        pkg.deformation_grid_for(img, 0)
    with pytest.raises(ValueError, match="all h components must be > 0"):
        pkg.make_image_grid((4, 4, 4), (1.0, 0.0, 1.0))


def test_deform_grid_matches_oracle(pkg, oracle):
    for m, h, my in [((7, 6, 5), (1.0, 1.3, 0.8), (4, 4, 3)), ((512, 512, 900), (0.7, 0.7, 0.7), (129, 129, 226)),
                     ((256, 256, 100), (0.97, 0.97, 2.5), (65, 65, 26))]:
        g = pkg.make_deform_grid(pkg.make_image_grid(m, h), my)
        assert list(g.h) == list(oracle.make_deform_grid(m, h, my))
