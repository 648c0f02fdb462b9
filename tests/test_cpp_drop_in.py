"""The C++ drop-in header (include/mfreg_b200.hpp): reference-style client code
compiles with g++ against it, links libmfreg_cuda.so, maps errors to the
reference's exception types, and (on a GPU) reproduces the reference's Objective
and Gauss-Newton trace bit for bit."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def _build(tmp_path):
    import paper_1804_10541_b200 as P
    if not os.path.exists(P._LIB_PATH):
        P.build()
    exe = str(tmp_path / "drop_in")
    libdir = os.path.dirname(P._LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "drop_in.cpp"), "-L", libdir, "-lmfreg_cuda",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    return exe


def test_drop_in_compiles_and_maps_errors(tmp_path):
    out = subprocess.run([_build(tmp_path), "host", str(tmp_path)], capture_output=True, text=True, check=True).stdout
    assert "deform 17 17 17 h 4" in out
    assert "invalid_argument: deformation grid finer than image grid" in out
    assert "io deform 17 17 17 14739 0.25" in out
    assert f"runtime_error: cannot open sidecar {tmp_path}/drop_in.def.missing.meta" in out


@pytest.mark.gpu
def test_drop_in_matches_reference(tmp_path, oracle):
    out = subprocess.run([_build(tmp_path), "gpu"], capture_output=True, text=True, check=True).stdout.splitlines()
    import paper_1804_10541_b200 as P
    m, h = (24, 20, 18), (0.97, 0.97, 2.5)
    img = P.make_image_grid(m, h)
    R = P.make_phantom(img) * 1000.0          # the same device generator the C++ client used
    T = P.warp_sinusoid(R, img, 3.0, 42)
    my, _ = oracle.deformation_grid_for(m, h, 4)
    o = oracle.objective(R, T, m, h, my, 10.0, 10.0, 1.0)
    J, D, S, _ = o.eval(o.identity())
    jl = [l for l in out if l.startswith("J ")][0].split()
    assert (float(jl[1]), float(jl[3]), float(jl[5])) == (J, D, S)
    y, trace, _ = o.minimize(o.identity(), "gn", __import__("oracle.oracle", fromlist=["OptConfig"]).OptConfig.defaults(max_iters=3))
    its = [l.split() for l in out if l.startswith("it ")]
    assert len(its) == len(trace)
    for row, ref in zip(its, trace):
        assert float(row[3]) == ref[2] and int(row[5]) == ref[1] and float(row[7]) == ref[6]


def _build_client(tmp_path):
    import paper_1804_10541_b200 as P
    if not os.path.exists(P._LIB_PATH):
        P.build()
    exe = str(tmp_path / "api_client")
    libdir = os.path.dirname(P._LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "api_client.cpp"), "-L", libdir, "-lmfreg_cuda",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    return exe


def test_api_client_compiles_unchanged(tmp_path):
    """The reference-style client (a user Problem, cg_solve / armijo_search with lambdas, the
    kernel-level ngf / volume / transfer / curvature / multilevel calls, LevelResult fields)
    compiles against the drop-in header exactly as it does against the reference headers."""
    assert os.path.exists(_build_client(tmp_path))


@pytest.mark.gpu
def test_api_client_matches_reference(tmp_path):
    """Every printed result (bit patterns and byte hashes) equals the unmodified reference's
    output on the same inputs (tests/golden/api_client_ref.txt, gen_api_client.py)."""
    out = subprocess.run([_build_client(tmp_path)], capture_output=True, text=True, check=True).stdout.splitlines()
    ref = open(os.path.join(ROOT, "tests", "golden", "api_client_ref.txt")).read().splitlines()
    assert len(out) == len(ref)
    bad = [(o, r) for o, r in zip(out, ref) if o != r]
    assert not bad, bad[:10]
