"""Volume, deformation and landmark files — the reference's `mfreg::io` API
(io.hpp; io.cpp:111-348) and the CLI `warp` command (tools/mfreg_cli.cpp:112-135)
over the C ABI. Same names, argument meaning and errors: file / format problems
raise RuntimeError with the reference's std::runtime_error text, length
mismatches raise ValueError (std::invalid_argument). Volume payloads are
converted to fp64 on the GPU; per-landmark errors and the warp run on the GPU."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import (DEVICE, HOST, GridDesc, _check, _empty_like_kind, _Grid, _ptr, _where_of, _as_input, lib)


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def _grid_from(g: _Grid, nodal: bool) -> GridDesc:
    return GridDesc(tuple(int(v) for v in g.m), tuple(float(v) for v in g.h), nodal)


def read_volume(path, device: bool = False):
    """io::read_volume -> (data, image GridDesc); data on the GPU when `device`."""
    g = _Grid()
    _check(lib().mfreg_cu_read_volume(_path(path), C.byref(g), None, HOST))
    grid = _grid_from(g, False)
    if device:
        import torch
        out = torch.empty(grid.count(), dtype=torch.float64, device="cuda")
    else:
        out = np.empty(grid.count())
    p, w = _ptr(out)
    _check(lib().mfreg_cu_read_volume(_path(path), C.byref(g), p, w))
    return out, grid


def write_volume(path, data, grid: GridDesc) -> None:
    """io::write_volume (MET_DOUBLE, LOCAL payload)."""
    w = _where_of(data)
    d = _as_input(data, w)
    if (d.numel() if hasattr(d, "numel") else d.size) != grid.count():
        raise ValueError("write_volume: data length does not match the grid")
    _check(lib().mfreg_cu_write_volume(_path(path), C.byref(grid.c()), _ptr(d)[0], w))


def write_deformation(path, y, grid: GridDesc) -> None:
    """io::write_deformation: raw little-endian doubles + '<path>.meta' sidecar."""
    w = _where_of(y)
    yy = _as_input(y, w)
    n = yy.numel() if hasattr(yy, "numel") else yy.size
    _check(lib().mfreg_cu_write_deformation(_path(path), _ptr(yy)[0], int(n), C.byref(grid.c()), w))


def read_deformation_grid(path) -> GridDesc:
    """io::read_deformation_grid (nodal grid from the sidecar)."""
    g = _Grid()
    _check(lib().mfreg_cu_read_deformation_grid(_path(path), C.byref(g)))
    return _grid_from(g, True)


def read_deformation(path, grid: GridDesc, device: bool = False):
    """io::read_deformation: the field (3 * grid.count()) checked against `grid`."""
    if device:
        import torch
        out = torch.empty(3 * grid.count(), dtype=torch.float64, device="cuda")
    else:
        out = np.empty(3 * grid.count())
    p, w = _ptr(out)
    _check(lib().mfreg_cu_read_deformation(_path(path), C.byref(grid.c()), p, w))
    return out


def read_landmarks(path, spacing) -> np.ndarray:
    """io::read_landmarks -> (N, 3) physical cell-centre coordinates."""
    sp = (C.c_double * 3)(*[float(v) for v in spacing])
    n = C.c_int64(0)
    _check(lib().mfreg_cu_read_landmarks(_path(path), sp, None, 0, C.byref(n)))
    out = np.empty((n.value, 3))
    _check(lib().mfreg_cu_read_landmarks(_path(path), sp, out.ctypes.data if n.value else None, n.value, C.byref(n)))
    return out


def landmark_error(fixed, moving, y, grid: GridDesc):
    """io::landmark_error -> (mean, stddev, count) of |phi(p_fixed) - p_moving|."""
    f = np.ascontiguousarray(np.asarray(fixed, dtype=np.float64).reshape(-1, 3))
    m = np.ascontiguousarray(np.asarray(moving, dtype=np.float64).reshape(-1, 3))
    w = _where_of(y)
    yy = _as_input(y, w)
    ny = yy.numel() if hasattr(yy, "numel") else yy.size
    mean, sd, cnt = C.c_double(), C.c_double(), C.c_int64()
    _check(lib().mfreg_cu_landmark_error(f.ctypes.data if len(f) else None, len(f), m.ctypes.data if len(m) else None,
                                         len(m), _ptr(yy)[0], int(ny), C.byref(grid.c()), w, C.byref(mean),
                                         C.byref(sd), C.byref(cnt)))
    return mean.value, sd.value, cnt.value


def warp_volume(vol, image: GridDesc, y, nodal: GridDesc):
    """CLI `warp` (mfreg_cli.cpp:112-135) without files: vol(P y) on the volume's grid."""
    w = _where_of(vol, y)
    v, yy = _as_input(vol, w), _as_input(y, w)
    out = _empty_like_kind(v, image.count())
    _check(lib().mfreg_cu_warp_volume(_ptr(v)[0], C.byref(image.c()), _ptr(yy)[0], C.byref(nodal.c()), _ptr(out)[0],
                                      w))
    return out


def warp_files(input_path, def_path, out_path) -> None:
    """CLI `warp` end to end: read the volume and the deformation, warp on the GPU,
    write the MET_DOUBLE result (tools/mfreg_cli.cpp:112-135)."""
    vol, img = read_volume(input_path, device=True)
    dg = read_deformation_grid(def_path)
    y = read_deformation(def_path, dg, device=True)
    out = warp_volume(vol, img, y, dg)
    write_volume(out_path, out, img)
