"""B200-native NGF + curvature matrix-free derivative path (arXiv 1804.10541).

Python host mirror of the reference C++ API (``/root/reference/proj/include/mfreg``)
over the C ABI in ``include/mfreg_cuda.h`` (``libmfreg_cuda.so``, built in-tree for
sm_100a). Every call runs on the GPU through that library; there is no CPU
fallback: importing this package fails loudly when the extension is missing.

Arrays may be numpy (host) or CUDA torch tensors (device, fp64, contiguous);
outputs come back as the same kind as the principal input.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Sequence

import numpy as np

from ._build import LIB as _LIB_PATH
from ._build import variant_lib as _variant_lib

if os.environ.get("MFREG_LIB_VARIANT"):  # A/B experiment builds (scripts/variants.py)
    _LIB_PATH = _variant_lib(os.environ["MFREG_LIB_VARIANT"])

__all__ = [
    "GridDesc", "NgfParams", "OptimizerConfig", "IterationRecord", "MultilevelConfig", "Method", "Mode",
    "make_image_grid", "make_deform_grid", "deformation_grid_for", "transfer_apply", "transfer_apply_transpose",
    "sample_deformed", "downsample", "prolong", "laplacian_apply", "curvature_value", "curvature_gradient",
    "curvature_hessian_vec", "NgfContext", "Objective", "cg_solve", "lbfgs_minimize", "gauss_newton_minimize",
    "register_multilevel", "make_phantom", "warp_sinusoid", "lib", "launch_count", "build",
]

PARITY, FAST = 0, 1
HOST, DEVICE = 0, 1


class Mode:
    PARITY = PARITY  # bitwise replica of the reference
    FAST = FAST      # tree reductions + factored GN Hv (max-rel <= 1e-9)
    FAST32 = 2       # FAST on single-precision image state and arithmetic (max-rel <= 1e-4)


class Method:
    LBFGS = 0        # mfreg::Method::Lbfgs
    GAUSS_NEWTON = 1  # mfreg::Method::GaussNewton


def build(force: bool = False) -> str:
    from ._build import build as _b
    return _b(force=force)


# ------------------------------------------------------------------ C structs
class _Grid(C.Structure):
    _fields_ = [("m", C.c_int64 * 3), ("h", C.c_double * 3)]


class _OptConfig(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("c1", C.c_double), ("beta", C.c_double), ("max_backtracks", C.c_int),
                ("cg_max_iters", C.c_int), ("cg_rel_tol", C.c_double), ("h0_max_iters", C.c_int),
                ("h0_rel_tol", C.c_double), ("lbfgs_history", C.c_int), ("gamma", C.c_double),
                ("tol_rel_j", C.c_double), ("tol_grad", C.c_double), ("tol_step", C.c_double)]


class _IterRecord(C.Structure):
    _fields_ = [("iter", C.c_int), ("cg_iters", C.c_int), ("j", C.c_double), ("distance", C.c_double),
                ("regularizer", C.c_double), ("grad_norm", C.c_double), ("step", C.c_double)]


class _MlConfig(C.Structure):
    _fields_ = [("levels", C.c_int), ("deform_ratio", C.c_int64), ("tau", C.c_double), ("rho", C.c_double),
                ("alpha", C.c_double), ("method", C.c_int), ("mode", C.c_int), ("opt", _OptConfig)]


_vp = C.c_void_p
_dp = C.c_void_p  # raw pointers (host or device) are passed as void*
_gp = C.POINTER(_Grid)

_SIGS = {
    "mfreg_cu_last_error": ([], C.c_char_p),
    "mfreg_cu_version": ([], C.c_int),
    "mfreg_cu_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "mfreg_cu_set_device": ([C.c_int], C.c_int),
    "mfreg_cu_synchronize": ([], C.c_int),
    "mfreg_cu_device_memory_peak": ([C.c_int, C.POINTER(C.c_int64)], C.c_int),
    "mfreg_cu_launch_count": ([], C.c_int64),
    "mfreg_cu_make_deform_grid": ([_gp, C.POINTER(C.c_int64), _gp], C.c_int),
    "mfreg_cu_deformation_grid_for": ([_gp, C.c_int64, _gp], C.c_int),
    "mfreg_cu_transfer_apply": ([_gp, _gp, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_transfer_apply_transpose": ([_gp, _gp, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_sample_deformed": ([_gp, _dp, _dp, C.c_int64, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_downsample": ([_gp, _dp, _dp, _gp, C.c_int], C.c_int),
    "mfreg_cu_laplacian_apply": ([_gp, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_curvature_value": ([_gp, _dp, C.POINTER(C.c_double), C.c_int, C.c_int], C.c_int),
    "mfreg_cu_curvature_gradient": ([_gp, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_curvature_hessian_vec": ([_gp, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_ngf_create": ([_dp, _gp, C.c_double, C.c_double, C.c_int, C.c_int, C.POINTER(_vp)], C.c_int),
    "mfreg_cu_ngf_destroy": ([_vp], C.c_int),
    "mfreg_cu_ngf_populate": ([_vp, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_ngf_value": ([_vp, C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_ngf_gradient": ([_vp, _dp, C.c_int], C.c_int),
    "mfreg_cu_ngf_hessian_vec": ([_vp, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_ngf_workspace": ([_vp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_objective_create": ([_dp, _dp, _gp, _gp, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                   C.POINTER(_vp)], C.c_int),
    "mfreg_cu_objective_destroy": ([_vp], C.c_int),
    "mfreg_cu_objective_dof": ([_vp, C.POINTER(C.c_int64)], C.c_int),
    "mfreg_cu_objective_min_spacing": ([_vp, C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_objective_identity": ([_vp, _dp, C.c_int], C.c_int),
    "mfreg_cu_objective_eval": ([_vp, _dp, _dp, C.c_int, C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_objective_last": ([_vp, C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_objective_gn_hessian_vec": ([_vp, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_read_volume": ([C.c_char_p, C.POINTER(_Grid), _dp, C.c_int], C.c_int),
    "mfreg_cu_write_volume": ([C.c_char_p, C.POINTER(_Grid), _dp, C.c_int], C.c_int),
    "mfreg_cu_write_deformation": ([C.c_char_p, _dp, C.c_int64, C.POINTER(_Grid), C.c_int], C.c_int),
    "mfreg_cu_read_deformation_grid": ([C.c_char_p, C.POINTER(_Grid)], C.c_int),
    "mfreg_cu_read_deformation": ([C.c_char_p, C.POINTER(_Grid), _dp, C.c_int], C.c_int),
    "mfreg_cu_read_landmarks": ([C.c_char_p, C.POINTER(C.c_double), _dp, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
    "mfreg_cu_landmark_error": ([_dp, C.c_int64, _dp, C.c_int64, _dp, C.c_int64, C.POINTER(_Grid), C.c_int,
                                 C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)], C.c_int),
    "mfreg_cu_warp_volume": ([_dp, C.POINTER(_Grid), _dp, C.POINTER(_Grid), _dp, C.c_int], C.c_int),
    "mfreg_cu_objective_profile_kernel": ([_vp, C.c_int, _dp, C.c_int, C.c_longlong, C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_objective_seed_hessian_vec": ([_vp, _dp, C.c_double, _dp, C.c_int], C.c_int),
    "mfreg_cu_objective_dot": ([_vp, _dp, _dp, C.c_int, C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_slab_partition": ([_gp, _gp, C.c_int, C.POINTER(C.c_int32)], C.c_int),
    "mfreg_cu_slab_partition_mode": ([_gp, _gp, C.c_int, C.c_int, C.POINTER(C.c_int32)], C.c_int),
    "mfreg_cu_objective_create_slab": ([_dp, _dp, _gp, _gp, C.c_double, C.c_double, C.c_double,
                                        C.POINTER(C.c_int32), C.c_int, C.POINTER(_vp)], C.c_int),
    "mfreg_cu_cg_solve": ([_vp, C.c_int, C.c_double, _dp, C.c_int, C.c_double, _dp, C.POINTER(C.c_int),
                           C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_int], C.c_int),
    "mfreg_cu_minimize": ([_vp, C.c_int, _dp, C.POINTER(_OptConfig), _dp, C.POINTER(_IterRecord), C.c_int,
                           C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int], C.c_int),
    "mfreg_cu_prolong": ([_gp, _gp, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_register_multilevel": ([_dp, _dp, _gp, C.POINTER(_MlConfig), _dp, _gp, C.POINTER(_IterRecord), C.c_int,
                                      C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int], C.c_int),
    "mfreg_cu_make_phantom": ([_gp, _dp, C.c_int], C.c_int),
    "mfreg_cu_warp_sinusoid": ([_gp, _dp, C.c_double, C.c_uint64, _dp, C.c_int], C.c_int),
    "mfreg_cu_scale": ([C.c_int64, C.c_double, _dp, C.c_int], C.c_int),
    "mfreg_cu_register_multilevel_ex": ([_dp, _dp, _gp, C.POINTER(_MlConfig), _dp, _gp, C.POINTER(_IterRecord),
                                         C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), _gp, _gp, _dp, C.c_int64,
                                         C.c_int], C.c_int),
    "mfreg_cu_vec_dot": ([_dp, _dp, C.c_int64, C.c_int, C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_vec_inf_norm": ([_dp, C.c_int64, C.c_int, C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_transfer_plan": ([_gp, _gp, _dp, _dp], C.c_int),
    "mfreg_cu_discrete_gradient": ([_gp, _dp, _dp, C.c_int64, _dp, C.c_int], C.c_int),
    "mfreg_cu_eps_norm": ([_dp, C.c_int64, C.c_double, _dp, C.c_int], C.c_int),
    "mfreg_cu_laplacian_at": ([_gp, _dp, _dp, C.c_int64, _dp, C.c_int], C.c_int),
    "mfreg_cu_nodal_interpolate": ([_gp, _dp, _dp, C.c_int64, _dp, C.c_int], C.c_int),
    "mfreg_cu_ngf_precomp": ([_dp, _gp, C.c_double, _dp, _dp, C.c_int], C.c_int),
    "mfreg_cu_ngf_tpl_grads": ([_vp, _dp, C.c_int], C.c_int),
    "mfreg_cu_offset_table": ([_gp, C.POINTER(C.c_int), _dp, _dp, _dp], C.c_int),
    "mfreg_cu_armijo_search": ([C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_problem_minimize": ([C.c_void_p, C.c_int64, C.c_int, _dp, C.POINTER(_OptConfig), _dp,
                                   C.POINTER(_IterRecord), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int],
                                  C.c_int),
    "mfreg_cu_comm_nccl_unique_id": ([C.c_void_p], C.c_int),
    "mfreg_cu_comm_create_nccl": ([C.c_void_p, C.c_int, C.c_int, C.POINTER(_vp)], C.c_int),
    "mfreg_cu_comm_create_local": ([C.c_int, C.POINTER(_vp)], C.c_int),
    "mfreg_cu_comm_destroy": ([_vp], C.c_int),
    "mfreg_cu_comm_rank": ([_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "mfreg_cu_slab_create": ([_vp, _dp, _dp, _gp, _gp, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                              C.POINTER(_vp)], C.c_int),
    "mfreg_cu_slab_destroy": ([_vp], C.c_int),
    "mfreg_cu_slab_info": ([_vp, C.POINTER(C.c_int32)], C.c_int),
    "mfreg_cu_slab_identity": ([_vp, _dp], C.c_int),
    "mfreg_cu_slab_eval": ([_vp, _dp, _dp, C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_slab_last": ([_vp, C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_slab_gn_hessian_vec": ([_vp, _dp, _dp], C.c_int),
    "mfreg_cu_slab_dot": ([_vp, _dp, _dp, C.POINTER(C.c_double)], C.c_int),
    "mfreg_cu_slab_gather": ([_vp, _dp], C.c_int),
    "mfreg_cu_slab_minimize": ([_vp, C.c_int, _dp, C.POINTER(_OptConfig), _dp, C.POINTER(_IterRecord), C.c_int,
                                C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "mfreg_cu_slab_register_multilevel": ([_vp, _dp, _dp, _gp, C.POINTER(_MlConfig), _dp, _gp, C.POINTER(_IterRecord),
                                           C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int], C.c_int),
    "mfreg_cu_problem_cg_solve": ([C.c_void_p, C.c_int64, C.c_int, C.c_double, _dp, C.c_int, C.c_double, _dp,
                                   C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_int], C.c_int),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded libmfreg_cuda.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"CUDA extension missing: {_LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(_LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


_FNS: dict = {}


def _lib_fn(name: str):
    """Cached ctypes function object (hot-path calls skip the attribute lookup)."""
    fn = _FNS.get(name)
    if fn is None:
        fn = _FNS[name] = getattr(lib(), name)
    return fn


def exported_symbols() -> list[str]:
    return list(_SIGS)


def device_memory_peak(reset: bool = False) -> int:
    """High-water mark (bytes) of the library's device allocations since load / the last reset."""
    v = C.c_int64()
    _check(lib().mfreg_cu_device_memory_peak(1 if reset else 0, C.byref(v)))
    return v.value


def launch_count() -> int:
    return int(lib().mfreg_cu_launch_count())


class CudaError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc:
        msg = lib().mfreg_cu_last_error().decode()
        if rc == 1:
            raise ValueError(msg)  # std::invalid_argument
        if rc == 3:
            raise CudaError(msg)
        raise RuntimeError(msg)  # std::logic_error / other


# ------------------------------------------------------------------ arrays
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(x):
    """(pointer, where) for a numpy array or a CUDA torch tensor (fp64, contiguous)."""
    if x is None:
        return None, HOST
    if _F64 is not None and getattr(x, "dtype", None) is _F64 and x.is_cuda and x.is_contiguous():
        return x.data_ptr(), DEVICE  # fast path
    if _is_torch(x):
        import torch
        if x.dtype != torch.float64 or not x.is_contiguous():
            raise ValueError("tensors must be contiguous float64")
        if not x.is_cuda:
            return _ptr(x.numpy())
        return x.data_ptr(), DEVICE
    a = x
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]):
        raise ValueError("arrays must be contiguous float64 numpy arrays or CUDA tensors")
    return a.ctypes.data, HOST


def _empty_like_kind(ref, n: int):
    if ref is not None and _is_torch(ref) and ref.is_cuda:
        import torch
        return torch.empty(n, dtype=torch.float64, device=ref.device)
    return np.empty(n, dtype=np.float64)


_F64 = None


def _as_input(x, where: int):
    """Make `x` match the location `where` (numpy for host, CUDA tensor for device)."""
    global _F64
    if where == DEVICE:
        if _F64 is None:
            import torch
            _F64 = torch.float64
        if x.dtype is _F64 and x.is_cuda and x.is_contiguous():  # fast path: already a CUDA fp64 tensor
            return x
        import torch
        if _is_torch(x):
            return x.to(device="cuda", dtype=torch.float64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    if _is_torch(x):
        return x.detach().cpu().numpy().astype(np.float64, copy=False)
    return np.ascontiguousarray(x, dtype=np.float64)


def _dev_f64(x) -> bool:
    """x is a contiguous CUDA float64 torch tensor (checked without importing torch)."""
    return _F64 is not None and getattr(x, "dtype", None) is _F64 and x.is_cuda and x.is_contiguous()


def _numel(x) -> int:
    return int(x.numel()) if _is_torch(x) else int(np.asarray(x).size)


def _need(x, n: int, msg: str) -> None:
    """Length check with the reference's std::invalid_argument text (raised as ValueError)."""
    if x is not None and _numel(x) != n:
        raise ValueError(msg)


def _same_side(*xs) -> int:
    """All operands host, or all CUDA tensors: a mixed call would hand a host pointer to a
    device kernel (or the reverse)."""
    ws = {_where_of(x) for x in xs if x is not None}
    if len(ws) > 1:
        raise ValueError("operands must all be host arrays or all CUDA tensors")
    return ws.pop() if ws else HOST


def _where_of(*xs) -> int:
    for x in xs:
        if x is not None and _is_torch(x) and x.is_cuda:
            return DEVICE
    return HOST


# ------------------------------------------------------------------ grids
@dataclasses.dataclass(frozen=True)
class GridDesc:
    """mfreg::GridDesc (grid.hpp:50-120)."""

    m: tuple
    h: tuple = (1.0, 1.0, 1.0)
    nodal: bool = False

    def count(self) -> int:
        return int(self.m[0] * self.m[1] * self.m[2])

    def cell_volume(self) -> float:
        return self.h[0] * self.h[1] * self.h[2]

    def extent(self, a: int) -> float:
        return (self.m[a] - 1) * self.h[a] if self.nodal else self.m[a] * self.h[a]

    def c(self) -> _Grid:
        return _Grid((C.c_int64 * 3)(*[int(v) for v in self.m]), (C.c_double * 3)(*[float(v) for v in self.h]))

    def point_coords(self):
        """All grid points, component-major (grid.hpp:91-101)."""
        ax = [(np.arange(self.m[a]) + (0.0 if self.nodal else 0.5)) * self.h[a] for a in range(3)]
        z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
        return np.concatenate([x.ravel(), y.ravel(), z.ravel()])


def make_image_grid(m: Sequence[int], h: Sequence[float] = (1.0, 1.0, 1.0)) -> GridDesc:
    g = GridDesc(tuple(int(v) for v in m), tuple(float(v) for v in h), False)
    for a in range(3):
        if g.m[a] < 1:
            raise ValueError("GridDesc: all m components must be >= 1")
        if not g.h[a] > 0.0:
            raise ValueError("GridDesc: all h components must be > 0")
    return g


def make_deform_grid(image: GridDesc, points: Sequence[int]) -> GridDesc:
    out = _Grid()
    _check(lib().mfreg_cu_make_deform_grid(C.byref(image.c()), (C.c_int64 * 3)(*[int(p) for p in points]),
                                           C.byref(out)))
    return GridDesc(tuple(out.m), tuple(out.h), True)


def deformation_grid_for(image: GridDesc, ratio: int) -> GridDesc:
    out = _Grid()
    _check(lib().mfreg_cu_deformation_grid_for(C.byref(image.c()), int(ratio), C.byref(out)))
    return GridDesc(tuple(out.m), tuple(out.h), True)


def _nodal(g: GridDesc) -> GridDesc:
    return g if g.nodal else GridDesc(g.m, g.h, True)


# ------------------------------------------------------------------ kernel API
def transfer_apply(nodal: GridDesc, image: GridDesc, y):
    """P y (transfer.cpp:49-86)."""
    _need(y, 3 * nodal.count(), "transfer_apply: length mismatch")
    w = _where_of(y)
    y = _as_input(y, w)
    out = _empty_like_kind(y, 3 * image.count())
    _check(lib().mfreg_cu_transfer_apply(C.byref(nodal.c()), C.byref(image.c()), _ptr(y)[0], _ptr(out)[0], w))
    return out


def transfer_apply_transpose(nodal: GridDesc, image: GridDesc, w_img):
    """P^T w (transfer.cpp:131-150), deterministic gather in the reference's order."""
    _need(w_img, 3 * image.count(), "transfer_apply_transpose: length mismatch")
    w = _where_of(w_img)
    w_img = _as_input(w_img, w)
    out = _empty_like_kind(w_img, 3 * nodal.count())
    _check(lib().mfreg_cu_transfer_apply_transpose(C.byref(nodal.c()), C.byref(image.c()), _ptr(w_img)[0],
                                                   _ptr(out)[0], w))
    return out


def sample_deformed(tpl, image: GridDesc, points):
    """T(points) and dT/dP (volume.cpp:76-94). Returns (values, partials[3n])."""
    if _numel(points) % 3:
        raise ValueError("sample_deformed: points length must be a multiple of 3")
    _need(tpl, image.count(), "sample_deformed: template length mismatch")
    w = _where_of(tpl, points)
    tpl, points = _as_input(tpl, w), _as_input(points, w)
    n = _numel(points) // 3
    vals, parts = _empty_like_kind(points, n), _empty_like_kind(points, 3 * n)
    _check(lib().mfreg_cu_sample_deformed(C.byref(image.c()), _ptr(tpl)[0], _ptr(points)[0], n, _ptr(vals)[0],
                                          _ptr(parts)[0], w))
    return vals, parts


def downsample(v, image: GridDesc):
    """Block-mean halving (volume.cpp:123-160). Returns (data, coarse grid)."""
    _need(v, image.count(), "downsample: volume length mismatch")
    w = _where_of(v)
    v = _as_input(v, w)
    og = _Grid()
    _check(lib().mfreg_cu_downsample(C.byref(image.c()), None, None, C.byref(og), w))
    cg = GridDesc(tuple(og.m), tuple(og.h), False)
    out = _empty_like_kind(v, cg.count())
    _check(lib().mfreg_cu_downsample(C.byref(image.c()), _ptr(v)[0], _ptr(out)[0], None, w))
    return out, cg


def prolong(y_coarse, coarse: GridDesc, fine: GridDesc):
    """Displacement prolongation (multilevel.cpp:78-115)."""
    _need(y_coarse, 3 * coarse.count(), "prolong: field length mismatch")
    w = _where_of(y_coarse)
    y_coarse = _as_input(y_coarse, w)
    out = _empty_like_kind(y_coarse, 3 * fine.count())
    _check(lib().mfreg_cu_prolong(C.byref(coarse.c()), C.byref(fine.c()), _ptr(y_coarse)[0], _ptr(out)[0], w))
    return out


def laplacian_apply(u_comp, g: GridDesc):
    _need(u_comp, g.count(), "laplacian_apply: length mismatch")
    w = _where_of(u_comp)
    u_comp = _as_input(u_comp, w)
    out = _empty_like_kind(u_comp, g.count())
    _check(lib().mfreg_cu_laplacian_apply(C.byref(g.c()), _ptr(u_comp)[0], _ptr(out)[0], w))
    return out


def curvature_value(u, g: GridDesc, mode: int = PARITY) -> float:
    _need(u, 3 * g.count(), "curvature_value: length must be 3*m^y")
    w = _where_of(u)
    u = _as_input(u, w)
    v = C.c_double()
    _check(lib().mfreg_cu_curvature_value(C.byref(g.c()), _ptr(u)[0], C.byref(v), int(mode), w))
    return v.value


def curvature_gradient(u, g: GridDesc):
    _need(u, 3 * g.count(), "curvature: buffer length mismatch")
    w = _where_of(u)
    u = _as_input(u, w)
    out = _empty_like_kind(u, 3 * g.count())
    _check(lib().mfreg_cu_curvature_gradient(C.byref(g.c()), _ptr(u)[0], _ptr(out)[0], w))
    return out


def curvature_hessian_vec(p, g: GridDesc):
    _need(p, 3 * g.count(), "curvature: buffer length mismatch")
    w = _where_of(p)
    p = _as_input(p, w)
    out = _empty_like_kind(p, 3 * g.count())
    _check(lib().mfreg_cu_curvature_hessian_vec(C.byref(g.c()), _ptr(p)[0], _ptr(out)[0], w))
    return out


@dataclasses.dataclass
class NgfParams:
    """mfreg::NgfParams (ngf.hpp:14-17)."""

    tau: float = 10.0
    rho: float = 10.0


class NgfContext:
    """make_ngf_precomp + NgfWorkspace + the NGF kernels (ngf.hpp:26-85), on the GPU."""

    def __init__(self, reference, image: GridDesc, params: NgfParams = NgfParams(), mode: int = PARITY):
        self.image = image
        self.n = image.count()
        if mode == Mode.FAST32:
            raise ValueError("NGF kernel API: FAST32 is an Objective mode (the kernel-level NGF API is fp64)")
        _need(reference, self.n, "NGF: reference length mismatch")
        w = _where_of(reference)
        reference = _as_input(reference, w)
        h = _vp()
        _check(lib().mfreg_cu_ngf_create(_ptr(reference)[0], C.byref(image.c()), float(params.tau), float(params.rho),
                                         int(mode), w, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            lib().mfreg_cu_ngf_destroy(self._h)
            self._h = None

    def populate(self, tpl, points) -> None:
        """populate_ngf_workspace (ngf.cpp:185-214)."""
        _need(tpl, self.n, "NGF: template length mismatch")
        _need(points, 3 * self.n, "transfer_apply: length mismatch")
        w = _same_side(tpl, points)
        tpl, points = _as_input(tpl, w), _as_input(points, w)
        _check(lib().mfreg_cu_ngf_populate(self._h, _ptr(tpl)[0], _ptr(points)[0], w))

    def value(self) -> float:
        v = C.c_double()
        _check(lib().mfreg_cu_ngf_value(self._h, C.byref(v)))
        return v.value

    def gradient(self, like=None):
        out = _empty_like_kind(like, 3 * self.n)
        p, w = _ptr(out)
        _check(lib().mfreg_cu_ngf_gradient(self._h, p, w))
        return out

    def hessian_vec(self, p):
        _need(p, 3 * self.n, "ngf_hessian_vec: vector length must be 3*m")
        w = _where_of(p)
        p = _as_input(p, w)
        out = _empty_like_kind(p, 3 * self.n)
        _check(lib().mfreg_cu_ngf_hessian_vec(self._h, _ptr(p)[0], _ptr(out)[0], w))
        return out

    def workspace(self) -> dict:
        n = self.n
        d = {k: np.empty(s * n) for k, s in [("values", 1), ("partials", 3), ("residual", 1), ("inv1", 1),
                                               ("inv2", 1), ("rho_hat", 7)]}
        _check(lib().mfreg_cu_ngf_workspace(self._h, *[d[k].ctypes.data for k in
                                                        ["values", "partials", "residual", "inv1", "inv2",
                                                         "rho_hat"]], HOST))
        return d


@dataclasses.dataclass
class OptimizerConfig:
    """mfreg::OptimizerConfig (optimizer.hpp:145-155), identical defaults."""

    max_iters: int = 20
    c1: float = 1e-4
    beta: float = 0.5
    max_backtracks: int = 10
    cg_max_iters: int = 50
    cg_rel_tol: float = 1e-2
    h0_max_iters: int = 20
    h0_rel_tol: float = 1e-2
    lbfgs_history: int = 5
    gamma: float = -1.0
    tol_rel_j: float = 1e-4
    tol_grad: float = 1e-4
    tol_step: float = 1e-3

    def c(self) -> _OptConfig:
        return _OptConfig(*[getattr(self, f[0]) for f in _OptConfig._fields_])


@dataclasses.dataclass
class IterationRecord:
    """mfreg::IterationRecord (optimizer.hpp:22-30)."""

    iter: int
    cg_iters: int
    j: float
    distance: float
    regularizer: float
    grad_norm: float
    step: float

    def as_tuple(self):
        return (self.iter, self.cg_iters, self.j, self.distance, self.regularizer, self.grad_norm, self.step)


def _records(buf, n) -> list:
    return [IterationRecord(r.iter, r.cg_iters, r.j, r.distance, r.regularizer, r.grad_norm, r.step)
            for r in buf[:n]]


class Objective:
    """mfreg::Objective (optimizer.hpp:53-106): J(y) = D_NGF(P y) + alpha S_curv(y) on the GPU.

    `gn_hessian_vec` / `last_*` refer to the most recent `eval` (value-only or not),
    as in the reference (optimizer.cpp:68-70,96).
    """

    def __init__(self, reference, tpl, image: GridDesc, deform: GridDesc, params: NgfParams = NgfParams(),
                 alpha: float = 1.0, mode: int = PARITY):
        self.image, self.deform, self.params, self._alpha, self.mode = image, _nodal(deform), params, alpha, mode
        _need(reference, image.count(), "Objective: reference length mismatch")
        _need(tpl, image.count(), "Objective: template length mismatch")
        w = _same_side(reference, tpl)
        reference, tpl = _as_input(reference, w), _as_input(tpl, w)
        h = _vp()
        _check(lib().mfreg_cu_objective_create(_ptr(reference)[0], _ptr(tpl)[0], C.byref(image.c()),
                                               C.byref(self.deform.c()), float(params.tau), float(params.rho),
                                               float(alpha), int(mode), w, C.byref(h)))
        self._h = h
        d = C.c_int64()
        _check(lib().mfreg_cu_objective_dof(self._h, C.byref(d)))
        self._dof = d.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            lib().mfreg_cu_objective_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def dof(self) -> int:
        return self._dof

    def alpha(self) -> float:
        return self._alpha

    def min_spacing(self) -> float:
        v = C.c_double()
        _check(lib().mfreg_cu_objective_min_spacing(self._h, C.byref(v)))
        return v.value

    def identity(self, like=None):
        out = _empty_like_kind(like, self._dof)
        p, w = _ptr(out)
        _check(lib().mfreg_cu_objective_identity(self._h, p, w))
        return out

    def eval(self, y, grad=None) -> float:
        """J(y); fills `grad` (same kind as y, length dof) when given."""
        _need(y, self._dof, "Objective::eval: y length mismatch")
        _need(grad, self._dof, "Objective::eval: grad length mismatch")
        if _dev_f64(y) and (grad is None or _dev_f64(grad)):  # direct path: CUDA fp64 contiguous tensors
            j = C.c_double()
            rc = _lib_fn("mfreg_cu_objective_eval")(self._h, y.data_ptr(), grad.data_ptr() if grad is not None else None,
                                                    DEVICE, C.byref(j))
            if rc:
                _check(rc)
            return j.value
        w = _same_side(y, grad)
        yy = _as_input(y, w)
        j = C.c_double()
        rc = _lib_fn("mfreg_cu_objective_eval")(self._h, _ptr(yy)[0], _ptr(grad)[0] if grad is not None else None, w,
                                                C.byref(j))
        if rc:
            _check(rc)
        return j.value

    def last_distance(self) -> float:
        d, r = C.c_double(), C.c_double()
        _check(lib().mfreg_cu_objective_last(self._h, C.byref(d), C.byref(r)))
        return d.value

    def last_regularizer(self) -> float:
        d, r = C.c_double(), C.c_double()
        _check(lib().mfreg_cu_objective_last(self._h, C.byref(d), C.byref(r)))
        return r.value

    def gn_hessian_vec(self, p, q=None):
        _need(p, self._dof, "transfer_apply: length mismatch")
        _need(q, self._dof, "transfer_apply_transpose: length mismatch")
        if q is not None and _dev_f64(p) and _dev_f64(q):  # direct path: CUDA fp64 contiguous tensors
            rc = _lib_fn("mfreg_cu_objective_gn_hessian_vec")(self._h, p.data_ptr(), q.data_ptr(), DEVICE)
            if rc:
                _check(rc)
            return q
        w = _same_side(p, q)
        p = _as_input(p, w)
        q = _empty_like_kind(p, self._dof) if q is None else q
        rc = _lib_fn("mfreg_cu_objective_gn_hessian_vec")(self._h, _ptr(p)[0], _ptr(q)[0], w)
        if rc:
            _check(rc)
        return q

    def profile_kernel(self, which: int, operand, reps: int = 10, flush_bytes: int = 256 << 20) -> float:
        """Average device ms of one fast-mode image-pass kernel (0 Hv, 1 eval, 2 warp),
        CUDA events recorded on the launching stream inside the library (bench support)."""
        ms = C.c_double(0.0)
        _check(lib().mfreg_cu_objective_profile_kernel(self._h, int(which), _ptr(operand)[0], int(reps),
                                                         int(flush_bytes), C.byref(ms)))
        return ms.value

    def seed_hessian_vec(self, p, gamma: float, q=None):
        _need(p, self._dof, "curvature: buffer length mismatch")
        _need(q, self._dof, "curvature: buffer length mismatch")
        w = _same_side(p, q)
        p = _as_input(p, w)
        q = _empty_like_kind(p, self._dof) if q is None else q
        _check(lib().mfreg_cu_objective_seed_hessian_vec(self._h, _ptr(p)[0], float(gamma), _ptr(q)[0], w))
        return q

    def dot(self, a, b) -> float:
        """vec_dot (optimizer.cpp:12-19) over the dof this objective owns."""
        _need(a, self._dof, "vec_dot: length mismatch")
        _need(b, self._dof, "vec_dot: length mismatch")
        w = _same_side(a, b)
        a, b = _as_input(a, w), _as_input(b, w)
        v = C.c_double()
        _check(lib().mfreg_cu_objective_dot(self._h, _ptr(a)[0], _ptr(b)[0], w, C.byref(v)))
        return v.value


def cg_solve(obj: Objective, b, max_iters: int = 50, rel_tol: float = 1e-2, seed: bool = False, gamma: float = 0.0):
    """cg_solve (optimizer.cpp:113-154) on obj's GN operator (or the seed operator). Returns (x, iters, relres, breakdown)."""
    _need(b, obj.dof(), "cg_solve: length mismatch")
    w = _where_of(b)
    b = _as_input(b, w)
    x = _empty_like_kind(b, obj.dof())
    it, br, rr = C.c_int(), C.c_int(), C.c_double()
    _check(lib().mfreg_cu_cg_solve(obj.handle, 1 if seed else 0, float(gamma), _ptr(b)[0], int(max_iters),
                                   float(rel_tol), _ptr(x)[0], C.byref(it), C.byref(rr), C.byref(br), w))
    return x, it.value, rr.value, bool(br.value)


def _minimize(obj: Objective, y0, cfg: OptimizerConfig | None, method: int):
    cfg = cfg or OptimizerConfig()
    _need(y0, obj.dof(), "Objective::eval: y length mismatch")
    w = _where_of(y0)
    y0 = _as_input(y0, w)
    y = _empty_like_kind(y0, obj.dof())
    cap = max(64, 4 * cfg.max_iters + 8)
    tr = (_IterRecord * cap)()
    nt, lsf = C.c_int(), C.c_int()
    oc = cfg.c()
    _check(lib().mfreg_cu_minimize(obj.handle, method, _ptr(y0)[0], C.byref(oc), _ptr(y)[0], tr, cap, C.byref(nt),
                                   C.byref(lsf), w))
    return y, _records(tr, min(nt.value, cap)), bool(lsf.value)


def lbfgs_minimize(obj: Objective, y0, cfg: OptimizerConfig | None = None):
    """lbfgs_minimize (optimizer.cpp:272-390). Returns (y, trace, line_search_failed)."""
    return _minimize(obj, y0, cfg, Method.LBFGS)


def gauss_newton_minimize(obj: Objective, y0, cfg: OptimizerConfig | None = None):
    """gauss_newton_minimize (optimizer.cpp:392-407). Returns (y, trace, line_search_failed)."""
    return _minimize(obj, y0, cfg, Method.GAUSS_NEWTON)


@dataclasses.dataclass
class MultilevelConfig:
    """mfreg::MultilevelConfig (multilevel.hpp:38-45) + execution mode."""

    levels: int = 3
    deform_ratio: int = 4
    ngf: NgfParams = dataclasses.field(default_factory=NgfParams)
    alpha: float = 1.0
    method: int = Method.LBFGS
    opt: OptimizerConfig = dataclasses.field(default_factory=OptimizerConfig)
    mode: int = PARITY


def register_multilevel(reference, tpl, image: GridDesc, cfg: MultilevelConfig | None = None):
    """register_multilevel (multilevel.cpp:117-145). Returns (y, deform_grid, per-level (traces, line_search_failed))."""
    cfg = cfg or MultilevelConfig()
    _need(reference, image.count(), "build_pyramid: image sizes differ")
    _need(tpl, image.count(), "build_pyramid: image sizes differ")
    w = _same_side(reference, tpl)
    reference, tpl = _as_input(reference, w), _as_input(tpl, w)
    dg = deformation_grid_for(image, cfg.deform_ratio)
    y = _empty_like_kind(reference, 3 * dg.count())
    mc = _MlConfig(int(cfg.levels), int(cfg.deform_ratio), float(cfg.ngf.tau), float(cfg.ngf.rho), float(cfg.alpha),
                   int(cfg.method), int(cfg.mode), cfg.opt.c())
    cap = max(64, cfg.levels * (cfg.opt.max_iters + 2))
    tr = (_IterRecord * cap)()
    li = (C.c_int * cfg.levels)()
    lsf = (C.c_int * cfg.levels)()
    og = _Grid()
    _check(lib().mfreg_cu_register_multilevel(_ptr(reference)[0], _ptr(tpl)[0], C.byref(image.c()), C.byref(mc),
                                              _ptr(y)[0], C.byref(og), tr, cap, li, lsf, w))
    levels, off = [], 0
    for l in range(cfg.levels):
        levels.append((_records(tr[off:off + li[l]], li[l]), bool(lsf[l])))
        off += li[l]
    return y, GridDesc(tuple(og.m), tuple(og.h), True), levels


def make_phantom(image: GridDesc, device: bool = False):
    """synthetic::make_phantom (synthetic.cpp:15-63), generated on the GPU."""
    if device:
        import torch
        out = torch.empty(image.count(), dtype=torch.float64, device="cuda")
    else:
        out = np.empty(image.count())
    p, w = _ptr(out)
    _check(lib().mfreg_cu_make_phantom(C.byref(image.c()), p, w))
    return out


def warp_sinusoid(vol, image: GridDesc, max_amp: float, seed: int):
    """warp_with(vol, make_sinusoid_warp(extent, max_amp, seed)) (synthetic.cpp:110-159), on the GPU."""
    w = _where_of(vol)
    vol = _as_input(vol, w)
    out = _empty_like_kind(vol, image.count())
    _check(lib().mfreg_cu_warp_sinusoid(C.byref(image.c()), _ptr(vol)[0], float(max_amp), C.c_uint64(seed),
                                        _ptr(out)[0], w))
    return out

from . import slab  # noqa: E402  (z-slab decomposition, multi-GPU)
from . import io  # noqa: E402  (volume / deformation / landmark files)
