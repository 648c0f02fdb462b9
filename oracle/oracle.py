"""TEST INFRASTRUCTURE ONLY — ctypes front end for the CPU checkers.

Two interchangeable back ends with the same symbol set:
  * ``ref``  — oracle/_ref/libmfreg_ref.so: the UNMODIFIED reference library
    (/root/reference/proj/src) compiled by oracle/Makefile, wrapped by
    oracle/ref_capi.cpp (prefix ``mref_``).
  * ``port`` — oracle/liboracle.so: the plain-C restatement in
    oracle/mfreg_oracle.c (prefix ``mport_``), pinned bitwise against ``ref``
    and the golden fixtures in tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
``--impl reference`` leg may import this module. It is the checker, never the
product: the product path (paper_1804_10541_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmfreg_ref.so")
PORT_SO = os.path.join(HERE, "liboracle.so")

_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class OptConfig(C.Structure):
    """mfreg::OptimizerConfig (optimizer.hpp:145-155), defaults identical."""

    _fields_ = [
        ("max_iters", C.c_int),
        ("c1", C.c_double),
        ("beta", C.c_double),
        ("max_backtracks", C.c_int),
        ("cg_max_iters", C.c_int),
        ("cg_rel_tol", C.c_double),
        ("h0_max_iters", C.c_int),
        ("h0_rel_tol", C.c_double),
        ("lbfgs_history", C.c_int),
        ("gamma", C.c_double),
        ("tol_rel_j", C.c_double),
        ("tol_grad", C.c_double),
        ("tol_step", C.c_double),
    ]

    @classmethod
    def defaults(cls, **kw):
        c = cls(20, 1e-4, 0.5, 10, 50, 1e-2, 20, 1e-2, 5, -1.0, 1e-4, 1e-4, 1e-3)
        for k, v in kw.items():
            setattr(c, k, v)
        return c


class IterRecord(C.Structure):
    """mfreg::IterationRecord (optimizer.hpp:22-30)."""

    _fields_ = [
        ("iter", C.c_int),
        ("cg_iters", C.c_int),
        ("j", C.c_double),
        ("distance", C.c_double),
        ("regularizer", C.c_double),
        ("grad_norm", C.c_double),
        ("step", C.c_double),
    ]

    def as_tuple(self):
        return (self.iter, self.cg_iters, self.j, self.distance, self.regularizer, self.grad_norm, self.step)


def _arr_i64(v):
    return (C.c_int64 * 3)(*[int(x) for x in v])


def _arr_d(v):
    return (C.c_double * 3)(*[float(x) for x in v])


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def build(ref: bool = True) -> None:
    """Compile the checker(s) with oracle/Makefile (port always, ref when the reference tree exists)."""
    targets = ["port"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def available(kind: str) -> bool:
    return os.path.exists(REF_SO if kind == "ref" else PORT_SO)


class Oracle:
    """One CPU checker back end ("ref" or "port")."""

    def __init__(self, kind: str = "ref"):
        self.kind = kind
        path = REF_SO if kind == "ref" else PORT_SO
        self.pre = "mref_" if kind == "ref" else "mport_"
        self.lib = C.CDLL(path)
        L = self.lib
        f = self._f
        f("last_error").restype = C.c_char_p
        f("set_threads").argtypes = [C.c_int]
        f("set_threads").restype = None
        f("thread_count").restype = C.c_int
        for name, args in {
            "make_phantom": [_i64p, _dp, _dp],
            "make_random_volume": [_i64p, _dp, C.c_uint64, C.c_int, _dp],
            "sinusoid_terms": [_dp, C.c_double, C.c_uint64, _dp, _ip, _dp],
            "warp_sinusoid": [_dp, _i64p, _dp, C.c_double, C.c_uint64, _dp],
            "warp_field": [_i64p, _dp, C.c_double, C.c_uint64, _i64p, _dp],
            "make_deform_grid": [_i64p, _dp, _i64p, _dp],
            "deformation_grid_for": [_i64p, _dp, C.c_int64, _i64p, _dp],
            "transfer_plan": [_i64p, _dp, _i64p, _dp, _i64p, _dp],
            "transfer_apply": [_i64p, _dp, _i64p, _dp, _dp, _dp],
            "transfer_apply_transpose": [_i64p, _dp, _i64p, _dp, _dp, _dp],
            "interpolate": [_dp, _i64p, _dp, _dp, _dp, _dp],
            "sample_deformed": [_dp, _i64p, _dp, _dp, C.c_int64, _dp, _dp],
            "downsample": [_dp, _i64p, _dp, _dp, _i64p, _dp],
            "ngf_populate": [C.c_void_p, _dp, _dp],
            "ngf_workspace": [C.c_void_p] + [_dp] * 8,
            "ngf_value": [C.c_void_p, _dp],
            "ngf_gradient": [C.c_void_p, _dp],
            "ngf_hessian_vec": [C.c_void_p, _dp, _dp],
            "ngf_rho": [C.c_void_p, C.c_int64, C.c_int, _dp],
            "laplacian_apply": [_dp, _i64p, _dp, _dp],
            "curvature_value": [_dp, _i64p, _dp, _dp],
            "curvature_gradient": [_dp, _i64p, _dp, _dp],
            "curvature_hessian_vec": [_dp, _i64p, _dp, _dp],
            "objective_identity": [C.c_void_p, _dp],
            "objective_eval": [C.c_void_p, _dp, _dp, _dp, _dp, _dp],
            "objective_gn_hessian_vec": [C.c_void_p, _dp, _dp],
            "objective_seed_hessian_vec": [C.c_void_p, _dp, C.c_double, _dp],
            "cg_solve": [C.c_void_p, C.c_int, C.c_double, _dp, C.c_int, C.c_double, _dp, _ip, _dp, _ip],
            "minimize": [C.c_void_p, C.c_int, _dp, C.POINTER(OptConfig), _dp, C.POINTER(IterRecord), C.c_int, _ip, _ip],
            "prolong": [_dp, _i64p, _dp, _i64p, _dp, _dp],
            "register_multilevel": [_dp, _dp, _i64p, _dp, C.c_int, C.c_int64, C.c_double, C.c_double, C.c_double,
                                    C.c_int, C.POINTER(OptConfig), _dp, C.POINTER(IterRecord), C.c_int, _ip, _ip],
        }.items():
            fn = f(name)
            fn.argtypes = args
            fn.restype = C.c_int
        f("ngf_create").argtypes = [_dp, _i64p, _dp, C.c_double, C.c_double]
        f("ngf_create").restype = C.c_void_p
        f("ngf_destroy").argtypes = [C.c_void_p]
        f("ngf_destroy").restype = None
        f("objective_create").argtypes = [_dp, _dp, _i64p, _dp, _i64p, C.c_double, C.c_double, C.c_double]
        f("objective_create").restype = C.c_void_p
        f("objective_destroy").argtypes = [C.c_void_p]
        f("objective_destroy").restype = None
        f("objective_dof").argtypes = [C.c_void_p]
        f("objective_dof").restype = C.c_int64
        if kind == "ref":
            f("oracle_image").argtypes = [C.c_void_p, _i64p, _dp, _dp, _dp]
            f("oracle_image").restype = C.c_int
        del L

    def _f(self, name):
        return getattr(self.lib, self.pre + name)

    def _call(self, name, *args):
        rc = self._f(name)(*args)
        if rc:
            msg = self._f("last_error")().decode()
            raise (ValueError if rc == 1 else RuntimeError)(msg)

    def set_threads(self, n: int) -> None:
        self._f("set_threads")(int(n))

    # ---------------- synthetic inputs
    def make_phantom(self, m, h=(1.0, 1.0, 1.0)) -> np.ndarray:
        out = np.empty(int(np.prod(m)))
        self._call("make_phantom", _arr_i64(m), _arr_d(h), _dptr(out))
        return out

    def make_random_volume(self, m, h, seed, passes=0) -> np.ndarray:
        out = np.empty(int(np.prod(m)))
        self._call("make_random_volume", _arr_i64(m), _arr_d(h), C.c_uint64(seed), int(passes), _dptr(out))
        return out

    def sinusoid_terms(self, extent, amp, seed):
        a = np.empty(9)
        fq = (C.c_int * 9)()
        ph = np.empty(9)
        self._call("sinusoid_terms", _arr_d(extent), float(amp), C.c_uint64(seed), _dptr(a), fq, _dptr(ph))
        return a.reshape(3, 3), np.array(list(fq)).reshape(3, 3), ph.reshape(3, 3)

    def warp_sinusoid(self, vol, m, h, amp, seed) -> np.ndarray:
        vol = np.ascontiguousarray(vol, dtype=np.float64)
        out = np.empty_like(vol)
        self._call("warp_sinusoid", _dptr(vol), _arr_i64(m), _arr_d(h), float(amp), C.c_uint64(seed), _dptr(out))
        return out

    def warp_field(self, m, h, amp, seed, my) -> np.ndarray:
        out = np.empty(3 * int(np.prod(my)))
        self._call("warp_field", _arr_i64(m), _arr_d(h), float(amp), C.c_uint64(seed), _arr_i64(my), _dptr(out))
        return out

    # ---------------- grids / transfer
    def make_deform_grid(self, m, h, my):
        hy = np.empty(3)
        self._call("make_deform_grid", _arr_i64(m), _arr_d(h), _arr_i64(my), _dptr(hy))
        return hy

    def deformation_grid_for(self, m, h, ratio):
        my = (C.c_int64 * 3)()
        hy = np.empty(3)
        self._call("deformation_grid_for", _arr_i64(m), _arr_d(h), int(ratio), my, _dptr(hy))
        return tuple(my), hy

    def transfer_plan(self, ms, hs, mt, ht):
        n = int(sum(mt))
        base = (C.c_int64 * n)()
        rem = np.empty(n)
        self._call("transfer_plan", _arr_i64(ms), _arr_d(hs), _arr_i64(mt), _arr_d(ht), base, _dptr(rem))
        return np.array(list(base), dtype=np.int64), rem

    def transfer_apply(self, ms, hs, mt, ht, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty(3 * int(np.prod(mt)))
        self._call("transfer_apply", _arr_i64(ms), _arr_d(hs), _arr_i64(mt), _arr_d(ht), _dptr(y), _dptr(out))
        return out

    def transfer_apply_transpose(self, ms, hs, mt, ht, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        out = np.empty(3 * int(np.prod(ms)))
        self._call("transfer_apply_transpose", _arr_i64(ms), _arr_d(hs), _arr_i64(mt), _arr_d(ht), _dptr(w), _dptr(out))
        return out

    # ---------------- image
    def interpolate(self, t, m, h, p):
        t = np.ascontiguousarray(t, dtype=np.float64)
        v = np.empty(1)
        g = np.empty(3)
        self._call("interpolate", _dptr(t), _arr_i64(m), _arr_d(h), _arr_d(p), _dptr(v), _dptr(g))
        return v[0], g

    def sample_deformed(self, t, m, h, points):
        t = np.ascontiguousarray(t, dtype=np.float64)
        points = np.ascontiguousarray(points, dtype=np.float64)
        n = points.size // 3
        vals = np.empty(n)
        parts = np.empty(3 * n)
        self._call("sample_deformed", _dptr(t), _arr_i64(m), _arr_d(h), _dptr(points), n, _dptr(vals), _dptr(parts))
        return vals, parts

    def downsample(self, v, m, h):
        v = np.ascontiguousarray(v, dtype=np.float64)
        mo = [(int(x) + 1) // 2 for x in m]
        out = np.empty(int(np.prod(mo)))
        mo_c = (C.c_int64 * 3)()
        ho = np.empty(3)
        self._call("downsample", _dptr(v), _arr_i64(m), _arr_d(h), _dptr(out), mo_c, _dptr(ho))
        return out, tuple(mo_c), ho

    # ---------------- curvature (nodal grid)
    def laplacian_apply(self, u, m, h):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty_like(u)
        self._call("laplacian_apply", _dptr(u), _arr_i64(m), _arr_d(h), _dptr(out))
        return out

    def curvature_value(self, u, m, h):
        u = np.ascontiguousarray(u, dtype=np.float64)
        v = np.empty(1)
        self._call("curvature_value", _dptr(u), _arr_i64(m), _arr_d(h), _dptr(v))
        return v[0]

    def curvature_gradient(self, u, m, h):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty_like(u)
        self._call("curvature_gradient", _dptr(u), _arr_i64(m), _arr_d(h), _dptr(out))
        return out

    def curvature_hessian_vec(self, u, m, h):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty_like(u)
        self._call("curvature_hessian_vec", _dptr(u), _arr_i64(m), _arr_d(h), _dptr(out))
        return out

    def prolong(self, yc, mc, hc, mf, hf):
        yc = np.ascontiguousarray(yc, dtype=np.float64)
        out = np.empty(3 * int(np.prod(mf)))
        self._call("prolong", _dptr(yc), _arr_i64(mc), _arr_d(hc), _arr_i64(mf), _arr_d(hf), _dptr(out))
        return out

    # ---------------- io.hpp (reference library only)
    def io_read_volume(self, path):
        """io::read_volume -> (data, m, h)"""
        m = (C.c_int64 * 3)()
        h = (C.c_double * 3)()
        self._call("io_read_volume", os.fsencode(str(path)), m, h, None)
        out = np.empty(int(m[0] * m[1] * m[2]))
        self._call("io_read_volume", os.fsencode(str(path)), m, h, _dptr(out))
        return out, tuple(int(v) for v in m), tuple(float(v) for v in h)

    def io_write_volume(self, path, data, m, h):
        data = np.ascontiguousarray(data, dtype=np.float64)
        self._call("io_write_volume", os.fsencode(str(path)), _arr_i64(m), _arr_d(h), _dptr(data))

    def io_write_deformation(self, path, y, m, h):
        y = np.ascontiguousarray(y, dtype=np.float64)
        self._call("io_write_deformation", os.fsencode(str(path)), _dptr(y), C.c_int64(y.size), _arr_i64(m), _arr_d(h))

    def io_read_deformation_grid(self, path):
        m = (C.c_int64 * 3)()
        h = (C.c_double * 3)()
        self._call("io_read_deformation_grid", os.fsencode(str(path)), m, h)
        return tuple(int(v) for v in m), tuple(float(v) for v in h)

    def io_read_deformation(self, path, m, h):
        out = np.empty(3 * int(np.prod(m)))
        self._call("io_read_deformation", os.fsencode(str(path)), _arr_i64(m), _arr_d(h), _dptr(out))
        return out

    def io_read_landmarks(self, path, spacing):
        n = C.c_int64()
        self._call("io_read_landmarks", os.fsencode(str(path)), _arr_d(spacing), None, C.c_int64(0), C.byref(n))
        out = np.empty((n.value, 3))
        self._call("io_read_landmarks", os.fsencode(str(path)), _arr_d(spacing), _dptr(out) if n.value else None,
                   C.c_int64(n.value), C.byref(n))
        return out

    def io_landmark_error(self, fixed, moving, y, m, h):
        f = np.ascontiguousarray(np.asarray(fixed, dtype=np.float64).reshape(-1, 3))
        mv = np.ascontiguousarray(np.asarray(moving, dtype=np.float64).reshape(-1, 3))
        y = np.ascontiguousarray(y, dtype=np.float64)
        mean, sd, cnt = C.c_double(), C.c_double(), C.c_int64()
        self._call("io_landmark_error", _dptr(f) if len(f) else None, C.c_int64(len(f)), _dptr(mv) if len(mv) else None,
                   C.c_int64(len(mv)), _dptr(y), C.c_int64(y.size), _arr_i64(m), _arr_d(h), C.byref(mean),
                   C.byref(sd), C.byref(cnt))
        return mean.value, sd.value, cnt.value

    # ---------------- contexts
    def ngf(self, ref, m, h, tau=10.0, rho=10.0) -> "NgfCtx":
        return NgfCtx(self, ref, m, h, tau, rho)

    def objective(self, ref, tpl, m, h, my, tau=10.0, rho=10.0, alpha=1.0) -> "ObjCtx":
        return ObjCtx(self, ref, tpl, m, h, my, tau, rho, alpha)

    def register_multilevel(self, ref, tpl, m, h, levels=3, ratio=4, tau=10.0, rho=10.0, alpha=1.0,
                            method="lbfgs", cfg: OptConfig | None = None):
        ref = np.ascontiguousarray(ref, dtype=np.float64)
        tpl = np.ascontiguousarray(tpl, dtype=np.float64)
        cfg = cfg or OptConfig.defaults()
        my, _ = self.deformation_grid_for(m, h, ratio)
        y = np.empty(3 * int(np.prod(my)))
        cap = 64 * levels + 64
        tr = (IterRecord * cap)()
        li = (C.c_int * levels)()
        lsf = (C.c_int * levels)()
        self._call("register_multilevel", _dptr(ref), _dptr(tpl), _arr_i64(m), _arr_d(h), int(levels), int(ratio),
                   float(tau), float(rho), float(alpha), 1 if method == "gn" else 0, C.byref(cfg), _dptr(y), tr, cap,
                   li, lsf)
        traces, off = [], 0
        for l in range(levels):
            traces.append([tr[off + k].as_tuple() for k in range(li[l])])
            off += li[l]
        return y, my, traces, list(lsf)


class NgfCtx:
    """Reference NGF kernel API (ngf.hpp:26-85) on a fixed reference image."""

    def __init__(self, o: Oracle, ref, m, h, tau, rho):
        self.o = o
        self.m = tuple(int(x) for x in m)
        self.n = int(np.prod(self.m))
        ref = np.ascontiguousarray(ref, dtype=np.float64)
        self.p = o._f("ngf_create")(_dptr(ref), _arr_i64(m), _arr_d(h), float(tau), float(rho))
        if not self.p:
            raise ValueError(o._f("last_error")().decode())

    def __del__(self):
        if getattr(self, "p", None):
            self.o._f("ngf_destroy")(self.p)
            self.p = None

    def populate(self, tpl, points):
        tpl = np.ascontiguousarray(tpl, dtype=np.float64)
        points = np.ascontiguousarray(points, dtype=np.float64)
        self.o._call("ngf_populate", self.p, _dptr(tpl), _dptr(points))

    def workspace(self) -> dict:
        n = self.n
        d = {k: np.empty(s * n) for k, s in [("values", 1), ("partials", 3), ("tpl_grads", 6), ("residual", 1),
                                               ("inv1", 1), ("inv2", 1), ("ref_grads", 6), ("ref_norms", 1)]}
        self.o._call("ngf_workspace", self.p, *[_dptr(d[k]) for k in
                                                 ["values", "partials", "tpl_grads", "residual", "inv1", "inv2",
                                                  "ref_grads", "ref_norms"]])
        return d

    def value(self) -> float:
        v = np.empty(1)
        self.o._call("ngf_value", self.p, _dptr(v))
        return v[0]

    def gradient(self) -> np.ndarray:
        out = np.empty(3 * self.n)
        self.o._call("ngf_gradient", self.p, _dptr(out))
        return out

    def hessian_vec(self, p) -> np.ndarray:
        p = np.ascontiguousarray(p, dtype=np.float64)
        out = np.empty(3 * self.n)
        self.o._call("ngf_hessian_vec", self.p, _dptr(p), _dptr(out))
        return out

    def rho(self, i, k) -> float:
        v = np.empty(1)
        self.o._call("ngf_rho", self.p, int(i), int(k), _dptr(v))
        return v[0]

    def oracle_image(self, my, p):
        """Sparse-matrix chain (oracle.cpp:223-293): (gradient, Hv) on the image grid. ref back end only."""
        p = np.ascontiguousarray(p, dtype=np.float64)
        g = np.empty(3 * self.n)
        hv = np.empty(3 * self.n)
        self.o._call("oracle_image", self.p, _arr_i64(my), _dptr(p), _dptr(g), _dptr(hv))
        return g, hv


class ObjCtx:
    """Reference Objective (optimizer.hpp:53-106) + solvers on it."""

    def __init__(self, o: Oracle, ref, tpl, m, h, my, tau, rho, alpha):
        self.o = o
        self._keep = (np.ascontiguousarray(ref, dtype=np.float64), np.ascontiguousarray(tpl, dtype=np.float64))
        self.p = o._f("objective_create")(_dptr(self._keep[0]), _dptr(self._keep[1]), _arr_i64(m), _arr_d(h),
                                          _arr_i64(my), float(tau), float(rho), float(alpha))
        if not self.p:
            raise ValueError(o._f("last_error")().decode())
        self.dof = int(o._f("objective_dof")(self.p))

    def __del__(self):
        if getattr(self, "p", None):
            self.o._f("objective_destroy")(self.p)
            self.p = None

    def identity(self):
        out = np.empty(self.dof)
        self.o._call("objective_identity", self.p, _dptr(out))
        return out

    def eval(self, y, want_grad=True):
        y = np.ascontiguousarray(y, dtype=np.float64)
        g = np.empty(self.dof) if want_grad else None
        j, dd, rr = np.empty(1), np.empty(1), np.empty(1)
        self.o._call("objective_eval", self.p, _dptr(y), _dptr(g) if want_grad else None, _dptr(j), _dptr(dd), _dptr(rr))
        return j[0], dd[0], rr[0], g

    def gn_hessian_vec(self, p):
        p = np.ascontiguousarray(p, dtype=np.float64)
        q = np.empty(self.dof)
        self.o._call("objective_gn_hessian_vec", self.p, _dptr(p), _dptr(q))
        return q

    def seed_hessian_vec(self, p, gamma):
        p = np.ascontiguousarray(p, dtype=np.float64)
        q = np.empty(self.dof)
        self.o._call("objective_seed_hessian_vec", self.p, _dptr(p), float(gamma), _dptr(q))
        return q

    def cg_solve(self, b, max_iters=50, rel_tol=1e-2, seed=False, gamma=0.0):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.dof)
        it, br = C.c_int(), C.c_int()
        rr = np.empty(1)
        self.o._call("cg_solve", self.p, 1 if seed else 0, float(gamma), _dptr(b), int(max_iters), float(rel_tol),
                     _dptr(x), C.byref(it), _dptr(rr), C.byref(br))
        return x, it.value, rr[0], bool(br.value)

    def minimize(self, y0, method="gn", cfg: OptConfig | None = None):
        y0 = np.ascontiguousarray(y0, dtype=np.float64)
        cfg = cfg or OptConfig.defaults()
        y = np.empty(self.dof)
        cap = 256
        tr = (IterRecord * cap)()
        nt, lsf = C.c_int(), C.c_int()
        self.o._call("minimize", self.p, 1 if method == "gn" else 0, _dptr(y0), C.byref(cfg), _dptr(y), tr, cap,
                     C.byref(nt), C.byref(lsf))
        return y, [tr[k].as_tuple() for k in range(min(nt.value, cap))], bool(lsf.value)
