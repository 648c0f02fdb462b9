"""z-slab decomposition of the objective across processes (SURVEY §8 row e).

The reference runs one address space with OpenMP (parallel.hpp:22-55) and has no
multi-process path; this module is the B200-native scale-out of the same
operators. One process per GPU; the image z axis is split at nodal-cell
boundaries (``slab_partition``, computed natively by ``mfreg_cu_slab_partition``):

* rank r evaluates the image planes [zlo, zhi) (plus 2-3 halo planes of state it
  recomputes from the replicated R / T), i.e. D and the P^T contributions of its
  planes, and owns the nodal planes [own_lo, own_hi) (curvature term, dot products);
* before an operator call the nodal operand (y or p) is made valid on
  [need_lo, need_hi) by a halo exchange with ranks r-1 / r+1 (``SlabExchange.halo``);
* after it, the P^T planes both neighbours touch ([own_hi, own_hi + bnd) of rank r)
  are summed on the owner r+1 (``SlabExchange.boundary``), always as
  own + neighbour (deterministic);
* scalars (D, alpha S, dot products) are all-gathered and added in rank order
  (deterministic, identical on every rank).

The only collectives are these point-to-point plane exchanges and one scalar
all-gather per reduction: no data-path all-reduce. ``TorchComm`` runs them over
``torch.distributed`` (NCCL over NVLink for CUDA tensors, gloo for CPU tensors);
``LoopbackHub`` runs N ranks as threads of one process (single-GPU tests).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import threading
from typing import Sequence

from . import (DEVICE, GridDesc, NgfParams, _as_input, _check, _nodal, _ptr, _vp, _where_of, lib)


@dataclasses.dataclass(frozen=True)
class SlabInfo:
    zlo: int       # image planes [zlo, zhi) evaluated by the rank
    zhi: int
    own_lo: int    # owned nodal planes [own_lo, own_hi)
    own_hi: int
    need_lo: int   # nodal operand planes read [need_lo, need_hi)
    need_hi: int
    bnd: int       # P^T planes [own_hi, own_hi + bnd) shared with rank r+1


def slab_partition(image: GridDesc, deform: GridDesc, nranks: int, mode: int = 1) -> list[SlabInfo]:
    """Split the image z axis over `nranks` ranks (ValueError when the slabs would be
    thinner than the operator halo); `mode` Mode.PARITY widens the operand halo to what the
    parity-mode slabs recompute."""
    tab = (C.c_int32 * (7 * nranks))()
    _check(lib().mfreg_cu_slab_partition_mode(C.byref(image.c()), C.byref(_nodal(deform).c()), int(nranks), int(mode),
                                              tab))
    return [SlabInfo(*tab[7 * r:7 * r + 7]) for r in range(nranks)]


# ------------------------------------------------------------------ communicators
class TorchComm:
    """Plane exchanges and scalar gathers over torch.distributed (any backend)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self._dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        # gloo moves host buffers only: CUDA planes are staged through host memory
        self._stage = dist.get_backend(group) == "gloo"

    def _global(self, r: int) -> int:
        return r if self.group is None else self._dist.get_global_rank(self.group, r)

    def exchange(self, sends, recvs) -> None:
        """sends / recvs: lists of (peer rank, contiguous tensor)."""
        dist = self._dist
        back = []
        if self._stage:
            sends = [(p, t.cpu() if t.is_cuda else t) for p, t in sends]
            staged = []
            for p, t in recvs:
                if t.is_cuda:
                    h = t.cpu()
                    back.append((t, h))
                    staged.append((p, h))
                else:
                    staged.append((p, t))
            recvs = staged
        ops = [dist.P2POp(dist.isend, t, self._global(p), self.group) for p, t in sends]
        ops += [dist.P2POp(dist.irecv, t, self._global(p), self.group) for p, t in recvs]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for t, h in back:
            t.copy_(h)

    def allgather(self, vals: Sequence[float], like) -> list[list[float]]:
        import torch
        t = torch.tensor(list(vals), dtype=torch.float64, device="cpu" if self._stage else like.device)
        out = [torch.empty_like(t) for _ in range(self.size)]
        self._dist.all_gather(out, t, group=self.group)
        return [o.tolist() for o in out]


class LoopbackHub:
    """N ranks as threads of one process sharing one device (tests, single-GPU runs).
    Every rank must issue the same sequence of exchanges / gathers (SPMD)."""

    def __init__(self, n: int):
        self.n = n
        self._bar = threading.Barrier(n)
        self._box: dict = {}

    def comm(self, rank: int) -> "LoopbackComm":
        return LoopbackComm(self, rank)


class LoopbackComm:
    def __init__(self, hub: LoopbackHub, rank: int):
        self.hub, self.rank, self.size = hub, rank, hub.n

    def exchange(self, sends, recvs) -> None:
        box = self.hub._box
        for p, t in sends:
            box[(self.rank, p)] = t
        self.hub._bar.wait()
        for p, t in recvs:
            t.copy_(box[(p, self.rank)])
        self.hub._bar.wait()  # all copies issued before any sender reuses its buffer
        for p, _ in sends:
            box.pop((self.rank, p), None)

    def allgather(self, vals: Sequence[float], like) -> list[list[float]]:
        box = self.hub._box
        box[("g", self.rank)] = list(vals)
        self.hub._bar.wait()
        out = [list(box[("g", r)]) for r in range(self.size)]
        self.hub._bar.wait()
        return out


# ------------------------------------------------------------------ exchange plan
class SlabExchange:
    """Halo exchange / shared-plane assembly / scalar sums for one rank's nodal vectors
    (flat torch tensors of length 3 * deform.count(), component-major, z slowest)."""

    def __init__(self, parts: Sequence[SlabInfo], rank: int, comm, deform: GridDesc):
        self.parts, self.rank, self.comm = list(parts), rank, comm
        self.me = self.parts[rank]
        self.m = tuple(int(v) for v in deform.m)

    def _planes(self, v, lo: int, hi: int):
        mx, my, mz = self.m
        return v.view(3, mz, my, mx)[:, lo:hi]

    def halo(self, v) -> None:
        """Overwrite v's halo planes [need_lo, own_lo) and [own_hi, need_hi) with the owners' values."""
        r, me, P = self.rank, self.me, self.parts
        sends, recvs, fills = [], [], []
        if r > 0:
            lo = P[r - 1]
            if lo.need_hi > me.own_lo:
                sends.append((r - 1, self._planes(v, me.own_lo, lo.need_hi).contiguous()))
            if me.need_lo < me.own_lo:
                buf = self._planes(v, me.need_lo, me.own_lo).contiguous()
                recvs.append((r - 1, buf))
                fills.append((me.need_lo, me.own_lo, buf))
        if r + 1 < len(P):
            up = P[r + 1]
            if up.need_lo < me.own_hi:
                sends.append((r + 1, self._planes(v, up.need_lo, me.own_hi).contiguous()))
            if me.need_hi > me.own_hi:
                buf = self._planes(v, me.own_hi, me.need_hi).contiguous()
                recvs.append((r + 1, buf))
                fills.append((me.own_hi, me.need_hi, buf))
        self.comm.exchange(sends, recvs)
        for lo_, hi_, buf in fills:
            self._planes(v, lo_, hi_).copy_(buf)

    def boundary(self, q) -> None:
        """Add the lower neighbour's P^T contributions to the shared owned planes."""
        r, me, P = self.rank, self.me, self.parts
        sends, recvs = [], []
        if r + 1 < len(P) and me.bnd:
            sends.append((r + 1, self._planes(q, me.own_hi, me.own_hi + me.bnd).contiguous()))
        buf = None
        if r > 0 and P[r - 1].bnd:
            buf = self._planes(q, me.own_lo, me.own_lo + P[r - 1].bnd).contiguous()
            recvs.append((r - 1, buf))
        self.comm.exchange(sends, recvs)
        if buf is not None:
            self._planes(q, me.own_lo, me.own_lo + P[r - 1].bnd).add_(buf)

    def allsum(self, vals: Sequence[float], like) -> list[float]:
        """Sum of `vals` over ranks, added in rank order (same result on every rank)."""
        g = self.comm.allgather(vals, like)
        out = list(g[0])
        for row in g[1:]:
            out = [a + b for a, b in zip(out, row)]
        return out


# ------------------------------------------------------------------ objective
class SlabObjective:
    """One rank's share of mfreg::Objective (optimizer.hpp:53-106) in `fast` mode.

    `reference` / `tpl`: the whole volume (replicated on every rank, device or host).
    Nodal vectors are full-length CUDA tensors of which the rank keeps its owned planes
    valid; `eval` / `gn_hessian_vec` refresh the operand's halo in place and return the
    global J (identical on all ranks) / the result on the owned planes.
    """

    def __init__(self, reference, tpl, image: GridDesc, deform: GridDesc, params: NgfParams = NgfParams(),
                 alpha: float = 1.0, comm=None):
        if comm is None:
            comm = TorchComm()
        self.image, self.deform, self.params, self._alpha, self.comm = image, _nodal(deform), params, alpha, comm
        self.parts = slab_partition(image, self.deform, comm.size)
        self.info = self.parts[comm.rank]
        w = _where_of(reference, tpl)
        reference, tpl = _as_input(reference, w), _as_input(tpl, w)
        s = self.info
        win = (C.c_int32 * 4)(s.zlo, s.zhi, s.own_lo, s.own_hi)
        h = _vp()
        _check(lib().mfreg_cu_objective_create_slab(_ptr(reference)[0], _ptr(tpl)[0], C.byref(image.c()),
                                                    C.byref(self.deform.c()), float(params.tau), float(params.rho),
                                                    float(alpha), win, w, C.byref(h)))
        self._h = h
        self._dof = 3 * self.deform.count()
        self.ex = SlabExchange(self.parts, comm.rank, comm, self.deform)
        self._last = (0.0, 0.0)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().mfreg_cu_objective_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass

    def dof(self) -> int:
        return self._dof

    def alpha(self) -> float:
        return self._alpha

    def identity(self, like):
        import torch
        out = torch.empty(self._dof, dtype=torch.float64, device=like.device)
        _check(lib().mfreg_cu_objective_identity(self._h, out.data_ptr(), DEVICE))
        return out

    @staticmethod
    def _dev(x):
        if _where_of(x) != DEVICE:
            raise ValueError("slab objectives take CUDA tensors")
        return x

    def eval(self, y, grad=None) -> float:
        y = self._dev(y)
        self.ex.halo(y)
        j = C.c_double()
        _check(lib().mfreg_cu_objective_eval(self._h, y.data_ptr(), self._dev(grad).data_ptr() if grad is not None
                                             else None, DEVICE, C.byref(j)))
        d, r = C.c_double(), C.c_double()
        _check(lib().mfreg_cu_objective_last(self._h, C.byref(d), C.byref(r)))
        if grad is not None:
            self.ex.boundary(grad)
        D, S = self.ex.allsum([d.value, r.value], y)
        self._last = (D, S)
        return D + S

    def last_distance(self) -> float:
        return self._last[0]

    def last_regularizer(self) -> float:
        return self._last[1]

    def gn_hessian_vec(self, p, q=None):
        import torch
        p = self._dev(p)
        q = torch.zeros_like(p) if q is None else self._dev(q)
        self.ex.halo(p)
        _check(lib().mfreg_cu_objective_gn_hessian_vec(self._h, p.data_ptr(), q.data_ptr(), DEVICE))
        self.ex.boundary(q)
        return q

    def dot(self, a, b) -> float:
        v = C.c_double()
        _check(lib().mfreg_cu_objective_dot(self._h, self._dev(a).data_ptr(), self._dev(b).data_ptr(), DEVICE,
                                            C.byref(v)))
        return self.ex.allsum([v.value], a)[0]

    def owned(self, v):
        """View of v's owned nodal planes, shape (3, own_hi - own_lo, my, mx)."""
        return self.ex._planes(v, self.info.own_lo, self.info.own_hi)

    def inf_norm(self, a, scale: float = 1.0) -> float:
        """max |scale * a_i| over all ranks' owned planes."""
        v = float((self.owned(a) * scale).abs().max())
        return max(row[0] for row in self.comm.allgather([v], a))

    def min_spacing(self) -> float:
        return min(self.deform.h)


# ------------------------------------------------------------------ distributed solvers
def cg_solve(so: SlabObjective, b, max_iters: int = 50, rel_tol: float = 1e-2):
    """cg_solve (optimizer.cpp:113-154) on the sharded GN operator: x0 = 0, the
    reference's scalar logic (breakdown on non-finite / non-positive <p,Ap>,
    relres = ||r|| / ||b||, beta = rr_new / rr); every dot is a sharded reduction.
    Returns (x, iters, relres, breakdown)."""
    import math

    import torch
    x = torch.zeros_like(b)
    r, p = b.clone(), b.clone()
    rr = so.dot(b, b)
    bnorm = math.sqrt(rr)
    iters, relres, breakdown = 0, 0.0, False
    if bnorm == 0.0:
        return x, iters, relres, breakdown
    ap = torch.zeros_like(b)
    for _ in range(max_iters):
        so.gn_hessian_vec(p, ap)
        pap = so.dot(p, ap)
        if not math.isfinite(pap) or pap <= 0.0:
            breakdown = not math.isfinite(pap)
            break
        alpha = rr / pap
        x.add_(p, alpha=alpha)
        r.add_(ap, alpha=-alpha)
        rr_new = so.dot(r, r)
        iters += 1
        relres = math.sqrt(rr_new) / bnorm
        if not math.isfinite(rr_new):
            breakdown = True
            break
        if relres <= rel_tol:
            break
        beta = rr_new / rr
        rr = rr_new
        p.mul_(beta).add_(r)
    return x, iters, relres, breakdown


def gauss_newton_minimize(so: SlabObjective, y0, cfg=None):
    """gauss_newton_minimize (optimizer.cpp:202-268) over z slabs: same control flow,
    stopping rules (optimizer.cpp:188-200) and Armijo backtracking
    (optimizer.cpp:156-175); J, norms and dots are global. Returns (y, trace,
    line_search_failed), identical on every rank."""
    import math

    from . import IterationRecord, OptimizerConfig
    cfg = cfg or OptimizerConfig()
    y = y0.clone()
    trace, lsf = [], False
    if cfg.max_iters <= 0:
        return y, trace, lsf
    grad = y.new_zeros(y.shape)
    y_trial = y.clone()
    j = so.eval(y, grad)
    g0 = math.sqrt(so.dot(grad, grad))
    min_hy = so.min_spacing()
    for it in range(cfg.max_iters):
        gnorm = math.sqrt(so.dot(grad, grad))
        rec = IterationRecord(it, 0, j, so.last_distance(), so.last_regularizer(), gnorm, 0.0)
        if gnorm <= cfg.tol_grad * g0:
            trace.append(rec)
            break
        d, rec.cg_iters, _, _ = cg_solve(so, -grad, cfg.cg_max_iters, cfg.cg_rel_tol)
        gdotd = so.dot(grad, d)
        dinf = so.inf_norm(d)
        eta = min(1.0, min_hy / dinf) if dinf > 0.0 else 1.0
        ok = False
        if gdotd < 0.0:
            for _ in range(cfg.max_backtracks + 1):
                torch_axpy_to(y, eta, d, y_trial)
                f = so.eval(y_trial, None)
                if math.isfinite(f) and f <= j + cfg.c1 * eta * gdotd:
                    ok = True
                    break
                eta *= cfg.beta
        if not ok:
            lsf = True
            trace.append(rec)
            break
        rec.step = eta
        j_prev = j
        torch_axpy_to(y, eta, d, y)
        step_inf = so.inf_norm(d, eta)
        j = so.eval(y, grad)
        trace.append(rec)
        gn = math.sqrt(so.dot(grad, grad))
        if (gn <= cfg.tol_grad * g0 or abs(j_prev - j) <= cfg.tol_rel_j * max(1.0, abs(j_prev))
                or step_inf <= cfg.tol_step * min_hy):
            break
    return y, trace, lsf


def torch_axpy_to(y, eta: float, d, out) -> None:
    """out = y + eta * d (optimizer.cpp:170, elementwise)."""
    import torch
    torch.add(y, d, alpha=eta, out=out)


# ------------------------------------------------------------------ native (C++) slabs
# The library's own z-slab path (csrc/slab.cu): the exchanges run over NCCL (or the
# in-process communicator) inside the C++ SlabProblem, and the device-resident solvers and
# the multilevel driver run sharded on it — no per-iteration Python or eager torch.
class NativeComm:
    """A C++ communicator handle: `nccl(rank, size)` (one process per GPU; the unique id is
    broadcast over torch.distributed) or `local(n)` (n ranks as threads of one process)."""

    def __init__(self, handle):
        self._h = handle
        r, s = C.c_int(), C.c_int()
        _check(lib().mfreg_cu_comm_rank(self._h, C.byref(r), C.byref(s)))
        self.rank, self.size = r.value, s.value

    @classmethod
    def nccl(cls, group=None) -> "NativeComm":
        import torch.distributed as dist
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        size = dist.get_world_size(group) if dist.is_initialized() else 1
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            _check(lib().mfreg_cu_comm_nccl_unique_id(uid))
        if size > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0 if group is None else dist.get_global_rank(group, 0), group=group)
            uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
        h = _vp()
        _check(lib().mfreg_cu_comm_create_nccl(uid, size, rank, C.byref(h)))
        return cls(h)

    @classmethod
    def local(cls, n: int) -> list["NativeComm"]:
        hs = (_vp * n)()
        _check(lib().mfreg_cu_comm_create_local(int(n), hs))
        return [cls(_vp(h)) for h in hs]

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().mfreg_cu_comm_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


class NativeSlab:
    """One rank's share of the objective in the library (mfreg_cu_slab_*): CUDA fp64 tensors of
    length 3 m^y; eval / gn_hessian_vec / dot return global values identical on every rank."""

    def __init__(self, comm: NativeComm, reference, tpl, image: GridDesc, deform: GridDesc,
                 params: NgfParams = NgfParams(), alpha: float = 1.0, mode: int = 1):
        """mode: Mode.FAST (default) or Mode.PARITY (bitwise the one-GPU parity objective)."""
        self.comm, self.image, self.deform = comm, image, _nodal(deform)
        w = _where_of(reference, tpl)
        reference, tpl = _as_input(reference, w), _as_input(tpl, w)
        h = _vp()
        _check(lib().mfreg_cu_slab_create(comm._h, _ptr(reference)[0], _ptr(tpl)[0], C.byref(image.c()),
                                          C.byref(self.deform.c()), float(params.tau), float(params.rho), float(alpha),
                                          int(mode), w, C.byref(h)))
        self._h = h
        tab = (C.c_int32 * 7)()
        _check(lib().mfreg_cu_slab_info(self._h, tab))
        self.info = SlabInfo(*tab)
        self._dof = 3 * self.deform.count()

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().mfreg_cu_slab_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def dof(self) -> int:
        return self._dof

    def identity(self, like):
        import torch
        out = torch.empty(self._dof, dtype=torch.float64, device=like.device)
        _check(lib().mfreg_cu_slab_identity(self._h, out.data_ptr()))
        return out

    def eval(self, y, grad=None) -> float:
        j = C.c_double()
        _check(lib().mfreg_cu_slab_eval(self._h, y.data_ptr(), grad.data_ptr() if grad is not None else None,
                                        C.byref(j)))
        return j.value

    def last(self):
        d, r = C.c_double(), C.c_double()
        _check(lib().mfreg_cu_slab_last(self._h, C.byref(d), C.byref(r)))
        return d.value, r.value

    def gn_hessian_vec(self, p, q):
        _check(lib().mfreg_cu_slab_gn_hessian_vec(self._h, p.data_ptr(), q.data_ptr()))
        return q

    def dot(self, a, b) -> float:
        v = C.c_double()
        _check(lib().mfreg_cu_slab_dot(self._h, a.data_ptr(), b.data_ptr(), C.byref(v)))
        return v.value

    def gather(self, v):
        _check(lib().mfreg_cu_slab_gather(self._h, v.data_ptr()))
        return v

    def minimize(self, y0, method: int, cfg=None):
        """gauss_newton_minimize / lbfgs_minimize, sharded; (y gathered on every rank, trace, lsf)."""
        import torch

        from . import OptimizerConfig, _IterRecord, _records
        cfg = cfg or OptimizerConfig()
        y = torch.empty_like(y0)
        cap = max(64, 4 * cfg.max_iters + 8)
        tr = (_IterRecord * cap)()
        nt, lsf = C.c_int(), C.c_int()
        oc = cfg.c()
        _check(lib().mfreg_cu_slab_minimize(self._h, int(method), y0.data_ptr(), C.byref(oc), y.data_ptr(), tr, cap,
                                            C.byref(nt), C.byref(lsf)))
        return y, _records(tr, min(nt.value, cap)), bool(lsf.value)


def register_multilevel_native(comm: NativeComm, reference, tpl, image: GridDesc, cfg=None):
    """register_multilevel (multilevel.cpp:117-145) over the communicator's z slabs (cfg.mode FAST
    or PARITY).
    Returns (y, deform_grid, per-level (trace, line_search_failed)), identical on every rank."""
    from . import FAST, MultilevelConfig, _empty_like_kind, _Grid, _IterRecord, _MlConfig, _records, deformation_grid_for
    cfg = cfg or MultilevelConfig(mode=FAST)
    w = _where_of(reference, tpl)
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
    _check(lib().mfreg_cu_slab_register_multilevel(comm._h, _ptr(reference)[0], _ptr(tpl)[0], C.byref(image.c()),
                                                   C.byref(mc), _ptr(y)[0], C.byref(og), tr, cap, li, lsf, w))
    levels, off = [], 0
    for l in range(cfg.levels):
        levels.append((_records(tr[off:off + li[l]], li[l]), bool(lsf[l])))
        off += li[l]
    return y, GridDesc(tuple(og.m), tuple(og.h), True), levels
