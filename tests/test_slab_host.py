"""CPU: the z-slab decomposition's host logic (SURVEY §8 row e) without a GPU.

* `slab_partition` (native, `mfreg_cu_slab_partition`): slabs tile the image z axis,
  split on nodal-cell boundaries, owned nodal planes partition the deformation
  grid, each rank's operand halo lies inside its neighbours' owned planes, and the
  shared P^T planes are exactly the ones both neighbours touch.
* `SlabExchange` over torch.distributed **gloo, world_size 2 and 3** (and the
  in-process loopback): halo exchange + shared-plane assembly + ordered scalar
  sums reproduce a full-domain operator with the same data dependencies as the
  objective (P, a +-3-plane image stencil standing in for the warp / NGF stencils,
  P^T of the rank's image planes, alpha * curvature Hessian on the owned planes).
  Every plane a rank does not own or receive is NaN, so a missing halo plane
  cannot go unnoticed.
"""
from __future__ import annotations

import os
import socket
import threading

import numpy as np
import pytest

from conftest import ROOT

IMG_M, IMG_H = (20, 18, 40), (1.0, 1.0, 1.5)


@pytest.fixture(scope="module")
def pkg():
    import paper_1804_10541_b200 as P
    if not os.path.exists(P._LIB_PATH):
        P.build()
    return P


def _base(mt, ms):
    k = np.arange(mt, dtype=np.float64)
    return np.clip(np.floor((k + 0.5) * (ms - 1) / mt).astype(np.int64), 0, ms - 2)  # transfer.cpp:24-35


@pytest.mark.parametrize("m,h,ratio,n", [
    ((20, 18, 40), (1.0, 1.0, 1.5), 4, 2), ((20, 18, 40), (1.0, 1.0, 1.5), 4, 3),
    ((16, 16, 128), (1.0, 1.0, 1.0), 4, 4), ((16, 16, 1024), (1.0, 1.0, 1.0), 4, 8),
    ((12, 12, 97), (0.97, 0.97, 2.5), 3, 5), ((8, 8, 64), (1.0, 1.0, 1.0), 1, 8),
])
def test_partition_invariants(pkg, m, h, ratio, n):
    img = pkg.make_image_grid(m, h)
    dg = pkg.deformation_grid_for(img, ratio)
    parts = pkg.slab.slab_partition(img, dg, n)
    mz, ms = m[2], dg.m[2]
    b = _base(mz, ms)
    assert parts[0].zlo == 0 and parts[-1].zhi == mz
    assert parts[0].own_lo == 0 and parts[-1].own_hi == ms
    for r, s in enumerate(parts):
        assert s.zlo < s.zhi and s.own_lo < s.own_hi
        if r:
            assert s.zlo == parts[r - 1].zhi and s.own_lo == parts[r - 1].own_hi
            assert b[s.zlo] != b[s.zlo - 1]            # split on a nodal-cell boundary
            assert s.own_lo == b[s.zlo]
            assert s.need_lo >= parts[r - 1].own_lo    # halo from the neighbour only
        if r + 1 < n:
            assert s.need_hi <= parts[r + 1].own_hi
            touched_hi = b[s.zhi - 1] + 2              # P^T of planes [zlo, zhi) reaches nodes < touched_hi
            assert s.bnd == max(0, touched_hi - s.own_hi)
        assert s.need_lo <= max(0, s.own_lo - 2) and s.need_hi >= min(ms, s.own_hi + 2)
        wlo, whi = max(0, s.zlo - 3), min(mz, s.zhi + 3)
        assert s.need_lo <= b[wlo] and s.need_hi >= b[whi - 1] + 2
    # near-even split of the image planes
    sizes = [s.zhi - s.zlo for s in parts]
    assert max(sizes) - min(sizes) <= 2 * (mz / (ms - 1)) + 1


@pytest.mark.parametrize("m,h,ratio,n", [
    ((20, 18, 40), (1.0, 1.0, 1.5), 4, 2), ((16, 16, 128), (1.0, 1.0, 1.0), 4, 4),
    ((16, 16, 1024), (1.0, 1.0, 1.0), 4, 8), ((12, 12, 97), (0.97, 0.97, 2.5), 3, 5),
])
def test_partition_parity_halo(pkg, m, h, ratio, n):
    """Parity-mode slabs recompute the per-voxel terms of the nodal slab below own_lo so each
    owned node's P^T gather runs complete on its rank: the operand halo covers the warp of
    [first plane of nodal slab own_lo - 1, zhi) +- 2 image planes, and still comes from the
    neighbours' owned planes only."""
    img = pkg.make_image_grid(m, h)
    dg = pkg.deformation_grid_for(img, ratio)
    fast = pkg.slab.slab_partition(img, dg, n)
    parts = pkg.slab.slab_partition(img, dg, n, pkg.Mode.PARITY)
    mz, ms = m[2], dg.m[2]
    b = _base(mz, ms)
    for r, (s, f) in enumerate(zip(parts, fast)):
        assert (s.zlo, s.zhi, s.own_lo, s.own_hi) == (f.zlo, f.zhi, f.own_lo, f.own_hi)  # same split
        z = s.zlo
        while s.own_lo > 0 and z > 0 and b[z - 1] >= s.own_lo - 1:
            z -= 1
        if s.own_lo > 0:
            assert b[z] == s.own_lo - 1  # first image plane of the nodal slab below own_lo
        wlo, whi = max(0, z - 2), min(mz, s.zhi + 2)
        assert s.need_lo <= b[wlo] and s.need_hi >= b[whi - 1] + 2
        if r:
            assert s.need_lo >= parts[r - 1].own_lo
        if r + 1 < n:
            assert s.need_hi <= parts[r + 1].own_hi


def test_partition_rejects_thin_slabs(pkg):
    img = pkg.make_image_grid((16, 16, 16))
    dg = pkg.deformation_grid_for(img, 4)
    with pytest.raises(ValueError):
        pkg.slab.slab_partition(img, dg, 8)
    with pytest.raises(ValueError):
        pkg.slab.slab_partition(img, dg, 0)


# ------------------------------------------------------------ toy operator with the objective's dependencies
def _toy_setup(pkg):
    img = pkg.make_image_grid(IMG_M, IMG_H)
    dg = pkg.deformation_grid_for(img, 4)
    rng = np.random.default_rng(7)
    p = rng.standard_normal(3 * dg.count())
    return img, dg, p


def _stencil(v, mz, lo, hi):
    """+-3-plane z stencil of an image 3-field (3, mz, my, mx), evaluated on planes [lo, hi)."""
    out = np.zeros_like(v)
    for i in range(lo, hi):
        acc = 0.0
        for k in range(-3, 4):
            acc = acc + v[:, min(max(i + k, 0), mz - 1)] / (1.0 + abs(k))
        out[:, i] = acc
    return out


def _toy_apply(o, img, dg, p, zlo, zhi, own_lo, own_hi, alpha=0.7):
    """Rank-local toy contribution; full domain with zlo=0, zhi=mz, own = all."""
    mt, ht, ms, hs = tuple(img.m), tuple(img.h), tuple(dg.m), tuple(dg.h)
    v = o.transfer_apply(ms, hs, mt, ht, p).reshape(3, mt[2], mt[1], mt[0])
    w = _stencil(v, mt[2], zlo, zhi)
    q = o.transfer_apply_transpose(ms, hs, mt, ht, w.ravel()).reshape(3, ms[2], ms[1], ms[0])
    c = o.curvature_hessian_vec(p, ms, hs).reshape(3, ms[2], ms[1], ms[0])
    q[:, own_lo:own_hi] += alpha * c[:, own_lo:own_hi]
    return q.ravel()


def _rank_body(rank, comm, results):
    import torch

    import paper_1804_10541_b200 as P
    from oracle.oracle import Oracle, available
    o = Oracle("ref" if available("ref") else "port")
    img, dg, p = _toy_setup(P)
    parts = P.slab.slab_partition(img, dg, comm.size)
    s = parts[rank]
    ex = P.slab.SlabExchange(parts, rank, comm, dg)
    ms = tuple(dg.m)
    # the rank holds only its owned planes; everything else is NaN until the halo arrives
    pl = torch.full((3 * dg.count(),), float("nan"), dtype=torch.float64)
    full = torch.from_numpy(p.copy())
    ex._planes(pl, s.own_lo, s.own_hi).copy_(ex._planes(full, s.own_lo, s.own_hi))
    ex.halo(pl)
    pv = pl.view(3, ms[2], ms[1], ms[0])
    assert torch.isfinite(pv[:, s.need_lo:s.need_hi]).all()
    q = torch.from_numpy(_toy_apply(o, img, dg, pl.numpy(), s.zlo, s.zhi, s.own_lo, s.own_hi))
    # planes this rank neither owns nor shares are garbage (NaN) -> zero before assembly
    qv = q.view(3, ms[2], ms[1], ms[0])
    keep = torch.zeros(ms[2], dtype=torch.bool)
    keep[s.own_lo:s.own_hi + s.bnd] = True
    qv[:, ~keep] = 0.0
    ex.boundary(q)
    d = float((ex._planes(full, s.own_lo, s.own_hi) * ex._planes(q, s.own_lo, s.own_hi)).sum())
    tot = ex.allsum([d, float(rank)], q)
    results[rank] = (ex._planes(q, s.own_lo, s.own_hi).clone().numpy(), tot)


def _gloo_worker(rank, world, port, queue):
    import torch.distributed as dist

    import paper_1804_10541_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        _rank_body(rank, P.slab.TorchComm(), res)
        queue.put((rank, res[rank]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _check_assembled(pkg, oracle, results, n):
    img, dg, p = _toy_setup(pkg)
    ms = tuple(dg.m)
    ref = _toy_apply(oracle, img, dg, p, 0, img.m[2], 0, ms[2]).reshape(3, ms[2], ms[1], ms[0])
    parts = pkg.slab.slab_partition(img, dg, n)
    scale = np.max(np.abs(ref))
    for r, s in enumerate(parts):
        got, tot = results[r]
        np.testing.assert_allclose(got, ref[:, s.own_lo:s.own_hi], rtol=0, atol=1e-12 * scale)
        assert tot[0] == results[0][1][0]                       # identical on every rank
        assert abs(tot[0] - float(np.dot(p, ref.ravel()))) <= 1e-12 * abs(float(np.dot(p, ref.ravel())))
        assert tot[1] == sum(range(n))


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_exchange_reproduces_full_domain(pkg, oracle, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = {}
    try:
        for _ in range(world):
            r, val = q.get(timeout=240)
            results[r] = val
    finally:
        for pr in procs:
            pr.join(timeout=60)
            if pr.is_alive():
                pr.kill()
    assert all(pr.exitcode == 0 for pr in procs)
    _check_assembled(pkg, oracle, results, world)


def test_loopback_slab_exchange_reproduces_full_domain(pkg, oracle):
    n = 3
    hub = pkg.slab.LoopbackHub(n)
    results, errs = {}, []

    def run(r):
        try:
            _rank_body(r, hub.comm(r), results)
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    _check_assembled(pkg, oracle, results, n)
