"""Parity mode across z slabs (csrc/slab.cu SlabProblem with Mode::Parity): the
sharded objective, its GN / L-BFGS trajectories and the sharded multilevel registration are
bitwise equal to the single-GPU parity objective, which the other tests pin bitwise to the
reference library (tests/test_gpu_parity.py, test_gpu_trajectory.py). Ranks run as threads of
one process on the one GPU (the in-process communicator; MFREG_NO_GRAPHS=1 since the threads
share the legacy stream); world size 1 goes through the NCCL communicator."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, threading
import numpy as np
import torch
sys.path.insert(0, {root!r})
import paper_1804_10541_b200 as P
from paper_1804_10541_b200 import slab as S

N = {n}
img = P.make_image_grid({m}, {h})
dg = P.deformation_grid_for(img, {ratio})
R = P.make_phantom(img, device=True); R.mul_(1000.0)
T = P.warp_sinusoid(R, img, 3.0, 42)
full = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, P.PARITY)
rng = np.random.default_rng(5)
y = torch.from_numpy(full.identity() + rng.uniform(-0.3, 0.3, full.dof())).cuda()
p = torch.from_numpy(rng.uniform(-1, 1, full.dof())).cuda()
g_full = torch.empty_like(y); q_full = torch.empty_like(y)
J = full.eval(y, g_full); D, Sreg = full.last_distance(), full.last_regularizer()
full.gn_hessian_vec(p, q_full)
pq_full = full.dot(p, q_full)
# the single-GPU parity objective is the reference library's objective bit for bit
sys.path.insert(0, {root!r} + "/oracle/..")
from oracle.oracle import Oracle, available
if available("ref"):
    o = Oracle("ref").objective(R.cpu().numpy(), T.cpu().numpy(), {m}, {h}, tuple(dg.m), 10.0, 10.0, 1.0)
    Jr, Dr, Sr, gr = o.eval(y.cpu().numpy())
    assert (J, D, Sreg) == (Jr, Dr, Sr) and np.array_equal(g_full.cpu().numpy(), gr)
    assert np.array_equal(q_full.cpu().numpy(), o.gn_hessian_vec(p.cpu().numpy()))
cfg = P.OptimizerConfig(max_iters=3, cg_max_iters=60)
yg_full, tr_full, _ = P.gauss_newton_minimize(full, y.clone(), cfg)
yl_full, trl_full, _ = P.lbfgs_minimize(full, y.clone(), P.OptimizerConfig(max_iters=4))
mc = P.MultilevelConfig(levels=2, method=P.Method.GAUSS_NEWTON, mode=P.PARITY,
                        opt=P.OptimizerConfig(max_iters=2, cg_max_iters=40))
y_ml, _, lv_full = P.register_multilevel(R, T, img, mc)
torch.cuda.synchronize()

comms = S.NativeComm.local(N) if N > 1 else [S.NativeComm.nccl()]
res = [None] * N
def rank(r):
    try:
        sl = S.NativeSlab(comms[r], R, T, img, dg, P.NgfParams(), 1.0, P.PARITY)
        yy, gg, pp, qq = y.clone(), torch.zeros_like(y), p.clone(), torch.zeros_like(y)
        j = sl.eval(yy, gg)
        d, s = sl.last()
        sl.gn_hessian_vec(pp, qq)
        pq = sl.dot(pp, qq)
        yg, tr, _ = sl.minimize(y.clone(), P.Method.GAUSS_NEWTON, cfg)
        yl, trl, _ = sl.minimize(y.clone(), P.Method.LBFGS, P.OptimizerConfig(max_iters=4))
        ym, _, lv = S.register_multilevel_native(comms[r], R, T, img, mc)
        torch.cuda.synchronize()
        res[r] = dict(info=sl.info, j=j, d=d, s=s, g=gg, q=qq, pq=pq, tr=tr, yg=yg, trl=trl, yl=yl, ym=ym, lv=lv)
    except Exception as e:  # surfaced below
        res[r] = e
th = [threading.Thread(target=rank, args=(r,)) for r in range(N)]
[t.start() for t in th]; [t.join() for t in th]
for r in res:
    if isinstance(r, Exception):
        raise r
mx, my, mz = dg.m
for r in res:
    lo, hi = r["info"].own_lo, r["info"].own_hi
    own = lambda v: v.view(3, mz, my, mx)[:, lo:hi]
    assert (r["j"], r["d"], r["s"]) == (J, D, Sreg), ((r["j"], r["d"], r["s"]), (J, D, Sreg))
    assert torch.equal(own(r["g"]), own(g_full)), float((own(r["g"]) - own(g_full)).abs().max())
    assert torch.equal(own(r["q"]), own(q_full)), float((own(r["q"]) - own(q_full)).abs().max())
    # <p, q> over the sharded q is the reference's vec_dot of the whole vectors
    assert r["pq"] == pq_full, (r["pq"], pq_full)
    assert [a.as_tuple() for a in r["tr"]] == [b.as_tuple() for b in tr_full]
    assert torch.equal(r["yg"], yg_full)
    assert [a.as_tuple() for a in r["trl"]] == [b.as_tuple() for b in trl_full]
    assert torch.equal(r["yl"], yl_full)
    for (ta, _), (tb, _) in zip(r["lv"], lv_full):
        assert [a.as_tuple() for a in ta] == [b.as_tuple() for b in tb]
    assert torch.equal(r["ym"], y_ml)
print("ok", N, [r["info"] for r in res])
"""

CASES = [((40, 36, 96), (0.97, 0.97, 1.5), 4), ((33, 20, 57), (1.0, 1.0, 1.0), 3)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0])))
@pytest.mark.parametrize("n", [1, 2, 3])
def test_parity_slabs_bitwise_single_gpu(n, case):
    m, h, ratio = case
    env = dict(os.environ, MFREG_NO_GRAPHS="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, n=n, m=m, h=h, ratio=ratio)], env=env,
                       capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stderr[-3000:]
    assert "ok" in r.stdout
