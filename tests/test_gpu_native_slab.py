"""The library's own multi-GPU path (csrc/slab.cu): the C++ SlabProblem under the
device-resident solvers and the sharded multilevel driver, against the single-GPU fast
objective. Ranks run as threads of one process on the one GPU (the in-process
communicator, MFREG_NO_GRAPHS=1 since several threads share the legacy stream), and the
NCCL communicator is exercised at world size 1 (one GPU per box here)."""
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
img = P.make_image_grid((40, 36, 96), (0.97, 0.97, 1.5))
dg = P.deformation_grid_for(img, 4)
R = P.make_phantom(img, device=True); R.mul_(1000.0)
T = P.warp_sinusoid(R, img, 3.0, 42)
full = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, P.FAST)
rng = np.random.default_rng(5)
y = torch.from_numpy(full.identity() + rng.uniform(-0.3, 0.3, full.dof())).cuda()
p = torch.from_numpy(rng.uniform(-1, 1, full.dof())).cuda()
g_full = torch.empty_like(y); q_full = torch.empty_like(y)
J = full.eval(y, g_full); D, Sreg = full.last_distance(), full.last_regularizer()
full.gn_hessian_vec(p, q_full)
pq_full = float((p * q_full).sum())
# At alpha = 1 the GN operator is ill-conditioned: CG stops at its cap and amplifies rounding
# (as in the reference itself, SURVEY H4); the sharded solver (its reductions add in a
# different fixed order) is compared on a better-conditioned problem, where the trajectories
# stay within 1e-5 (measured <= 1e-6)
cfg = P.OptimizerConfig(max_iters=4, cg_max_iters=400, cg_rel_tol=1e-10)
# solver comparisons on a better-conditioned problem (alpha = 100): CG converges, so the
# trajectory no longer amplifies the reductions' rounding
A = 100.0
full_a = P.Objective(R, T, img, dg, P.NgfParams(), A, P.FAST)
_, tr_full, _ = P.gauss_newton_minimize(full_a, y.clone(), cfg)
mc = P.MultilevelConfig(levels=2, method=P.Method.GAUSS_NEWTON, mode=P.FAST, alpha=A,
                        opt=P.OptimizerConfig(max_iters=3, cg_max_iters=400, cg_rel_tol=1e-10))
y_ml, _, lv_full = P.register_multilevel(R, T, img, mc)
torch.cuda.synchronize()

comms = S.NativeComm.local(N) if N > 1 else [S.NativeComm.nccl()]
res = [None] * N
def rank(r):
    try:
        sl = S.NativeSlab(comms[r], R, T, img, dg)
        yy, gg, pp, qq = y.clone(), torch.zeros_like(y), p.clone(), torch.zeros_like(y)
        j = sl.eval(yy, gg)
        d, s = sl.last()
        sl.gn_hessian_vec(pp, qq)
        pq = sl.dot(pp, qq)
        sa = S.NativeSlab(comms[r], R, T, img, dg, P.NgfParams(), A)
        yg, tr, lsf = sa.minimize(y.clone(), P.Method.GAUSS_NEWTON, cfg)
        ym, _, lv = S.register_multilevel_native(comms[r], R, T, img, mc)
        torch.cuda.synchronize()
        res[r] = dict(info=sl.info, j=j, d=d, s=s, g=gg, q=qq, pq=pq, tr=tr, ym=ym, lv=lv)
    except Exception as e:  # surfaced below
        res[r] = e
th = [threading.Thread(target=rank, args=(r,)) for r in range(N)]
[t.start() for t in th]; [t.join() for t in th]
for r in res:
    if isinstance(r, Exception):
        raise r
mx, my, mz = dg.m
rel = lambda a, b: float((a - b).abs().max() / b.abs().max())
for r in res:
    assert abs(r["j"] - J) <= 1e-12 * abs(J) and abs(r["d"] - D) <= 1e-12 * abs(D) and abs(r["s"] - Sreg) <= 1e-12 * abs(Sreg)
    lo, hi = r["info"].own_lo, r["info"].own_hi
    own = lambda v: v.view(3, mz, my, mx)[:, lo:hi]
    assert rel(own(r["g"]), own(g_full)) <= 1e-9, rel(own(r["g"]), own(g_full))
    assert rel(own(r["q"]), own(q_full)) <= 1e-9, rel(own(r["q"]), own(q_full))
    assert abs(r["pq"] - pq_full) <= 1e-9 * abs(pq_full)
    # sharded reductions add in a different order than the single-GPU ones (both fixed)
    print("gn", [(a.cg_iters, a.j) for a in r["tr"]], [(b.cg_iters, b.j) for b in tr_full])
    print("ml", [[a.j for a in ta] for ta, _ in r["lv"]], [[b.j for b in tb] for tb, _ in lv_full])
    print("ym", rel(r["ym"], y_ml))
    assert len(r["tr"]) == len(tr_full)
    assert abs(r["tr"][0].j - tr_full[0].j) <= 1e-12 * abs(tr_full[0].j)
    for a, b in zip(r["tr"], tr_full):
        # CG stops at its 400-iteration cap here, so the trajectory amplifies the reductions'
        # rounding: measured 3e-7 / 3e-7 / 6e-6 at iterations 1-3 with the reference-order P y and
        # 1.4e-6 / 2.1e-4 / 6e-5 with the separable one (the operators agree to 1e-12 / 1e-9 above)
        tol = 1e-5 if a.iter < 2 else 1e-3
        assert abs(a.j - b.j) <= tol * abs(b.j), (a.as_tuple(), b.as_tuple())
    for lvl, ((ta, _), (tb, _)) in enumerate(zip(r["lv"], lv_full)):
        assert len(ta) == len(tb), (lvl, len(ta), len(tb))
        for a, b in zip(ta, tb):
            assert abs(a.j - b.j) <= 1e-5 * abs(b.j), ("level", lvl, a.as_tuple(), b.as_tuple())
    assert rel(r["ym"], y_ml) <= 1e-4
# identical scalars and results on every rank
for r in res[1:]:
    assert r["j"] == res[0]["j"] and [t.j for t in r["tr"]] == [t.j for t in res[0]["tr"]]
    assert torch.equal(r["ym"], res[0]["ym"])
print("ok", N, [tuple(r["info"].__dict__.values()) if hasattr(r["info"], "__dict__") else r["info"] for r in res])
"""


@pytest.mark.parametrize("n", [1, 2, 3])
def test_native_slabs_match_single_gpu(n):
    env = dict(os.environ, MFREG_NO_GRAPHS="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, n=n)], env=env, capture_output=True, text=True,
                       timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stderr[-3000:]
    assert "ok" in r.stdout
