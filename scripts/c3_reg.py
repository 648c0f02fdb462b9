"""C3 (256x256x100, h = (0.97, 0.97, 2.5), 4-level L-BFGS) wall times per mode + landmark error."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1804_10541_b200 as P
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "c3_lbfgs.npz"))
m, h = tuple(int(v) for v in g["m"]), tuple(float(v) for v in g["h"])
img = P.make_image_grid(m, h)
R = P.make_phantom(img, device=True); R.mul_(1000.0)
T = P.warp_sinusoid(R, img, 3.0, 42)
for name, mode in (("parity", P.Mode.PARITY), ("fast", P.Mode.FAST), ("fast32", P.Mode.FAST32)):
    for method, mname in ((P.Method.LBFGS, "lbfgs"), (P.Method.GAUSS_NEWTON, "gn")):
        cfg = P.MultilevelConfig(levels=4, method=method, mode=mode)
        P.register_multilevel(R, T, img, P.MultilevelConfig(levels=4, method=method, mode=mode, opt=P.OptimizerConfig(max_iters=1)))
        torch.cuda.synchronize(); t0 = time.perf_counter()
        y, dg, lv = P.register_multilevel(R, T, img, cfg)
        torch.cuda.synchronize(); t = time.perf_counter() - t0
        la = P.io.landmark_error(g["fixed"], g["moving"], y, dg)
        print(f"{name} {mname}: {t:.3f} s, iters {[len(tr) for tr, _ in lv]}, cg {sum(r.cg_iters for tr, _ in lv for r in tr)}, landmark error {la[0]:.4f}", flush=True)
