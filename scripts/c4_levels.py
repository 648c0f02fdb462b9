"""Single-level Gauss-Newton wall time at each C4 pyramid size (fast mode): where the
multilevel wall goes, level by level."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_10541_b200 as P

mode = P.Mode.FAST32 if "--fast32" in sys.argv else P.Mode.FAST
for m in ((128, 128, 225), (256, 256, 450), (512, 512, 900)):
    img = P.make_image_grid(m, (0.7, 0.7, 0.7))  # C4 spacing (exercises the tie hazard H1)
    R = P.make_phantom(img, device=True)
    R.mul_(1000.0)
    T = P.warp_sinusoid(R, img, 3.0, 42)
    cfg = P.MultilevelConfig(levels=1, deform_ratio=4, method=P.Method.GAUSS_NEWTON, mode=mode)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        y, dg, levels = P.register_multilevel(R, T, img, cfg)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        tr = levels[0][0]
        cg = int(sum(r.cg_iters for r in tr))
        print(f"{m}: rep {rep} wall {wall:.3f} s, outer {len(tr)}, cg {cg}, {wall / max(cg, 1) * 1e3:.3f} ms per cg", flush=True)
    del R, T, y
