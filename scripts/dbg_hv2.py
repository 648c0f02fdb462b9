"""Debug aid: hv2 vs legacy fused Hv on one shape; prints where they differ."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10541_b200 as P
m = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (70, 30, 23)
h = (0.97, 0.97, 2.5)
img = P.make_image_grid(m, h); dg = P.deformation_grid_for(img, 4)
R = P.make_phantom(img) * 1000.0; T = P.warp_sinusoid(R, img, 3.0, 42)
res = []
for legacy in ("1", "0"):
    os.environ["MFREG_NO_HV2"] = legacy
    o = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, P.Mode.FAST)
    rng = np.random.default_rng(11)
    y = o.identity() + rng.uniform(-0.4, 0.4, o.dof()); p = rng.uniform(-1, 1, o.dof())
    g = np.empty(o.dof()); o.eval(y, g)
    res.append(o.gn_hessian_vec(p))
d = np.abs(res[1] - res[0]).reshape(3, dg.m[2], dg.m[1], dg.m[0])
print("grid", dg.m, "max", d.max(), "rel", d.max() / np.abs(res[0]).max())
idx = np.argwhere(d > 1e-9 * np.abs(res[0]).max())
print("bad count", len(idx))
for c in range(3):
    for ax, nm in ((1, "z"), (2, "y"), (3, "x")):
        sel = idx[idx[:, 0] == c]
        if len(sel): print("comp", c, nm, np.unique(sel[:, ax]))
