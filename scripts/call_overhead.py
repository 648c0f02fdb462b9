"""Host-side cost of one public-API call (tiny grid, device tensors)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_10541_b200 as P
img = P.make_image_grid((16, 16, 16)); dg = P.deformation_grid_for(img, 4)
R = P.make_phantom(img, device=True); T = P.warp_sinusoid(R, img, 3.0, 42)
o = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, P.Mode.FAST)
y = torch.from_numpy(dg.point_coords()).cuda(); g = torch.empty_like(y); q = torch.empty_like(y)
for _ in range(20): o.eval(y, g); o.gn_hessian_vec(y, q)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N): o.gn_hessian_vec(y, q)
torch.cuda.synchronize(); th = (time.perf_counter() - t0) / N
t0 = time.perf_counter()
for _ in range(N): o.eval(y, g)
te = (time.perf_counter() - t0) / N
print(f"per call: gn_hessian_vec {th*1e6:.1f} us (async), eval {te*1e6:.1f} us (incl. sync)")
