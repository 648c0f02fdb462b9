"""Wall time per public-API call at 128^3 (fast): device tensors vs pinned host arrays,
and the raw pinned H2D / D2H copy time of one nodal vector (what e2e adds per transfer)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_10541_b200 as P
img = P.make_image_grid((128, 128, 128)); dg = P.deformation_grid_for(img, 4)
R = P.make_phantom(img, device=True); R.mul_(1000.0); T = P.warp_sinusoid(R, img, 3.0, 42)
o = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, P.Mode.FAST)
nd = 3 * dg.count()
y = torch.from_numpy(dg.point_coords()).cuda(); p = torch.rand(nd, dtype=torch.float64, device="cuda")
g = torch.empty_like(y); q = torch.empty_like(y)
yh = y.cpu().pin_memory().numpy(); ph = p.cpu().pin_memory().numpy()
gh = torch.empty(nd, dtype=torch.float64).pin_memory().numpy(); qh = torch.empty(nd, dtype=torch.float64).pin_memory().numpy()
def t(f, n=200):
    for _ in range(10): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e6
print(f"eval device {t(lambda: o.eval(y, g)):.1f} us, host {t(lambda: o.eval(yh, gh)):.1f} us")
print(f"hv   device {t(lambda: (o.gn_hessian_vec(p, q), torch.cuda.synchronize())):.1f} us, host {t(lambda: o.gn_hessian_vec(ph, qh)):.1f} us")
ht = torch.from_numpy(yh); dt = torch.empty_like(y)
print(f"H2D {nd*8/1e3:.0f} KB {t(lambda: (dt.copy_(ht, non_blocking=True), torch.cuda.synchronize())):.1f} us, "
      f"D2H {t(lambda: (torch.from_numpy(gh).copy_(dt, non_blocking=True), torch.cuda.synchronize())):.1f} us")
