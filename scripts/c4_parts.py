"""C4 finest level (512x512x900): objective creation, eval, GN Hv times (fast / fast32)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_10541_b200 as P
m = (512, 512, 900)
img = P.make_image_grid(m, (0.7, 0.7, 0.7))  # C4 spacing
R = P.make_phantom(img, device=True); R.mul_(1000.0)
T = P.warp_sinusoid(R, img, 3.0, 42)
dg = P.deformation_grid_for(img, 4)
gen = torch.Generator(device="cuda").manual_seed(8)
nd = 3 * dg.count()
y = torch.from_numpy(dg.point_coords()).cuda() + (torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 0.6 - 0.3)
p = torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 2.0 - 1.0
for name, mode in (("fast", P.Mode.FAST), ("fast32", P.Mode.FAST32)):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    obj = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, mode)
    torch.cuda.synchronize(); tc = time.perf_counter() - t0
    g = torch.empty_like(y); q = torch.empty_like(y)
    obj.eval(y, g); obj.gn_hessian_vec(p, q); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): obj.eval(y, g)
    torch.cuda.synchronize(); te = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    for _ in range(20): obj.gn_hessian_vec(p, q)
    torch.cuda.synchronize(); th = (time.perf_counter() - t0) / 20
    kh = obj.profile_kernel(0, p, 5, 0); ke = obj.profile_kernel(1, p, 5, 0); kw = obj.profile_kernel(2, y, 5, 0)
    print(f"{name}: create {tc*1e3:.0f} ms, eval {te*1e3:.2f} ms, hv {th*1e3:.3f} ms | kernels hv {kh:.3f} ev {ke:.3f} warp {kw:.3f} ms", flush=True)
    del obj

# one CG solve (50 iterations) at the finest level, and the Armijo value-only eval
obj = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, P.Mode.FAST)
g = torch.empty_like(y)
obj.eval(y, g)
b = -g
torch.cuda.synchronize(); t0 = time.perf_counter()
x, it, rr, br = P.cg_solve(obj, b, 50, 1e-2)
torch.cuda.synchronize(); tcg = time.perf_counter() - t0
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): obj.eval(y)
torch.cuda.synchronize(); tv = (time.perf_counter() - t0) / 5
print(f"cg: {it} iterations {tcg*1e3:.1f} ms ({tcg/max(it,1)*1e3:.3f} ms/iter); value-only eval {tv*1e3:.2f} ms", flush=True)
