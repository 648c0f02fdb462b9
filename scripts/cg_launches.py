"""One eval(y, grad) and a 4-iteration CG solve at any size (M=mx,my,mz H=spacing; default C4)
inside a cudaProfilerStart/Stop window, for `ncu --profile-from-start off` launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_10541_b200 as P
mode = {"fast": P.Mode.FAST, "fast32": P.Mode.FAST32}[sys.argv[1] if len(sys.argv) > 1 else "fast"]
m = tuple(int(v) for v in os.environ.get("M", "512,512,900").split(","))
hh = float(os.environ.get("H", "0.7")); img = P.make_image_grid(m, (hh, hh, hh))
R = P.make_phantom(img, device=True); R.mul_(1000.0)
T = P.warp_sinusoid(R, img, 3.0, 42)
dg = P.deformation_grid_for(img, 4)
gen = torch.Generator(device="cuda").manual_seed(8)
nd = 3 * dg.count()
y = torch.from_numpy(dg.point_coords()).cuda() + (torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 0.6 - 0.3)
obj = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, mode)
g = torch.empty_like(y)
obj.eval(y, g)
P.cg_solve(obj, -g, 2, 1e-12)
torch.cuda.synchronize()
torch.cuda.profiler.start()
obj.eval(y, g)
P.cg_solve(obj, -g, 4, 1e-12)
obj.eval(y)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
