"""North-star case C4: full multilevel Gauss-Newton registration of a 512x512x900
synthetic CT pair on one B200 (fast mode), wall time and per-level iterations."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_10541_b200 as P

args = [a for a in sys.argv[1:] if not a.startswith("--")]
m = tuple(int(v) for v in args[:3]) if len(args) >= 3 else (512, 512, 900)
mode = P.Mode.FAST32 if "--fast32" in sys.argv else P.Mode.FAST
img = P.make_image_grid(m, (0.7, 0.7, 0.7))  # C4 spacing (exercises the tie hazard H1)
t0 = time.perf_counter()
R = P.make_phantom(img, device=True)
R.mul_(1000.0)
T = P.warp_sinusoid(R, img, 3.0, 42)
torch.cuda.synchronize()
print(f"inputs {m}: {time.perf_counter() - t0:.2f} s, {torch.cuda.memory_allocated() / 1e9:.1f} GB")
cfg = P.MultilevelConfig(levels=3, deform_ratio=4, method=P.Method.GAUSS_NEWTON, mode=mode)
print("mode", "FAST32" if mode == P.Mode.FAST32 else "FAST")
for rep in range(int(os.environ.get("REPS", "2"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    y, dg, levels = P.register_multilevel(R, T, img, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    its = [len(t) for t, _ in levels]
    cg = [int(sum(r.cg_iters for r in t)) for t, _ in levels]
    print(f"rep {rep}: wall {wall:.3f} s, outer {its}, cg {cg}, final J {levels[-1][0][-1].j:.6g}, "
          f"peak mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB (torch)", flush=True)
