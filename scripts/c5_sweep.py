"""C5: 1024^3 derivative-only sweep on one B200 (gradient + GN Hv), fast / fast32.

Prints device times (CUDA events, median of 5) per operator, Gvoxel/s, the HBM roofline
fraction of the canonical bytes, and two size-independent checks at this size: Hv
symmetry <H p1, p2> = <p1, H p2> (exact up to rounding), and J / <g, p1> of fast against
fast32 (independent arithmetic). The central-difference gradient check is printed for
several steps; on the piecewise-trilinear phantom it levels off near 1e-3 (interpolation
kinks), so it is a sanity check, not a tolerance."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_10541_b200 as P

m = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (1024, 1024, 1024)
modes = [a for a in sys.argv[1:] if a in ("fast", "fast32")] or ["fast", "fast32"]
img = P.make_image_grid(m)
dg = P.deformation_grid_for(img, 4)
R = P.make_phantom(img, device=True)
R.mul_(1000.0)
T = P.warp_sinusoid(R, img, 3.0, 42)
gen = torch.Generator(device="cuda").manual_seed(8)
nd = 3 * dg.count()
y = torch.from_numpy(dg.point_coords()).cuda() + (torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 0.6 - 0.3)
p1 = torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 2.0 - 1.0
p2 = torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 2.0 - 1.0
n = img.count()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = float(peak["hbm_gbs"])
out = {"image": list(m), "nodal": list(dg.m), "voxels": n}
for name in modes:
    mode = P.Mode.FAST32 if name == "fast32" else P.Mode.FAST
    obj = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, mode)
    g = torch.empty_like(y)
    q1 = torch.empty_like(y)
    q2 = torch.empty_like(y)
    obj.eval(y, g)
    obj.gn_hessian_vec(p1, q1)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    te, th = [], []
    for _ in range(5):
        ev[0].record()
        obj.eval(y, g)
        ev[1].record()
        obj.gn_hessian_vec(p1, q1)
        ev[2].record()
        torch.cuda.synchronize()
        te.append(ev[0].elapsed_time(ev[1]))
        th.append(ev[1].elapsed_time(ev[2]))
    te.sort()
    th.sort()
    me, mh = te[2], th[2]
    obj.gn_hessian_vec(p2, q2)
    a, b = float(q1 @ p2), float(p1 @ q2)
    sym = abs(a - b) / max(abs(a), abs(b))
    gv = float(g @ p1)
    fds = {}
    for eps in (1e-2, 1e-3, 1e-4, 1e-5):
        fp, fm = obj.eval(y + eps * p1), obj.eval(y - eps * p1)
        fds[eps] = abs((fp - fm) / (2 * eps) - gv) / abs(gv)
    fd = min(fds.values())
    print(name, "gradient FD rel by eps", fds, "J", obj.eval(y), "g.v", gv, flush=True)
    bpv = 20.0 if name == "fast32" else 40.0
    out[name] = {"ms_grad_eval": me, "ms_gn_hv": mh, "gvox_s_step": n / ((me + mh) * 1e6),
                 "gvox_s_hv": n / (mh * 1e6), "hv_frac_canonical": bpv * n / (mh * 1e6) / hbm,
                 "hv_symmetry_rel": sym, "gradient_fd_rel_best": fd, "J": obj.eval(y), "g_dot_p1": gv,
                 "device_mem_used_gb": (torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9}
    print(name, json.dumps(out[name]), flush=True)
    del obj, g, q1, q2
    torch.cuda.empty_cache()
print(json.dumps(out))
