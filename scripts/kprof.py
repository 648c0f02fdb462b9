"""Per-kernel device times of the fast image passes (CUDA events on the launching stream, L2
flushed before every launch) at one workload; for A/B runs of kernel variants.

    python scripts/kprof.py [--m 512 512 900] [--h 0.7 0.7 0.7] [--mode fast|fast32] [--reps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1804_10541_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, nargs=3, default=(512, 512, 900))
    ap.add_argument("--h", type=float, nargs=3, default=(0.7, 0.7, 0.7))
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    mode = {"fast": P.Mode.FAST, "fast32": P.Mode.FAST32}[a.mode]
    img = P.make_image_grid(a.m, a.h)
    dg = P.deformation_grid_for(img, 4)
    R = P.make_phantom(img, device=True)
    R.mul_(1000.0)
    T = P.warp_sinusoid(R, img, 3.0, 42)
    gen = torch.Generator(device="cuda").manual_seed(8)
    nd = 3 * dg.count()
    y = torch.from_numpy(dg.point_coords()).cuda() + (torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 0.6 - 0.3)
    p = torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 2.0 - 1.0
    obj = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, mode)
    g = torch.empty_like(y)
    q = torch.empty_like(y)
    for _ in range(3):
        j = obj.eval(y, g)
        obj.gn_hessian_vec(p, q)
    torch.cuda.synchronize()
    n = img.count()
    out = {"tag": a.tag, "m": a.m, "mode": a.mode, "J": j, "gsum": float(g.abs().sum()), "qsum": float(q.abs().sum())}
    for name, which, opnd in (("hv_pass", 0, p), ("eval_pass", 1, p), ("warp", 2, y)):
        ms = obj.profile_kernel(which, opnd, a.reps)
        out[name] = {"ms": round(ms, 4), "gvox_s": round(n / ms / 1e6, 2), "frac40": round(40 * n / ms / 1e6 / 6554.9, 4)}
    # operator times (events around the calls): gradient eval, value-only eval (Armijo trial), GN Hv
    def ev_ms(fn, reps=a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return round(e0.elapsed_time(e1) / reps, 4)
    out["op_ms"] = {"eval_grad": ev_ms(lambda: obj.eval(y, g)), "eval_value": ev_ms(lambda: obj.eval(y)),
                    "gn_hv": ev_ms(lambda: (obj.eval(y, g), obj.gn_hessian_vec(p, q)), 3)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
