"""Host-buffer call timing at C4: eval / gn_hessian_vec with pinned host buffers (pipelined copies)
against the same calls on device buffers, wall clock per call (median of --reps).

    python scripts/pipe_probe.py [--reps 7] [--mode fast]
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1804_10541_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--m", type=int, nargs=3, default=(512, 512, 900))
    a = ap.parse_args()
    img = P.make_image_grid(a.m, (0.7, 0.7, 0.7))
    dg = P.deformation_grid_for(img, 4)
    R = P.make_phantom(img, device=True)
    R.mul_(1000.0)
    T = P.warp_sinusoid(R, img, 3.0, 42)
    mode = {"fast": P.Mode.FAST, "fast32": P.Mode.FAST32}[a.mode]
    obj = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, mode)
    nd = 3 * dg.count()
    gen = torch.Generator(device="cuda").manual_seed(3)
    y = torch.from_numpy(dg.point_coords()).cuda() + (torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 0.6 - 0.3)
    p = torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 2.0 - 1.0
    g = torch.empty_like(y)
    q = torch.empty_like(y)
    yh, ph = y.cpu().pin_memory().numpy(), p.cpu().pin_memory().numpy()
    gh = torch.empty(nd, dtype=torch.float64).pin_memory().numpy()
    qh = torch.empty(nd, dtype=torch.float64).pin_memory().numpy()

    def timed(fn):
        ts = []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts)

    for _ in range(2):
        obj.eval(y, g)
        obj.gn_hessian_vec(p, q)
        obj.eval(yh, gh)
        obj.gn_hessian_vec(ph, qh)
    r = {"eval_dev": timed(lambda: obj.eval(y, g)), "hv_dev": timed(lambda: obj.gn_hessian_vec(p, q)),
         "eval_host": timed(lambda: obj.eval(yh, gh)), "hv_host": timed(lambda: obj.gn_hessian_vec(ph, qh))}
    print(" ".join(f"{k} {v:.3f} ms" for k, v in r.items()), f"(nodal vector {nd * 8 / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
