"""Kernel micro-bench: eval(y, grad) and gn_hessian_vec(p) at a given image size.

    python scripts/kbench.py 128 128 128 [--iters 20] [--mode fast]

Prints per-operator device times (CUDA events, L2 flushed between iterations)
and the Hv / eval rates in Gvoxel/s and GB/s of the canonical bytes.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1804_10541_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("m", type=int, nargs=3)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--h", type=float, nargs=3, default=(1.0, 1.0, 1.0))
    ap.add_argument("--no-flush", action="store_true")
    a = ap.parse_args()
    mode = {"fast": P.Mode.FAST, "fast32": P.Mode.FAST32, "parity": P.Mode.PARITY}[a.mode]
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
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    te, th = [], []
    for it in range(a.iters + 3):
        if not a.no_flush:
            flush.fill_(float(it))
        ev[0].record()
        obj.eval(y, g)
        ev[1].record()
        obj.gn_hessian_vec(p, q)
        ev[2].record()
        torch.cuda.synchronize()
        if it >= 3:
            te.append(ev[0].elapsed_time(ev[1]))
            th.append(ev[1].elapsed_time(ev[2]))
    te.sort()
    th.sort()
    n = img.count()
    me, mh = te[len(te) // 2], th[len(th) // 2]
    print(f"m={tuple(a.m)} n={n/1e6:.1f}M eval {me*1e3:.1f} us ({n/me/1e6:.2f} Gvox/s, {48*n/me/1e6:.0f} GB/s canon) "
          f"hv {mh*1e3:.1f} us ({n/mh/1e6:.2f} Gvox/s, {40*n/mh/1e6:.0f} GB/s canon, frac {40*n/mh/1e6/6550:.3f})")


if __name__ == "__main__":
    main()
