"""Command line of the B200 path, mirroring the reference CLI (tools/mfreg_cli.cpp:26-158):

    python -m paper_1804_10541_b200 register --fixed F.mha --moving M.mha --out-deformation y.def
                                         [--out-warped W.mha] [--alpha 1] [--tau 10] [--edge-rho 10]
                                         [--levels 3] [--deform-ratio 4] [--optimizer lbfgs|gn]
                                         [--max-iters 20] [--mode parity|fast|fast32]
    python -m paper_1804_10541_b200 warp --input V.mha --deformation y.def --out W.mha
    python -m paper_1804_10541_b200 eval-landmarks --fixed-landmarks f.txt --moving-landmarks m.txt
                                         --deformation y.def [--spacing sx sy sz]

    python -m paper_1804_10541_b200 selftest [--seed 1234] [--quick]

Same options, defaults and printed keys as the reference (`--threads` has no
counterpart: the device path has no CPU worker pool). The extra `--mode`
selects the execution mode; `parity` (default) reproduces the reference's
numbers bit for bit. `selftest` runs the reference's self-consistency suites
(mfreg_cli.cpp:171-296) on the device: the sparse-matrix oracle checks become
fast-vs-parity checks (the parity objective is the bitwise replica of the
reference), plus grid-transfer adjointness, GN symmetry / PSD and the
finite-difference gradient check.
"""
from __future__ import annotations

import argparse
import sys
import time

import numpy as np


def _cmd_register(a) -> int:
    import paper_1804_10541_b200 as P
    fixed, img = P.io.read_volume(a.fixed)
    moving, img_m = P.io.read_volume(a.moving)
    if img_m.m != img.m:  # build_pyramid (multilevel.cpp:13-17)
        raise ValueError("build_pyramid: image sizes differ")
    mode = {"parity": P.Mode.PARITY, "fast": P.Mode.FAST, "fast32": P.Mode.FAST32}[a.mode]
    cfg = P.MultilevelConfig(levels=a.levels, deform_ratio=a.deform_ratio, ngf=P.NgfParams(a.tau, a.edge_rho),
                             alpha=a.alpha, method=P.Method.GAUSS_NEWTON if a.optimizer == "gn" else P.Method.LBFGS,
                             opt=P.OptimizerConfig(max_iters=a.max_iters), mode=mode)
    P.device_memory_peak(reset=True)
    t0 = time.perf_counter()
    y, dg, levels = P.register_multilevel(fixed, moving, img, cfg)
    elapsed = time.perf_counter() - t0
    out = sys.stdout.write
    out("command: register\n")
    out(f"fixed: {a.fixed}\nmoving: {a.moving}\n")
    out(f"alpha: {a.alpha:g}\ntau: {a.tau:g}\nedge-rho: {a.edge_rho:g}\nlevels: {a.levels}\n")
    out(f"optimizer: {a.optimizer}\n")
    # per-level grids as the multilevel driver built them (multilevel.cpp:9-49)
    sizes = [img]
    for _ in range(1, a.levels):
        g = sizes[-1]
        sizes.append(P.GridDesc(tuple((m + 1) // 2 for m in g.m), tuple(2 * h for h in g.h), False))
    sizes = sizes[::-1]  # coarsest first, as the result's levels
    for l, (trace, _) in enumerate(levels):
        ig = sizes[l]
        lg = P.deformation_grid_for(ig, a.deform_ratio)
        out(f"level.{l}.image-size: {ig.m[0]} {ig.m[1]} {ig.m[2]}\n")
        out(f"level.{l}.deform-size: {lg.m[0]} {lg.m[1]} {lg.m[2]}\n")
        out(f"level.{l}.iterations: {len(trace)}\n")
        for it in trace:
            out(f"level.{l}.iter.{it.iter}: J={it.j:.10e} D={it.distance:.10e} aS={it.regularizer:.10e} "
                f"grad={it.grad_norm:.4e} step={it.step:.3g} cg={it.cg_iters}\n")
    u = (np.asarray(y) - dg.point_coords()).reshape(3, -1)
    disp = np.sqrt((u * u).sum(axis=0))
    out(f"final.max-displacement: {disp.max():.6e}\nfinal.mean-displacement: {disp.mean():.6e}\n")
    out(f"runtime-seconds: {elapsed:.3f}\n")
    # the reference reports its host scratch peak (counters.hpp:30-47); here: the device high-water
    # mark of the library's allocations during the registration
    out(f"peak-derivative-buffer-bytes: {P.device_memory_peak()}\n")
    P.io.write_deformation(a.out_deformation, y, dg)
    out(f"wrote-deformation: {a.out_deformation}\n")
    if a.out_warped:
        P.io.write_volume(a.out_warped, P.io.warp_volume(moving, img, y, dg), img)
        out(f"wrote-warped: {a.out_warped}\n")
    return 0


def _cmd_warp(a) -> int:
    import paper_1804_10541_b200 as P
    P.io.warp_files(a.input, a.deformation, a.out)
    sys.stdout.write(f"command: warp\nwrote: {a.out}\n")
    return 0


def _cmd_eval_landmarks(a) -> int:
    import paper_1804_10541_b200 as P
    fixed = P.io.read_landmarks(a.fixed_landmarks, a.spacing)
    moving = P.io.read_landmarks(a.moving_landmarks, a.spacing)
    dg = P.io.read_deformation_grid(a.deformation)
    y = P.io.read_deformation(a.deformation, dg)
    b = P.io.landmark_error(fixed, moving, dg.point_coords(), dg)
    f = P.io.landmark_error(fixed, moving, y, dg)
    sys.stdout.write(f"command: eval-landmarks\nlandmarks: {b[2]}\n")
    sys.stdout.write(f"error-before: {b[0]:.6f} +- {b[1]:.6f}\nerror-after: {f[0]:.6f} +- {f[1]:.6f}\n")
    return 0


def _cmd_selftest(a) -> int:
    import paper_1804_10541_b200 as P
    failures = 0

    def check(name, ok):
        nonlocal failures
        sys.stdout.write(f"selftest.{name}: {'pass' if ok else 'FAIL'}\n")
        failures += 0 if ok else 1

    # 6^3 image, 4^3 nodes, smoothed random volumes, tau = rho = 1 (mfreg_cli.cpp:172-180)
    rng = np.random.default_rng(a.seed)
    m = (6, 6, 6)
    img = P.make_image_grid(m)
    dg = P.make_deform_grid(img, (4, 4, 4))

    def smooth_random():
        v = rng.uniform(0.0, 1.0, m[::-1])
        p = np.pad(v, 1, mode="edge")
        s_ = (p[1:-1, 1:-1, 1:-1] + p[:-2, 1:-1, 1:-1] + p[2:, 1:-1, 1:-1] + p[1:-1, :-2, 1:-1] + p[1:-1, 2:, 1:-1]
              + p[1:-1, 1:-1, :-2] + p[1:-1, 1:-1, 2:]) / 7.0
        return np.ascontiguousarray(s_.ravel())

    R, T = smooth_random(), smooth_random()
    objs = {md: P.Objective(R, T, img, dg, P.NgfParams(1.0, 1.0), 1.0, md) for md in (P.Mode.PARITY, P.Mode.FAST)}
    y = objs[P.Mode.PARITY].identity() + rng.uniform(-0.3, 0.3, 3 * dg.count())
    grads = {}
    for md, o in objs.items():
        g = np.empty(o.dof())
        o.eval(y, g)
        grads[md] = g
    scale = max(1.0, float(np.max(np.abs(grads[P.Mode.PARITY]))))
    check("parity-gradient", float(np.max(np.abs(grads[P.Mode.FAST] - grads[P.Mode.PARITY]))) <= 1e-12 * scale)
    p = rng.uniform(-0.3, 0.3, y.size)
    qp = objs[P.Mode.PARITY].gn_hessian_vec(p)
    qf = objs[P.Mode.FAST].gn_hessian_vec(p)
    scale = max(1.0, float(np.max(np.abs(qp))))
    check("parity-hvp", float(np.max(np.abs(qf - qp))) <= 1e-12 * scale)
    w = rng.uniform(-0.3, 0.3, 3 * img.count())
    a_ = float(np.dot(P.transfer_apply(dg, img, y), w))
    b_ = float(np.dot(y, P.transfer_apply_transpose(dg, img, w)))
    check("transfer-adjoint", abs(a_ - b_) <= 1e-12 * max(1.0, abs(a_)))
    obj = objs[P.Mode.PARITY]
    sym = psd = True
    for _ in range(3 if a.quick else 10):
        p = rng.uniform(-0.3, 0.3, y.size)
        r = rng.uniform(-0.3, 0.3, y.size)
        q, hq = obj.gn_hessian_vec(p), obj.gn_hessian_vec(r)
        sym = sym and abs(float(q @ r) - float(p @ hq)) <= 1e-12 * max(1.0, abs(float(q @ r)))
        psd = psd and float(q @ p) >= -1e-10 * float(p @ p)
    check("gn-symmetry", sym)
    check("gn-psd", psd)
    if not a.quick:
        g = np.empty(obj.dof())
        obj.eval(y, g)
        ok = True
        for _ in range(5):
            v = rng.uniform(-0.3, 0.3, y.size)
            gv = float(g @ v)
            best = 1e9
            for eps in (1e-4, 1e-5, 1e-6):
                fp, fm = obj.eval(y + eps * v), obj.eval(y - eps * v)
                best = min(best, abs((fp - fm) / (2.0 * eps) - gv) / max(1e-12, abs(gv)))
            ok = ok and best <= 1e-6
        check("gradient-fd", ok)
    sys.stdout.write(f"selftest.failures: {failures}\n")
    return 0 if failures == 0 else 1


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1804_10541_b200",
                                 description="Deformable 3D image registration (NGF + curvature), B200 path")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("register", help="register a moving volume onto a fixed volume")
    r.add_argument("--fixed", required=True)
    r.add_argument("--moving", required=True)
    r.add_argument("--out-deformation", required=True)
    r.add_argument("--out-warped", default="")
    r.add_argument("--alpha", type=float, default=1.0)
    r.add_argument("--tau", type=float, default=10.0)
    r.add_argument("--edge-rho", type=float, default=10.0)
    r.add_argument("--levels", type=int, default=3)
    r.add_argument("--deform-ratio", type=int, default=4)
    r.add_argument("--optimizer", choices=["lbfgs", "gn"], default="lbfgs")
    r.add_argument("--max-iters", type=int, default=20)
    r.add_argument("--mode", choices=["parity", "fast", "fast32"], default="parity")
    w = sub.add_parser("warp", help="apply a stored deformation to a volume")
    w.add_argument("--input", required=True)
    w.add_argument("--deformation", required=True)
    w.add_argument("--out", required=True)
    e = sub.add_parser("eval-landmarks", help="landmark error before/after registration")
    e.add_argument("--fixed-landmarks", required=True)
    e.add_argument("--moving-landmarks", required=True)
    e.add_argument("--deformation", required=True)
    e.add_argument("--spacing", type=float, nargs=3, default=[1.0, 1.0, 1.0])
    st = sub.add_parser("selftest", help="run built-in derivative verification suites")
    st.add_argument("--seed", type=int, default=1234)
    st.add_argument("--quick", action="store_true")
    a = ap.parse_args(argv)
    try:
        return {"register": _cmd_register, "warp": _cmd_warp, "eval-landmarks": _cmd_eval_landmarks,
                "selftest": _cmd_selftest}[a.cmd](a)
    except Exception as ex:  # the reference CLI: "error: <what>" on stderr, exit 1
        sys.stderr.write(f"error: {ex}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
