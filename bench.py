"""Benchmark: NGF + curvature derivative evaluation on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): 128^3 synthetic CT-like phantom (x1000)
warped by a sinusoid (amp 3 voxels, seed 42), nodal grid 33^3 (ratio 4), tau =
rho = 10, alpha = 1; y = identity + U(-0.3, 0.3), p ~ U(-1, 1).

One step = one gradient evaluation Objective::eval(y, grad) + one Gauss-Newton
Hessian-vector product Objective::gn_hessian_vec(p) — the two derivative
operators the GN/CG solver is made of. `value` counts
image voxels processed by derivative evaluations per second (2 m per step),
inputs resident in HBM, L2 flushed between steps, device time from CUDA events.
`e2e` is the same step through the C ABI with HOST buffers (y, p in; grad, q
out), so H2D/D2H copies are inside the timed region. The full 3-level
Gauss-Newton registration of the same pair (the metric's second half) is timed
once and reported under `gn_registration`.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode fast|parity]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M = (128, 128, 128)
H = (1.0, 1.0, 1.0)
RATIO = 4
LEVELS = 3
B_CANON_GRAD = 48.0  # R, T read; T_w, dT written (fp64)
B_CANON_HV = 40.0    # R, T_w, dT read (fp64)
# dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu --set full
# capture of the same workload (profiles/), or None when not captured for this build
TRAFFIC = {"hv_pass": 171.05e6, "eval_pass": 147.62e6, "warp": 29.42e6}  # bytes/launch, profiles/r1c_ncu_full.md
METRIC = "NGF+curvature derivative eval Gvoxel/s (%HBM roofline); full GN registration wall s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["fast", "parity"], default="fast")
    ap.add_argument("--no-gn", action="store_true", help="skip the full GN registration timing")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-c4", action="store_true", help="skip the 512x512x900 (C4) registrations")
    return ap.parse_args()


def dist_init(n):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        # one GPU per rank; MFREG_BENCH_BACKEND=gloo (with ranks sharing devices) exercises the
        # N > 1 code path on a single-GPU box — never used for reported numbers
        backend = os.environ.get("MFREG_BENCH_BACKEND", "nccl")
        local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            try:
                pw.append(float(parts[2]))
            except ValueError:
                pass
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "sm_mhz_min": min(sm) if sm else None, "power_w_max": max(pw) if pw else None}


def measured_hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def make_inputs_gpu(P, torch):
    img = P.make_image_grid(M, H)
    dg = P.deformation_grid_for(img, RATIO)
    R = P.make_phantom(img, device=True)
    R.mul_(1000.0)
    T = P.warp_sinusoid(R, img, 3.0, 42)
    gen = torch.Generator(device="cuda").manual_seed(8)
    nd = 3 * dg.count()
    xid = torch.from_numpy(dg.point_coords()).cuda()
    y = xid + (torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 0.6 - 0.3)
    p = torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 2.0 - 1.0
    return img, dg, R, T, y, p


def cpu_reference_rate(R, T, y, p, steps: int, threads: int):
    """Reference CPU implementation (oracle/_ref, else the C port) timed on host cores."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("ref") else "port"
    o = Oracle("ref" if kind == "reference" else "port")
    o.set_threads(threads)
    my = [((M[a] + RATIO - 1) // RATIO + 1) for a in range(3)]
    obj = o.objective(R, T, M, H, my, 10.0, 10.0, 1.0)
    obj.eval(y)  # warm
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        obj.eval(y)
        obj.gn_hessian_vec(p)
        ts.append(time.perf_counter() - t0)
    n = int(np.prod(M))
    t = statistics.median(ts)
    return 2.0 * n / t / 1e9, kind, (threads if kind == "reference" else 1), t


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    import torch
    import paper_1804_10541_b200 as P
    torch.cuda.set_device(0)
    img, dg, R, T, y, p = make_inputs_gpu(P, torch)
    R, T, y, p = (x.cpu().numpy() for x in (R, T, y, p))
    threads = os.cpu_count() or 1
    steps = max(1, min(args.steps, 5))
    rate, kind, cores, t = cpu_reference_rate(R, T, y, p, steps, threads)
    line = {"metric": METRIC, "value": rate, "unit": "Gvoxel/s", "n_gpus": world, "steps": steps,
            "warmup": 1, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (phantom x1000, sinusoid warp amp 3 seed 42)",
            "config": {"workload": "C2 finest level: 128^3 image / 33^3 nodal, eval(grad) + gn_hessian_vec",
                       "image": list(M), "nodal": list(dg.m), "threads": threads},
            "impl": "reference",
            "cpu_baseline": {"value": rate, "unit": "Gvoxel/s", "cores": cores, "kind": kind,
                             "sample": f"{steps} steps of eval(y,grad)+gn_hessian_vec(p) at 128^3, median"},
            "e2e": {"value": rate, "unit": "Gvoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    import torch
    import paper_1804_10541_b200 as P
    torch.cuda.set_device(local)
    mode = P.Mode.FAST if args.mode == "fast" else P.Mode.PARITY
    img, dg, R, T, y, p = make_inputs_gpu(P, torch)
    n = img.count()
    nd = 3 * dg.count()
    obj = P.Objective(R, T, img, dg, P.NgfParams(10.0, 10.0), 1.0, mode)
    grad = torch.empty_like(y)
    q = torch.empty_like(y)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")  # > 126 MB L2

    def step():
        obj.eval(y, grad)
        obj.gn_hessian_vec(p, q)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0 = P.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    with Clocks(local) as ck:
        for k in range(args.steps):
            flush.zero_()
            a, b, c = ev[k]
            a.record()
            obj.eval(y, grad)
            b.record()
            obj.gn_hessian_vec(p, q)
            c.record()
        torch.cuda.synchronize()
    barrier(world)
    launches = P.launch_count() - l0
    t_eval = [e[0].elapsed_time(e[1]) for e in ev]
    t_hv = [e[1].elapsed_time(e[2]) for e in ev]
    ms_step = max_over_ranks(sum(t_eval) / args.steps + sum(t_hv) / args.steps, world)
    ms_eval = statistics.mean(t_eval)
    ms_hv = statistics.mean(t_hv)
    value = 2.0 * n * world / (ms_step * 1e-3) / 1e9
    clocks = ck.summary()

    # e2e through the C ABI with HOST buffers (pinned; H2D of y, p and D2H of grad, q inside
    # the timed region, every step)
    yh = y.cpu().pin_memory().numpy()
    ph = p.cpu().pin_memory().numpy()
    gh = torch.empty(nd, dtype=torch.float64).pin_memory().numpy()
    qh = torch.empty(nd, dtype=torch.float64).pin_memory().numpy()
    for _ in range(2):
        obj.eval(yh, gh)
        obj.gn_hessian_vec(ph, qh)
    barrier(world)
    t0 = time.perf_counter()
    k_e2e = max(3, args.steps // 2)
    for _ in range(k_e2e):
        obj.eval(yh, gh)
        obj.gn_hessian_vec(ph, qh)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / k_e2e, world)
    e2e = {"value": 2.0 * n * world / e2e_s / 1e9, "unit": "Gvoxel/s", "h2d_bytes_per_step": 2 * nd * 8,
           "d2h_bytes_per_step": 2 * nd * 8 + 16, "ms_per_step": e2e_s * 1e3}

    peak, peak_kind = measured_hbm_peak()
    roofline = None
    if mode == P.Mode.FAST:
        # per-kernel device time: CUDA events recorded on the launching stream inside the
        # library, L2 flushed (256 MB write) before every launch (outside the interval)
        reps = max(5, args.steps)
        obj.eval(y, grad)
        k_ms = {"hv_pass": obj.profile_kernel(0, p, reps), "eval_pass": obj.profile_kernel(1, p, reps),
                "warp": obj.profile_kernel(2, y, reps)}
        obj.eval(y, grad)
        # algorithmic bytes per image voxel: Hv pass reads the
        # canonical state R, T_w, dT (40 B); eval pass reads R, T_w, dT (40 B); warp reads T
        # and writes T_w, dT (8 + 32 B)
        b_alg = {"hv_pass": B_CANON_HV, "eval_pass": 40.0, "warp": 40.0}
        kern = {k: {"ms": v, "achieved_gbs": b_alg[k] * n / (v * 1e-3) / 1e9, "algorithmic_bytes_per_voxel": b_alg[k],
                    "frac": b_alg[k] * n / (v * 1e-3) / 1e9 / peak} for k, v in k_ms.items()}
        dom = max(k_ms, key=k_ms.get)
        names = {"hv_pass": "k_hv2 (GN Hv image pass: P p, dr, dr^T, dT, P^T partials)",
                 "eval_pass": "k_ev2 (NGF eval pass: rho-hat, r, D partials, gradient dr^T r, P^T partials)",
                 "warp": "k_warp_fast (P y, trilinear T, dT/dP)"}
        roofline = {"bound": "hbm", "achieved": kern[dom]["achieved_gbs"], "peak": peak, "unit": "GB/s",
                    "frac": kern[dom]["frac"], "traffic": TRAFFIC.get(dom), "traffic_unit": "bytes/launch (ncu dram read+write)",
                    "algorithmic_bytes_per_launch": b_alg[dom] * n, "kernel": names[dom],
                    "algorithmic_bytes_per_voxel": b_alg[dom], "units_per_launch": n, "peak_source": peak_kind,
                    "kernels": kern,
                    "operators": {"gn_hessian_vec": {"ms": ms_hv, "frac": B_CANON_HV * n / (ms_hv * 1e-3) / 1e9 / peak},
                                  "eval_grad": {"ms": ms_eval, "frac": B_CANON_GRAD * n / (ms_eval * 1e-3) / 1e9 / peak}}}

    gn = None
    if not args.no_gn:
        cfg = P.MultilevelConfig(levels=LEVELS, deform_ratio=RATIO, method=P.Method.GAUSS_NEWTON, mode=mode)
        P.register_multilevel(R, T, img, P.MultilevelConfig(levels=LEVELS, method=P.Method.GAUSS_NEWTON, mode=mode,
                                                              opt=P.OptimizerConfig(max_iters=1)))
        walls = []
        for _ in range(3):  # host-driven solver loops: median of 3 runs (single runs vary 2x on a busy host)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            yy, dgf, levels = P.register_multilevel(R, T, img, cfg)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        wall = max_over_ranks(statistics.median(walls), world)
        gn = {"wall_s": wall, "wall_s_runs": walls, "mode": args.mode, "levels": LEVELS,
              "outer_iters": [len(t) for t, _ in levels],
              "cg_iters": int(sum(r.cg_iters for t, _ in levels for r in t)),
              "final_J": levels[-1][0][-1].j if levels[-1][0] else None,
              "reference_cpu_s_8thr_container": 519.0}

    # the optional fp32 mode (FAST32) on the same workload: operator rate and kernel times
    fast32 = None
    if mode == P.Mode.FAST and world == 1:
        o32 = P.Objective(R, T, img, dg, P.NgfParams(10.0, 10.0), 1.0, P.Mode.FAST32)
        for _ in range(3):
            o32.eval(y, grad)
            o32.gn_hessian_vec(p, q)
        torch.cuda.synchronize()
        ev32 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for a_, b_ in ev32:
            flush.zero_()
            a_.record()
            o32.eval(y, grad)
            o32.gn_hessian_vec(p, q)
            b_.record()
        torch.cuda.synchronize()
        ms32 = statistics.mean(a_.elapsed_time(b_) for a_, b_ in ev32)
        reps = max(5, args.steps)
        k32 = {"hv_pass": o32.profile_kernel(0, p, reps), "eval_pass": o32.profile_kernel(1, p, reps),
               "warp": o32.profile_kernel(2, y, reps)}
        fast32 = {"value": 2.0 * n / (ms32 * 1e-3) / 1e9, "unit": "Gvoxel/s", "ms_per_step": ms32,
                  "kernels_ms": k32, "tolerance": "max-rel 1e-4 vs reference (tests/test_gpu_fast32.py)",
                  "algorithmic_bytes_per_voxel_hv": 20.0,
                  "hv_frac": 20.0 * n / (k32["hv_pass"] * 1e-3) / 1e9 / peak}
        del o32

    # north-star case C4: full 3-level GN registration of a 512x512x900 pair on this GPU,
    # fp64 (FAST) and the optional fp32 mode (FAST32); wall clock from the host
    gn_c4 = None
    if not args.no_c4 and world == 1 and mode == P.Mode.FAST:
        gn_c4 = {"image": [512, 512, 900], "levels": LEVELS, "method": "gauss-newton"}
        img4 = P.make_image_grid((512, 512, 900), H)
        R4 = P.make_phantom(img4, device=True)
        R4.mul_(1000.0)
        T4 = P.warp_sinusoid(R4, img4, 3.0, 42)
        ck4 = Clocks(local).__enter__()  # clocks over the C4 runs (sustained load: power cap shows here)
        for name, md in (("fast", P.Mode.FAST), ("fast32", P.Mode.FAST32)):
            cfg4 = P.MultilevelConfig(levels=LEVELS, deform_ratio=RATIO, method=P.Method.GAUSS_NEWTON, mode=md)
            walls = []
            for _ in range(2):  # cold (first registration in the process), then warm (pooled memory)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _, _, lv4 = P.register_multilevel(R4, T4, img4, cfg4)
                torch.cuda.synchronize()
                walls.append(time.perf_counter() - t0)
            gn_c4[name] = {"wall_s": walls[0], "wall_s_warm": walls[1], "outer_iters": [len(t) for t, _ in lv4],
                           "cg_iters": int(sum(r.cg_iters for t, _ in lv4 for r in t)),
                           "final_J": lv4[-1][0][-1].j if lv4[-1][0] else None}
        ck4.__exit__(None, None, None)
        gn_c4["clocks"] = ck4.summary()
        del R4, T4

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        rate, kind, cores, t = cpu_reference_rate(R.cpu().numpy(), T.cpu().numpy(), yh, ph, 3, threads)
        cpu = {"value": rate, "unit": "Gvoxel/s", "cores": cores, "kind": kind,
               "sample": f"3 steps of eval(y,grad)+gn_hessian_vec(p) at 128^3 ({t:.2f} s/step median)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "Gvoxel/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (phantom x1000, sinusoid warp amp 3 seed 42)",
                "config": {"workload": "C2 finest level: 128^3 image / 33^3 nodal, eval(grad) + gn_hessian_vec",
                           "image": list(M), "nodal": list(dg.m), "mode": args.mode,
                           "l2": "flushed between steps (256 MB write); per-step state 350 MB > L2",
                           "parallelism": "single GPU"},
                "ms_grad_eval": ms_eval, "ms_gn_hv": ms_hv,
                "gvox_s_grad_eval": n / (ms_eval * 1e-3) / 1e9, "gvox_s_gn_hv": n / (ms_hv * 1e-3) / 1e9,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "gn_registration": gn, "gn_registration_c4": gn_c4,
                "fast32": fast32}
        print(json.dumps(line), flush=True)


def run_slabs(args, rank, world, local):
    """N > 1: weak scaling over z slabs. The global volume is
    128 x 128 x (128 N) (nodal 33 x 33 x (32 N + 1)); rank r evaluates its
    128-plane slab. Every step performs the real halo exchanges, shared-plane
    sums and scalar all-gathers over NCCL (slab.py)."""
    import torch
    import paper_1804_10541_b200 as P
    torch.cuda.set_device(local)
    if args.mode != "fast":
        raise SystemExit("z slabs run in fast mode")
    gm = (M[0], M[1], M[2] * world)
    img = P.make_image_grid(gm, H)
    dg = P.deformation_grid_for(img, RATIO)
    R = P.make_phantom(img, device=True)
    R.mul_(1000.0)
    T = P.warp_sinusoid(R, img, 3.0, 42)
    gen = torch.Generator(device="cuda").manual_seed(8)
    nd = 3 * dg.count()
    y = torch.from_numpy(dg.point_coords()).cuda() + (torch.rand(nd, generator=gen, device="cuda",
                                                                 dtype=torch.float64) * 0.6 - 0.3)
    p = torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 2.0 - 1.0
    so = P.slab.SlabObjective(R, T, img, dg, P.NgfParams(10.0, 10.0), 1.0, P.slab.TorchComm())
    s = so.info
    n_loc = (s.zhi - s.zlo) * gm[0] * gm[1]
    n_glob = img.count()
    grad = torch.zeros_like(y)
    q = torch.zeros_like(y)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        so.eval(y, grad)
        so.gn_hessian_vec(p, q)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0 = P.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    with Clocks(local) as ck:
        for k in range(args.steps):
            flush.zero_()
            a, b, c = ev[k]
            a.record()
            so.eval(y, grad)
            b.record()
            so.gn_hessian_vec(p, q)
            c.record()
        torch.cuda.synchronize()
    barrier(world)
    launches = P.launch_count() - l0
    t_eval = [e[0].elapsed_time(e[1]) for e in ev]
    t_hv = [e[1].elapsed_time(e[2]) for e in ev]
    ms_step = max_over_ranks(sum(t_eval) / args.steps + sum(t_hv) / args.steps, world)
    ms_eval = max_over_ranks(statistics.mean(t_eval), world)
    ms_hv = max_over_ranks(statistics.mean(t_hv), world)
    value = 2.0 * n_glob / (ms_step * 1e-3) / 1e9
    clocks = ck.summary()
    # e2e: y, p from pinned host memory, grad and q back to the host, every step
    yh, ph = y.cpu().pin_memory(), p.cpu().pin_memory()
    gh, qh = torch.empty_like(yh).pin_memory(), torch.empty_like(ph).pin_memory()
    yd, pd = torch.empty_like(y), torch.empty_like(p)

    def e2e_step():
        yd.copy_(yh, non_blocking=True)
        pd.copy_(ph, non_blocking=True)
        so.eval(yd, grad)
        so.gn_hessian_vec(pd, q)
        gh.copy_(grad, non_blocking=True)
        qh.copy_(q, non_blocking=True)
        torch.cuda.synchronize()

    e2e_step()
    barrier(world)
    t0 = time.perf_counter()
    k_e2e = max(3, args.steps // 2)
    for _ in range(k_e2e):
        e2e_step()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / k_e2e, world)
    e2e = {"value": 2.0 * n_glob / e2e_s / 1e9, "unit": "Gvoxel/s", "h2d_bytes_per_step": 2 * nd * 8 * world,
           "d2h_bytes_per_step": 2 * nd * 8 * world, "ms_per_step": e2e_s * 1e3}
    peak, peak_kind = measured_hbm_peak()
    achieved = B_CANON_HV * n_loc / (ms_hv * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None, "kernel": "gn_hessian_vec per rank (slab incl. halo exchange)",
                "algorithmic_bytes_per_voxel": B_CANON_HV, "peak_source": peak_kind}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "Gvoxel/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (phantom x1000, sinusoid warp amp 3 seed 42)",
                "config": {"workload": f"C2 finest level per GPU: 128^3 image slab of {list(gm)} / nodal {list(dg.m)}, "
                                       "eval(grad) + gn_hessian_vec",
                           "image": list(gm), "nodal": list(dg.m), "mode": args.mode,
                           "l2": "flushed between steps (256 MB write)",
                           "parallelism": f"z slabs x{world} (halo exchange + shared-plane sums over NCCL)"},
                "ms_grad_eval": ms_eval, "ms_gn_hv": ms_hv, "roofline": roofline, "cpu_baseline": None,
                "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
                "gn_registration": None}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_init(args.gpus)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    elif world > 1:
        run_slabs(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
