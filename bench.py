"""Benchmark: NGF + curvature derivative evaluation on B200 (BASELINE.json metric).

Headline workload (BASELINE.json configs[3], "C4", the largest configuration that fits one
GPU): the finest level of the 512x512x900 thorax-abdomen-shaped pair, spacing h = 0.7 (the
interpolation-tie hazard of SURVEY H1), nodal grid 129x129x226 (ratio 4); R = the
reference's phantom x1000, T = R warped by its sinusoid (amp 3 voxels, seed 42), tau = rho
= 10, alpha = 1; y = identity + U(-0.3, 0.3), p ~ U(-1, 1).

One step = one gradient evaluation Objective::eval(y, grad) + one Gauss-Newton
Hessian-vector product Objective::gn_hessian_vec(p) — the two derivative operators the
GN/CG solver is made of. `value` counts image voxels processed by
derivative evaluations per second (2 m per step), inputs resident in HBM (per-step state
> 20 GB, far larger than L2; L2 also flushed between steps), device time from CUDA events.
`e2e` is the same step through the C ABI with HOST buffers (y, p in; grad, q out), so the
H2D/D2H copies are inside the timed region. The full 3-level Gauss-Newton registration of
the C4 pair (the metric's second half) is timed under `gn_registration_c4`.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c2] [--mode fast|parity]
"""
from __future__ import annotations

import argparse
import hashlib
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

RATIO = 4
LEVELS = 3
# (image size, spacing, CPU-baseline sample of the same workload)
WORKLOADS = {
    "c4": {"m": (512, 512, 900), "h": (0.7, 0.7, 0.7), "sample_m": (512, 512, 24),
           "name": "C4 finest level: 512x512x900 image (h=0.7) / 129x129x226 nodal, eval(grad) + gn_hessian_vec"},
    "c2": {"m": (128, 128, 128), "h": (1.0, 1.0, 1.0), "sample_m": (128, 128, 128),
           "name": "C2 finest level: 128^3 image / 33^3 nodal, eval(grad) + gn_hessian_vec"},
    # BASELINE configs[4]: the derivative-only sweep (no registration; fp64 state ~103 GB on one
    # GPU, so the FAST32 line, which would need a second objective, is left out)
    "c5": {"m": (1024, 1024, 1024), "h": (1.0, 1.0, 1.0), "sample_m": (1024, 1024, 8), "derivative_only": True,
           "name": "C5 derivative sweep: 1024^3 image / 257^3 nodal, eval(grad) + gn_hessian_vec"},
}
B_CANON_GRAD = 48.0  # R, T read; T_w, dT written (fp64)
B_CANON_HV = 40.0    # R, T_w, dT read (fp64)
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")  # written by scripts/ncu_traffic.py
METRIC = "NGF+curvature derivative eval Gvoxel/s (%HBM roofline); full GN registration wall s"
DATA = "synthetic (reference phantom x1000, sinusoid warp amp 3 seed 42)"


def csrc_sha() -> str:
    """Hash of the CUDA sources: an ncu traffic capture is only quoted for the build it measured."""
    d = os.path.join(ROOT, "paper_1804_10541_b200", "csrc")
    h = hashlib.sha256()
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh")):
            with open(os.path.join(d, f), "rb") as fh:
                h.update(f.encode() + fh.read())
    return h.hexdigest()[:16]


def traffic_for(workload: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture
    of this workload and source hash (profiles/traffic.json), else None; plus the capture's
    fp64-pipe / issue-active / DRAM percentages of that kernel."""
    try:
        with open(TRAFFIC_FILE) as f:
            t = json.load(f)
        e = t[workload][kernel]
        if e.get("csrc_sha") != csrc_sha():
            return None, f"capture {e.get('csrc_sha')} is for other sources", {}
        extra = {k: e[k] for k in ("fp64_pipe_pct", "issue_active_pct", "dram_pct_of_peak") if k in e}
        return float(e["bytes"]), e.get("source", "profiles/traffic.json"), extra
    except Exception as exc:  # noqa: BLE001
        return None, f"no capture ({type(exc).__name__})", {}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--mode", choices=["fast", "parity"], default="fast")
    ap.add_argument("--no-gn", action="store_true", help="skip the full GN registration timings")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-fast32", action="store_true", help="skip the optional fp32 mode lines")
    ap.add_argument("--slabs", action="store_true", help="run the z-slab path even at N=1 (checks that code path)")
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


def fp64_peak():
    """Measured DFMA throughput of this GPU model (scripts/probe/fp64_peak.cu, profiles/), for the
    fp64 ridge the kernels' fp64-pipe percentages refer to."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_fp64_peak.json")) as f:
            return float(json.load(f)["dfma_tflops"])
    except Exception:  # noqa: BLE001
        return None


def measured_hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"




def make_inputs_gpu(P, torch, wl: str):
    """The workload on the GPU: the reference's phantom and sinusoid warp re-implemented as
    device generators (bitwise equal to synthetic.cpp, tests/test_capi_host.py)."""
    m, h = WORKLOADS[wl]["m"], WORKLOADS[wl]["h"]
    img = P.make_image_grid(m, h)
    dg = P.deformation_grid_for(img, RATIO)
    R = P.make_phantom(img, device=True)
    R.mul_(1000.0)
    T = P.warp_sinusoid(R, img, 3.0, 42)
    gen = torch.Generator(device="cuda").manual_seed(8)
    nd = 3 * dg.count()
    xid = torch.from_numpy(dg.point_coords()).cuda()
    y = xid + (torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 0.6 - 0.3)
    p = torch.rand(nd, generator=gen, device="cuda", dtype=torch.float64) * 2.0 - 1.0
    del xid
    return img, dg, R, T, y, p


def cpu_reference_sample(wl: str, steps: int, threads: int, warmup: int = 1):
    """The reference CPU implementation (oracle/_ref = the unmodified reference library, else
    the C port) on a bounded sample of the workload: the same spacing, ratio and inputs
    generated by the reference's own synthetic.cpp, on a z sub-slab (C4: 512x512x24). Only
    the checker library is loaded — never libmfreg_cuda.so. Returns per-voxel timings."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("ref") else "port"
    o = Oracle("ref" if kind == "reference" else "port")
    o.set_threads(threads)
    m, h = WORKLOADS[wl]["sample_m"], WORKLOADS[wl]["h"]
    R = o.make_phantom(m, h) * 1000.0
    T = o.warp_sinusoid(R, m, h, 3.0, 42)
    my, _ = o.deformation_grid_for(m, h, RATIO)
    obj = o.objective(R, T, m, h, my, 10.0, 10.0, 1.0)
    rng = np.random.default_rng(8)
    y = obj.identity() + rng.uniform(-0.3, 0.3, obj.dof)
    p = rng.uniform(-1.0, 1.0, obj.dof)
    for _ in range(max(1, warmup)):  # untimed warm-up steps
        obj.eval(y)
        obj.gn_hessian_vec(p)
    te, th, tv = [], [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        obj.eval(y)
        t1 = time.perf_counter()
        obj.gn_hessian_vec(p)
        t2 = time.perf_counter()
        obj.eval(y, want_grad=False)
        t3 = time.perf_counter()
        te.append(t1 - t0)
        th.append(t2 - t1)
        tv.append(t3 - t2)
    n = int(np.prod(m))
    step = statistics.median(a + b for a, b in zip(te, th))
    return {"kind": kind, "cores": threads if kind == "reference" else 1, "n": n, "m": list(m),
            "value": 2.0 * n / step / 1e9, "s_per_step": step,
            "s_per_vox_eval": statistics.median(te) / n, "s_per_vox_hv": statistics.median(th) / n,
            "s_per_vox_value": statistics.median(tv) / n,
            "sample": f"{steps} steps of eval(y,grad)+gn_hessian_vec(p) on a {m[0]}x{m[1]}x{m[2]} z sub-slab "
                      f"(h={h[0]}, inputs from the reference's synthetic.cpp), median; Gvoxel/s per voxel "
                      f"is size-independent (the reference kernels are linear in the voxel count)"}


def measured_registration_64(P, threads: int):
    """A full registration timed on both sides (no extrapolation): the 64^3 phantom pair (h = 1,
    phantom x1000, sinusoid amp 3 seed 42, the reference's own generators), 3-level Gauss-Newton
    with the reference's defaults (multilevel.cpp:117-145) - the unmodified reference library
    (oracle/_ref) on the host's threads against this library in fast and parity mode on the GPU,
    with the parity field compared bitwise to the reference's."""
    import torch
    from oracle.oracle import Oracle, available
    if not available("ref"):
        return None
    o = Oracle("ref")
    o.set_threads(threads)
    m, h = (64, 64, 64), (1.0, 1.0, 1.0)
    R = o.make_phantom(m, h) * 1000.0
    T = o.warp_sinusoid(R, m, h, 3.0, 42)
    t0 = time.perf_counter()
    y_ref, _, tr, _ = o.register_multilevel(R, T, m, h, levels=3, method="gn")
    t_ref = time.perf_counter() - t0
    img = P.make_image_grid(m, h)
    out = {"workload": "64^3 h=1 phantom pair, 3-level GN, reference defaults", "reference_cpu_s": t_ref,
           "cores": threads, "reference_outer_iters": [len(t) for t in tr],
           "reference_cg_iters": int(sum(r[1] for t in tr for r in t))}
    for name, md in (("fast", P.Mode.FAST), ("parity", P.Mode.PARITY)):
        cfg = P.MultilevelConfig(levels=3, method=P.Method.GAUSS_NEWTON, mode=md)
        walls = []
        for _ in range(2 if name == "fast" else 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            y, _, lv = P.register_multilevel(R, T, img, cfg)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        y = np.asarray(y)
        out[f"ours_{name}_s"] = min(walls)
        if name == "parity":
            out["parity_y_bitwise_equal"] = bool(np.array_equal(y.view(np.uint64), y_ref.view(np.uint64)))
        else:
            d = np.abs(y - y_ref).reshape(3, -1) / np.array(h)[:, None]
            out["fast_vs_reference_max_voxel"] = float(d.max())
    out["speedup_fast"] = t_ref / out["ours_fast_s"]
    return out


def cpu_gn_model(cpu: dict, levels_gpu, img_counts):
    """CPU reference wall time of the same multilevel GN run, extrapolated from the measured
    per-voxel costs: per level, (outer iterations) gradient evals + (CG iterations) GN Hv +
    (line-search trials) value-only evals, with the iteration counts of the GPU run."""
    t = 0.0
    for (trace, _), n in zip(levels_gpu, img_counts):
        outer = len(trace)
        cg = sum(r.cg_iters for r in trace)
        t += n * (outer * cpu["s_per_vox_eval"] + cg * cpu["s_per_vox_hv"] + 2 * outer * cpu["s_per_vox_value"])
    return t


def bench_config(wl: dict, mode: str, world: int, slabs: bool) -> dict:
    """The workload description both arms print (the reference arm runs it on a bounded sample,
    described in its cpu_baseline); nodal points as deformation_grid_for (multilevel.cpp:39-49)."""
    nodal = [max(2, (m + RATIO - 1) // RATIO + 1) for m in wl["m"]]
    par = f"z slabs x{world} (C++ SlabProblem; NCCL plane exchanges)" if (world > 1 or slabs) else "single GPU"
    return {"workload": wl["name"], "image": list(wl["m"]), "spacing": list(wl["h"]), "nodal": nodal, "mode": mode,
            "l2": "inputs larger than L2 (per-step state > 20 GB at C4) and L2 flushed between steps (256 MB write)",
            "parallelism": par}


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path on the host cores, on a
    bounded sample of the same workload (rank 0 only). Loads oracle/_ref only."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # the driver's K and W (one step ~0.5 s on the sub-slab), capped so that a large K still
    # finishes within a few minutes
    steps, warmup = max(1, min(args.steps, 100)), max(1, min(args.warmup, 10))
    cpu = cpu_reference_sample(args.workload, steps, threads, warmup)
    wl = WORKLOADS[args.workload]
    line = {"metric": METRIC, "value": cpu["value"], "unit": "Gvoxel/s", "n_gpus": world, "steps": steps,
            "warmup": warmup, "ms_per_step": cpu["s_per_step"] * 1e3, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": bench_config(wl, args.mode, world, args.slabs),
            "impl": "reference",
            "cpu_baseline": {"value": cpu["value"], "unit": "Gvoxel/s", "cores": cpu["cores"], "kind": cpu["kind"],
                             "sample": cpu["sample"]},
            "e2e": {"value": cpu["value"], "unit": "Gvoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def time_steps(obj, y, grad, p, q, steps, flush, torch):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        flush.zero_()
        a, b, c = ev[k]
        a.record()
        obj.eval(y, grad)
        b.record()
        obj.gn_hessian_vec(p, q)
        c.record()
    torch.cuda.synchronize()
    return [e[0].elapsed_time(e[1]) for e in ev], [e[1].elapsed_time(e[2]) for e in ev]


def run_ours(args, rank, world, local):
    import torch
    import paper_1804_10541_b200 as P
    torch.cuda.set_device(local)
    mode = P.Mode.FAST if args.mode == "fast" else P.Mode.PARITY
    wl = WORKLOADS[args.workload]
    img, dg, R, T, y, p = make_inputs_gpu(P, torch, args.workload)
    n = img.count()
    nd = 3 * dg.count()
    obj = P.Objective(R, T, img, dg, P.NgfParams(10.0, 10.0), 1.0, mode)
    grad = torch.empty_like(y)
    q = torch.empty_like(y)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")  # > 126 MB L2

    for _ in range(args.warmup):
        obj.eval(y, grad)
        obj.gn_hessian_vec(p, q)
    torch.cuda.synchronize()
    l0 = P.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    with Clocks(local) as ck:
        t_eval, t_hv = time_steps(obj, y, grad, p, q, args.steps, flush, torch)
    barrier(world)
    launches = P.launch_count() - l0
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
    k_e2e = max(3, args.steps // 2)
    t0 = time.perf_counter()
    for _ in range(k_e2e):
        obj.eval(yh, gh)
        obj.gn_hessian_vec(ph, qh)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / k_e2e, world)
    e2e = {"value": 2.0 * n * world / e2e_s / 1e9, "unit": "Gvoxel/s", "h2d_bytes_per_step": 2 * nd * 8,
           "d2h_bytes_per_step": 2 * nd * 8 + 16, "ms_per_step": e2e_s * 1e3,
           "path": "Objective.eval / gn_hessian_vec with pinned numpy buffers through the C ABI"}

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
        kern = {}
        for k, v in k_ms.items():
            tr, src, extra = traffic_for(args.workload, k)
            kern[k] = {"ms": v, "achieved_gbs": b_alg[k] * n / (v * 1e-3) / 1e9, "algorithmic_bytes_per_voxel": b_alg[k],
                       "frac": b_alg[k] * n / (v * 1e-3) / 1e9 / peak, "traffic": tr, "traffic_source": src,
                       "share_of_step": v / ms_step, **{f"ncu_{x}": y for x, y in extra.items()}}
        dom = max(k_ms, key=k_ms.get)
        names = {"hv_pass": "k_hv2 (GN Hv image pass: P p, dr, dr^T, dT, P^T partials)",
                 "eval_pass": "k_ev2 (NGF eval pass: rho-hat, r, D partials, gradient dr^T r, P^T partials)",
                 "warp": "k_warp_z (P y, trilinear T, dT/dP; z-marching)"}
        roofline = {"bound": "hbm", "achieved": kern[dom]["achieved_gbs"], "peak": peak, "unit": "GB/s",
                    "frac": kern[dom]["frac"], "traffic": kern[dom]["traffic"],
                    "traffic_unit": "bytes/launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
                    "traffic_source": kern[dom]["traffic_source"],
                    "algorithmic_bytes_per_launch": b_alg[dom] * n, "kernel": names[dom],
                    "algorithmic_bytes_per_voxel": b_alg[dom], "units_per_launch": n, "peak_source": peak_kind,
                    "kernels": kern,
                    "fp64_peak_tflops": fp64_peak(),
                    "operators": {"gn_hessian_vec": {"ms": ms_hv, "frac": B_CANON_HV * n / (ms_hv * 1e-3) / 1e9 / peak},
                                  "eval_grad": {"ms": ms_eval, "frac": B_CANON_GRAD * n / (ms_eval * 1e-3) / 1e9 / peak}}}

    # the optional fp32 mode (FAST32) on the same workload: operator rate and Hv kernel time
    fast32 = None
    if mode == P.Mode.FAST and world == 1 and not args.no_fast32 and not wl.get("derivative_only"):
        o32 = P.Objective(R, T, img, dg, P.NgfParams(10.0, 10.0), 1.0, P.Mode.FAST32)
        for _ in range(3):
            o32.eval(y, grad)
            o32.gn_hessian_vec(p, q)
        torch.cuda.synchronize()
        te32, th32 = time_steps(o32, y, grad, p, q, args.steps, flush, torch)
        ms32 = statistics.mean(te32) + statistics.mean(th32)
        reps = max(5, args.steps)
        k32 = {"hv_pass": o32.profile_kernel(0, p, reps), "eval_pass": o32.profile_kernel(1, p, reps),
               "warp": o32.profile_kernel(2, y, reps)}
        fast32 = {"value": 2.0 * n / (ms32 * 1e-3) / 1e9, "unit": "Gvoxel/s", "ms_per_step": ms32,
                  "kernels_ms": k32, "tolerance": "max-rel 1e-4 vs reference (tests/test_gpu_fast32.py)",
                  "algorithmic_bytes_per_voxel_hv": 20.0,
                  "hv_frac": 20.0 * n / (k32["hv_pass"] * 1e-3) / 1e9 / peak}
        del o32
    del obj
    torch.cuda.synchronize()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        cpu = cpu_reference_sample(args.workload, 3, threads)

    # the metric's second half: the full 3-level GN registration of this pair on this GPU,
    # wall clock from the host (cold = first registration in the process, then warm); the
    # same run in FAST32; the CPU reference's wall time for the same iteration counts,
    # extrapolated from its measured per-voxel costs
    gn = None
    if not args.no_gn and world == 1 and mode == P.Mode.FAST and not wl.get("derivative_only"):
        gn = {"workload": f"{wl['m'][0]}x{wl['m'][1]}x{wl['m'][2]} h={wl['h'][0]}, {LEVELS} levels, ratio {RATIO}",
              "method": "gauss-newton"}
        sizes, mm = [], list(wl["m"])
        for _ in range(LEVELS):
            sizes.append(int(np.prod(mm)))
            mm = [(v + 1) // 2 for v in mm]
        sizes = sizes[::-1]  # coarsest first, as the level traces
        ckg = Clocks(local).__enter__()
        for name, md in (("fast", P.Mode.FAST), ("fast32", P.Mode.FAST32)):
            if name == "fast32" and args.no_fast32:
                continue
            cfg = P.MultilevelConfig(levels=LEVELS, deform_ratio=RATIO, method=P.Method.GAUSS_NEWTON, mode=md)
            walls = []
            for _ in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _, _, lv = P.register_multilevel(R, T, img, cfg)
                torch.cuda.synchronize()
                walls.append(time.perf_counter() - t0)
            gn[name] = {"wall_s": walls[0], "wall_s_warm": walls[1], "outer_iters": [len(t) for t, _ in lv],
                        "cg_iters": int(sum(r.cg_iters for t, _ in lv for r in t)),
                        "final_J": lv[-1][0][-1].j if lv[-1][0] else None}
            if name == "fast" and cpu is not None:
                gn["reference_cpu_wall_s_extrapolated"] = cpu_gn_model(cpu, lv, sizes)
                gn["reference_cpu_model"] = ("per level: outer x eval(grad) + CG x gn_hessian_vec + 2 x outer value-only "
                                             "evals, iteration counts of this run, per-voxel costs of cpu_baseline "
                                             f"({cpu['cores']} threads)")
        ckg.__exit__(None, None, None)
        gn["clocks"] = ckg.summary()
        if rank == 0 and not args.no_cpu:
            gn["measured_registration_64"] = measured_registration_64(P, os.cpu_count() or 1)

    if rank == 0:
        cpu_line = None
        if cpu is not None:
            cpu_line = {"value": cpu["value"], "unit": "Gvoxel/s", "cores": cpu["cores"], "kind": cpu["kind"],
                        "sample": cpu["sample"]}
        line = {"metric": METRIC, "value": value, "unit": "Gvoxel/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": DATA,
                "config": bench_config(wl, args.mode, world, args.slabs),
                "ms_grad_eval": ms_eval, "ms_gn_hv": ms_hv,
                "gvox_s_grad_eval": n / (ms_eval * 1e-3) / 1e9, "gvox_s_gn_hv": n / (ms_hv * 1e-3) / 1e9,
                "roofline": roofline, "cpu_baseline": cpu_line, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "gn_registration": gn, "fast32": fast32}
        print(json.dumps(line), flush=True)


def run_slabs(args, rank, world, local):
    """N > 1: strong scaling of the same workload over z slabs in the library (csrc/slab.cu,
    DESIGN.md §8): rank r evaluates its slab of the global volume; every step performs the
    real NCCL plane exchanges, shared-plane sums and rank-ordered scalar all-gathers inside the
    C++ SlabProblem. The sharded multilevel GN registration is timed under gn_registration."""
    import torch
    import paper_1804_10541_b200 as P
    from paper_1804_10541_b200 import slab as S
    torch.cuda.set_device(local)
    md = P.PARITY if args.mode == "parity" else P.FAST  # parity: bitwise the one-GPU parity objective
    wl = WORKLOADS[args.workload]
    img, dg, R, T, y, p = make_inputs_gpu(P, torch, args.workload)
    nd = 3 * dg.count()
    comm = S.NativeComm.nccl()
    sl = S.NativeSlab(comm, R, T, img, dg, P.NgfParams(10.0, 10.0), 1.0, md)
    s = sl.info
    n_loc = (s.zhi - s.zlo) * wl["m"][0] * wl["m"][1]
    n_glob = img.count()
    grad = torch.zeros_like(y)
    q = torch.zeros_like(y)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    class _Step:  # time_steps() drives eval / gn_hessian_vec
        def eval(self, yy, gg):
            return sl.eval(yy, gg)

        def gn_hessian_vec(self, pp, qq):
            return sl.gn_hessian_vec(pp, qq)

    for _ in range(args.warmup):
        sl.eval(y, grad)
        sl.gn_hessian_vec(p, q)
    torch.cuda.synchronize()
    l0 = P.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    with Clocks(local) as ck:
        t_eval, t_hv = time_steps(_Step(), y, grad, p, q, args.steps, flush, torch)
    barrier(world)
    launches = P.launch_count() - l0
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
        sl.eval(yd, grad)
        sl.gn_hessian_vec(pd, q)
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
           "d2h_bytes_per_step": 2 * nd * 8 * world, "ms_per_step": e2e_s * 1e3,
           "path": "NativeSlab eval / gn_hessian_vec (C ABI mfreg_cu_slab_*) with pinned host copies"}
    peak, peak_kind = measured_hbm_peak()
    achieved = B_CANON_HV * n_loc / (ms_hv * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None, "kernel": "gn_hessian_vec per rank (slab incl. NCCL halo exchange)",
                "algorithmic_bytes_per_voxel": B_CANON_HV, "units_per_launch": n_loc, "peak_source": peak_kind}
    gn = None
    if not args.no_gn and not wl.get("derivative_only"):
        cfg = P.MultilevelConfig(levels=LEVELS, deform_ratio=RATIO, method=P.Method.GAUSS_NEWTON, mode=md)
        walls = []
        for _ in range(2):  # cold, then warm
            barrier(world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, _, lv = S.register_multilevel_native(comm, R, T, img, cfg)
            torch.cuda.synchronize()
            walls.append(max_over_ranks(time.perf_counter() - t0, world))
        gn = {"workload": f"{wl['m'][0]}x{wl['m'][1]}x{wl['m'][2]} h={wl['h'][0]}, {LEVELS} levels, ratio {RATIO}",
              "method": "gauss-newton", "fast": {"wall_s": walls[0], "wall_s_warm": walls[1],
                                                 "outer_iters": [len(t) for t, _ in lv],
                                                 "cg_iters": int(sum(r.cg_iters for t, _ in lv for r in t)),
                                                 "final_J": lv[-1][0][-1].j if lv[-1][0] else None},
              "parallelism": f"z slabs x{world} (C++ SlabProblem, NCCL)"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "Gvoxel/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": DATA,
                "config": bench_config(wl, args.mode, world, True),
                "ms_grad_eval": ms_eval, "ms_gn_hv": ms_hv, "roofline": roofline, "cpu_baseline": None,
                "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "gn_registration": gn}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_init(args.gpus)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    elif world > 1 or args.slabs:
        run_slabs(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
