"""TEST INFRASTRUCTURE ONLY — generates tests/golden/*.npz from the UNMODIFIED
reference library (oracle/_ref/libmfreg_ref.so, built from /root/reference by
oracle/Makefile). Run in the build container (the reference tree is not on the
GPU box); the fixtures are committed.

    python oracle/gen_golden.py

Cases mirror the reference's own test builders: random smoothed volumes with
y = identity + U(-0.4, 0.4) (tests/test_ngf.cpp:31-56, tests/acceptance.cpp:65-89),
anisotropic/tie-heavy phantom cases, degenerate axes (m = 1, 2),
and short solver / multilevel trajectories.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle, OptConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def nodal_coords(my, hy):
    ax = [np.arange(my[a]) * hy[a] for a in range(3)]
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return np.concatenate([x.ravel(), y.ravel(), z.ravel()])


def operator_case(o: Oracle, name, m, h, my, tau, rho, alpha, kind, seed, jitter):
    m, h, my = tuple(m), tuple(h), tuple(my)
    if kind == "random":
        ref = o.make_random_volume(m, h, seed, 1)
        tpl = o.make_random_volume(m, h, seed + 1, 1)
    else:
        ref = o.make_phantom(m, h) * 1000.0
        tpl = o.warp_sinusoid(ref, m, h, 3.0, 42)
    hy = o.make_deform_grid(m, h, my)
    rng = np.random.default_rng(seed + 2)
    y = nodal_coords(my, hy) + (rng.uniform(-jitter, jitter, 3 * int(np.prod(my))) if jitter else 0.0)
    n = int(np.prod(m))
    p_img = rng.uniform(-1.0, 1.0, 3 * n)
    w_img = rng.uniform(-1.0, 1.0, 3 * n)
    p_nod = rng.uniform(-1.0, 1.0, 3 * int(np.prod(my)))
    yhat = o.transfer_apply(my, hy, m, h, y)
    ptw = o.transfer_apply_transpose(my, hy, m, h, w_img)
    base, rem = o.transfer_plan(my, hy, m, h)
    ngf = o.ngf(ref, m, h, tau, rho)
    ngf.populate(tpl, yhat)
    ws = ngf.workspace()
    rho_hat = np.concatenate([[ngf.rho(i, k) for i in range(n)] for k in range(7)])
    D = ngf.value()
    g_img = ngf.gradient()
    hv_img = ngf.hessian_vec(p_img)
    obj = o.objective(ref, tpl, m, h, my, tau, rho, alpha)
    J, Dd, S, grad = obj.eval(y)
    Jv, Dv, Sv, _ = obj.eval(y, want_grad=False)
    gn = obj.gn_hessian_vec(p_nod)
    seed_hv = obj.seed_hessian_vec(p_nod, 1e-3)
    u = y - obj.identity()
    curv_val = o.curvature_value(u, my, hy)
    curv_grad = o.curvature_gradient(u, my, hy)
    lap = o.laplacian_apply(u[: int(np.prod(my))], my, hy)
    cg_x, cg_it, cg_rr, cg_bd = obj.cg_solve(-grad, 50, 1e-2)
    d = dict(m=np.array(m), h=np.array(h), my=np.array(my), hy=hy, tau=tau, rho=rho, alpha=alpha, ref=ref, tpl=tpl,
             y=y, p_img=p_img, w_img=w_img, p_nod=p_nod, yhat=yhat, ptw=ptw, plan_base=base, plan_rem=rem,
             values=ws["values"], partials=ws["partials"], residual=ws["residual"], inv1=ws["inv1"], inv2=ws["inv2"],
             tpl_grads=ws["tpl_grads"], ref_grads=ws["ref_grads"], rho_hat=rho_hat, D=D, g_img=g_img, hv_img=hv_img,
             J=J, Dobj=Dd, S=S, grad=grad, Jv=Jv, gn_hv=gn, seed_hv=seed_hv, u=u, curv_val=curv_val,
             curv_grad=curv_grad, lap=lap, cg_x=cg_x, cg_iters=cg_it, cg_relres=cg_rr)
    np.savez_compressed(os.path.join(OUT, f"op_{name}.npz"), **d)
    print(f"op_{name}: n={n} D={D:.6g} J={J:.6g} cg={cg_it}")


def solver_case(o: Oracle, name, m, h, my, tau, rho, alpha, method, max_iters):
    m, h, my = tuple(m), tuple(h), tuple(my)
    ref = o.make_phantom(m, h) * 1000.0
    tpl = o.warp_sinusoid(ref, m, h, 3.0, 42)
    obj = o.objective(ref, tpl, m, h, my, tau, rho, alpha)
    cfg = OptConfig.defaults(max_iters=max_iters)
    y, trace, lsf = obj.minimize(obj.identity(), method, cfg)
    np.savez_compressed(os.path.join(OUT, f"solve_{name}.npz"), m=np.array(m), h=np.array(h), my=np.array(my),
                        tau=tau, rho=rho, alpha=alpha, method=method, max_iters=max_iters, ref=ref, tpl=tpl, y=y,
                        trace=np.array(trace, dtype=np.float64), lsf=lsf)
    print(f"solve_{name}: {method} iters={len(trace)} lsf={lsf} J={trace[-1][2]:.6g}")


def config_case(o: Oracle, name, m, h, ratio, method, max_iters):
    """BASELINE configs[0] (C1: 256x256 single-level GN) and its quasi-2D variant C1'
    (SURVEY §8(d)). The test regenerates the inputs with the reference library (oracle
    fixture), so only their hashes are stored next to the trace and the final y."""
    import hashlib
    m, h = tuple(m), tuple(h)
    ref = o.make_phantom(m, h) * 1000.0
    tpl = o.warp_sinusoid(ref, m, h, 3.0, 42)
    my, _ = o.deformation_grid_for(m, h, ratio)
    obj = o.objective(ref, tpl, m, h, my, 10.0, 10.0, 1.0)
    cfg = OptConfig.defaults(max_iters=max_iters)
    y, trace, lsf = obj.minimize(obj.identity(), method, cfg)
    np.savez_compressed(os.path.join(OUT, f"cfg_{name}.npz"), m=np.array(m), h=np.array(h), my=np.array(my),
                        ratio=ratio, method=method, max_iters=max_iters, y=y, trace=np.array(trace, dtype=np.float64),
                        lsf=lsf, ref_sha=hashlib.sha256(ref.tobytes()).hexdigest(),
                        tpl_sha=hashlib.sha256(tpl.tobytes()).hexdigest())
    print(f"cfg_{name}: {method} iters={len(trace)} lsf={lsf} J={trace[-1][2] if trace else None}")


def sinusoid_displacement(terms, extent, pts):
    """synthetic.cpp:91-107 SinusoidWarp::displacement at (N, 3) points (numpy restatement)."""
    amp, freq, phase = terms
    x = pts / np.asarray(extent)[None, :]
    u = np.zeros_like(pts)
    for t in range(amp.shape[0]):
        w = np.ones(len(pts))
        for a in range(3):
            w = w * np.sin(np.pi * freq[t][a] * x[:, a] + phase[t][a] * x[:, a] * (1.0 - x[:, a]))
        for d in range(3):
            u[:, d] += amp[t][d] * w
    return u


def c3_landmarks(o: Oracle, m, h, count=300, seed=3):
    """300 seeded landmark voxels; moving = phi^-1(fixed) by the fixed-point inversion of
    tests/acceptance.cpp:476-487 (40 iterations of q = p - u(q))."""
    extent = [m[a] * h[a] for a in range(3)]
    terms = o.sinusoid_terms(extent, 3.0, 42)
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, m, (count, 3))
    fixed = (idx + 0.5) * np.asarray(h)
    q = fixed.copy()
    for _ in range(40):
        q = fixed - sinusoid_displacement(terms, extent, q)
    return fixed, q


def c3_case(o: Oracle):
    """BASELINE configs[2] (C3): DIR-Lab-shaped 256x256x100, h = (0.97, 0.97, 2.5), 4-level
    L-BFGS, landmark-style check: trace, y hash and the landmark errors
    (io::landmark_error before / after) of the unmodified reference."""
    import hashlib
    m, h = (256, 256, 100), (0.97, 0.97, 2.5)
    ref = o.make_phantom(m, h) * 1000.0
    tpl = o.warp_sinusoid(ref, m, h, 3.0, 42)
    y, my, traces, lsf = o.register_multilevel(ref, tpl, m, h, levels=4, method="lbfgs")
    hy = o.make_deform_grid(m, h, my)
    fixed, moving = c3_landmarks(o, m, h)
    before = o.io_landmark_error(fixed, moving, nodal_coords(my, hy), my, hy)
    after = o.io_landmark_error(fixed, moving, y, my, hy)
    flat = np.array([r for t in traces for r in t], dtype=np.float64)
    np.savez_compressed(os.path.join(OUT, "c3_lbfgs.npz"), m=np.array(m), h=np.array(h), my=np.array(my), levels=4,
                        trace=flat, level_iters=np.array([len(t) for t in traces]), lsf=np.array(lsf),
                        y_sha=hashlib.sha256(y.tobytes()).hexdigest(), ref_sha=hashlib.sha256(ref.tobytes()).hexdigest(),
                        tpl_sha=hashlib.sha256(tpl.tobytes()).hexdigest(), lm_before=np.array(before[:2]),
                        lm_after=np.array(after[:2]), fixed=fixed, moving=moving)
    print(f"c3_lbfgs: iters={[len(t) for t in traces]} landmark error {before[0]:.4f} -> {after[0]:.4f}")


def c2_case(o: Oracle):
    """BASELINE configs[1] (C2): 128^3 phantom pair, 3-level Gauss-Newton with the reference's
    default OptimizerConfig (multilevel.cpp:117-145): per-level traces, final y (about 9 min
    on 8 threads in the build container)."""
    import hashlib
    m, h = (128, 128, 128), (1.0, 1.0, 1.0)
    ref = o.make_phantom(m, h) * 1000.0
    tpl = o.warp_sinusoid(ref, m, h, 3.0, 42)
    y, my, traces, lsf = o.register_multilevel(ref, tpl, m, h, levels=3, method="gn")
    flat = np.array([r for t in traces for r in t], dtype=np.float64)
    np.savez_compressed(os.path.join(OUT, "c2_gn.npz"), m=np.array(m), h=np.array(h), my=np.array(my), levels=3,
                        trace=flat, level_iters=np.array([len(t) for t in traces]), lsf=np.array(lsf), y=y,
                        ref_sha=hashlib.sha256(ref.tobytes()).hexdigest(),
                        tpl_sha=hashlib.sha256(tpl.tobytes()).hexdigest())
    print(f"c2_gn: iters={[len(t) for t in traces]} cg={int(flat[:, 1].sum())} J={flat[-1, 2]:.6f}")


def multilevel_case(o: Oracle, name, m, h, levels, method, max_iters):
    m, h = tuple(m), tuple(h)
    ref = o.make_phantom(m, h) * 1000.0
    tpl = o.warp_sinusoid(ref, m, h, 3.0, 42)
    cfg = OptConfig.defaults(max_iters=max_iters)
    y, my, traces, lsf = o.register_multilevel(ref, tpl, m, h, levels=levels, method=method, cfg=cfg)
    flat = np.array([r for t in traces for r in t], dtype=np.float64)
    np.savez_compressed(os.path.join(OUT, f"ml_{name}.npz"), m=np.array(m), h=np.array(h), levels=levels,
                        method=method, max_iters=max_iters, ref=ref, tpl=tpl, y=y, my=np.array(my), trace=flat,
                        level_iters=np.array([len(t) for t in traces]), lsf=np.array(lsf))
    print(f"ml_{name}: {method} levels={levels} iters={[len(t) for t in traces]}")


def main():
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1 and sys.argv[1] == "c2":  # only the C2 registration
        o = Oracle("ref")
        o.set_threads(os.cpu_count() or 1)
        c2_case(o)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "configs":  # only the config cases
        o = Oracle("ref")
        o.set_threads(os.cpu_count() or 1)
        config_case(o, "c1", (256, 256, 1), (1.0, 1.0, 1.0), 4, "gn", 20)
        config_case(o, "c1p", (256, 256, 8), (1.0, 1.0, 1.0), 4, "gn", 3)
        c3_case(o)
        c2_case(o)
        return
    o = Oracle("ref")
    o.set_threads(1)
    operator_case(o, "rand_aniso", (7, 6, 5), (1.0, 1.3, 0.8), (4, 4, 3), 1.0, 1.0, 1.0, "random", 11, 0.4)
    operator_case(o, "rand_cube", (8, 8, 8), (1.0, 1.0, 1.0), (5, 5, 5), 10.0, 10.0, 0.5, "random", 2000, 0.4)
    operator_case(o, "phantom_ties", (12, 10, 9), (0.97, 0.97, 2.5), (4, 4, 4), 10.0, 10.0, 1.0, "phantom", 5, 0.0)
    operator_case(o, "phantom_h07", (14, 11, 10), (0.7, 0.7, 0.7), (5, 4, 4), 10.0, 10.0, 1.0, "phantom", 6, 0.3)
    operator_case(o, "slab_z1", (9, 7, 1), (1.0, 1.0, 1.0), (4, 3, 2), 1.0, 1.0, 1.0, "random", 21, 0.4)
    operator_case(o, "thin_x1", (1, 6, 7), (1.0, 1.0, 1.0), (2, 3, 4), 1.0, 1.0, 1.0, "random", 31, 0.3)
    operator_case(o, "thin_x2y2", (2, 2, 9), (1.0, 0.5, 1.0), (2, 2, 4), 1.0, 1.0, 1.0, "random", 41, 0.3)
    operator_case(o, "thin_x3", (3, 5, 4), (1.0, 1.0, 1.0), (3, 3, 3), 1.0, 1.0, 1.0, "random", 51, 0.3)
    solver_case(o, "gn", (10, 9, 8), (1.0, 1.0, 1.0), (4, 4, 3), 10.0, 10.0, 1.0, "gn", 6)
    solver_case(o, "lbfgs", (10, 9, 8), (1.0, 1.0, 1.0), (4, 4, 3), 10.0, 10.0, 1.0, "lbfgs", 8)
    multilevel_case(o, "gn2", (16, 14, 12), (1.0, 1.0, 1.0), 2, "gn", 4)
    multilevel_case(o, "lbfgs2", (18, 16, 14), (0.97, 0.97, 2.5), 2, "lbfgs", 6)
    o.set_threads(os.cpu_count() or 1)  # the reference's results are thread-count invariant
    config_case(o, "c1", (256, 256, 1), (1.0, 1.0, 1.0), 4, "gn", 20)
    config_case(o, "c1p", (256, 256, 8), (1.0, 1.0, 1.0), 4, "gn", 3)
    c3_case(o)


if __name__ == "__main__":
    main()
