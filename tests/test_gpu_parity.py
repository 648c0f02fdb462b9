"""GPU parity: the CUDA path (through the C ABI) against the reference.

* `parity` mode must be BITWISE identical to the reference library on every
  golden fixture (operators, solver trajectories, multilevel) and on fresh
  inputs checked against the CPU oracle at run time;
* `fast` mode (tree reductions, factored GN Hv) must agree to max-rel <= 1e-9
  (north_star tolerance for fp64), metric of tests/acceptance.cpp:40-50.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import bits_equal, golden_files, load, max_rel, tup

pytestmark = pytest.mark.gpu
FAST_TOL = 1e-9


@pytest.fixture(scope="module")
def P():
    import paper_1804_10541_b200 as P
    return P


def _grids(P, g):
    img = P.make_image_grid(tup(g["m"]), tup(g["h"], float))
    dg = P.make_deform_grid(img, tup(g["my"]))
    return img, dg


@pytest.mark.parametrize("path", golden_files("op"), ids=lambda p: p.split("/")[-1])
def test_operators_bitwise_parity(P, path):
    g = load(path)
    img, dg = _grids(P, g)
    assert bits_equal(dg.h, g["hy"])
    assert bits_equal(P.transfer_apply(dg, img, g["y"]), g["yhat"])
    assert bits_equal(P.transfer_apply_transpose(dg, img, g["w_img"]), g["ptw"])
    vals, parts = P.sample_deformed(g["tpl"], img, g["yhat"])
    assert bits_equal(vals, g["values"]) and bits_equal(parts, g["partials"])
    params = P.NgfParams(float(g["tau"]), float(g["rho"]))
    ngf = P.NgfContext(g["ref"], img, params, P.Mode.PARITY)
    ngf.populate(g["tpl"], g["yhat"])
    ws = ngf.workspace()
    for k in ("values", "partials", "residual", "inv1", "inv2", "rho_hat"):
        assert bits_equal(ws[k], g[k]), k
    assert bits_equal(ngf.value(), g["D"])
    assert bits_equal(ngf.gradient(), g["g_img"])
    assert bits_equal(ngf.hessian_vec(g["p_img"]), g["hv_img"])
    obj = P.Objective(g["ref"], g["tpl"], img, dg, params, float(g["alpha"]), P.Mode.PARITY)
    grad = np.empty(obj.dof())
    J = obj.eval(g["y"], grad)
    assert bits_equal([J, obj.last_distance(), obj.last_regularizer()], [g["J"], g["Dobj"], g["S"]])
    assert bits_equal(grad, g["grad"])
    assert bits_equal(obj.gn_hessian_vec(g["p_nod"]), g["gn_hv"])
    assert bits_equal(obj.seed_hessian_vec(g["p_nod"], 1e-3), g["seed_hv"])
    assert bits_equal(obj.eval(g["y"]), g["Jv"])  # value-only
    x, it, rr, bd = P.cg_solve(obj, -g["grad"])
    assert it == int(g["cg_iters"]) and bits_equal(x, g["cg_x"]) and bits_equal(rr, g["cg_relres"])
    ny = dg.count()
    assert bits_equal(P.curvature_value(g["u"], dg), g["curv_val"])
    assert bits_equal(P.curvature_gradient(g["u"], dg), g["curv_grad"])
    assert bits_equal(P.curvature_hessian_vec(g["u"], dg), g["curv_grad"])
    assert bits_equal(P.laplacian_apply(g["u"][:ny], dg), g["lap"])


@pytest.mark.parametrize("path", golden_files("op"), ids=lambda p: p.split("/")[-1])
def test_operators_fast_mode_tolerance(P, path):
    g = load(path)
    img, dg = _grids(P, g)
    params = P.NgfParams(float(g["tau"]), float(g["rho"]))
    ngf = P.NgfContext(g["ref"], img, params, P.Mode.FAST)
    ngf.populate(g["tpl"], g["yhat"])
    assert max_rel(ngf.value(), g["D"]) <= FAST_TOL
    assert max_rel(ngf.gradient(), g["g_img"]) <= FAST_TOL
    assert max_rel(ngf.hessian_vec(g["p_img"]), g["hv_img"]) <= FAST_TOL
    obj = P.Objective(g["ref"], g["tpl"], img, dg, params, float(g["alpha"]), P.Mode.FAST)
    grad = np.empty(obj.dof())
    J = obj.eval(g["y"], grad)
    assert max_rel(J, g["J"]) <= FAST_TOL
    assert max_rel(grad, g["grad"]) <= FAST_TOL
    assert max_rel(obj.gn_hessian_vec(g["p_nod"]), g["gn_hv"]) <= FAST_TOL
    assert max_rel(P.curvature_value(g["u"], dg, P.Mode.FAST), g["curv_val"]) <= FAST_TOL


@pytest.mark.parametrize("path", golden_files("solve"), ids=lambda p: p.split("/")[-1])
def test_solver_trajectory_bitwise(P, path):
    g = load(path)
    img, dg = _grids(P, g)
    obj = P.Objective(g["ref"], g["tpl"], img, dg, P.NgfParams(float(g["tau"]), float(g["rho"])), float(g["alpha"]),
                      P.Mode.PARITY)
    cfg = P.OptimizerConfig(max_iters=int(g["max_iters"]))
    fn = P.gauss_newton_minimize if str(g["method"]) == "gn" else P.lbfgs_minimize
    y, trace, lsf = fn(obj, obj.identity(), cfg)
    assert bits_equal(np.array([r.as_tuple() for r in trace], dtype=np.float64), g["trace"])
    assert bits_equal(y, g["y"]) and lsf == bool(g["lsf"])


@pytest.mark.parametrize("path", golden_files("ml"), ids=lambda p: p.split("/")[-1])
def test_multilevel_bitwise(P, path):
    g = load(path)
    img = P.make_image_grid(tup(g["m"]), tup(g["h"], float))
    cfg = P.MultilevelConfig(levels=int(g["levels"]),
                             method=P.Method.GAUSS_NEWTON if str(g["method"]) == "gn" else P.Method.LBFGS,
                             opt=P.OptimizerConfig(max_iters=int(g["max_iters"])), mode=P.Mode.PARITY)
    y, dg, levels = P.register_multilevel(g["ref"], g["tpl"], img, cfg)
    assert dg.m == tup(g["my"])
    flat = np.array([r.as_tuple() for tr, _ in levels for r in tr], dtype=np.float64)
    assert bits_equal(flat, g["trace"])
    assert bits_equal(y, g["y"])


# ---- fresh inputs, checked against the CPU oracle at run time ----------------------
CASES = [((40, 36, 32), (0.97, 0.97, 2.5), 4, 0.3), ((33, 29, 17), (0.7, 0.7, 0.7), 3, 0.3),
         ((48, 40, 36), (1.0, 1.0, 1.0), 4, 0.4), ((64, 48, 1), (1.0, 1.0, 1.0), 4, 0.3)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0])))
def test_objective_vs_oracle(P, oracle, case):
    m, h, ratio, jit = case
    R = oracle.make_phantom(m, h) * 1000.0
    T = oracle.warp_sinusoid(R, m, h, 3.0, 42)
    my, hy = oracle.deformation_grid_for(m, h, ratio)
    o = oracle.objective(R, T, m, h, my, 10.0, 10.0, 1.0)
    rng = np.random.default_rng(7)
    for y in (o.identity(), o.identity() + rng.uniform(-jit, jit, o.dof)):
        J, D, S, grad = o.eval(y)
        p = rng.uniform(-1, 1, o.dof)
        hv = o.gn_hessian_vec(p)
        img = P.make_image_grid(m, h)
        dg = P.deformation_grid_for(img, ratio)
        for mode in (P.Mode.PARITY, P.Mode.FAST):
            obj = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, mode)
            g = np.empty(obj.dof())
            j = obj.eval(y, g)
            q = obj.gn_hessian_vec(p)
            if mode == P.Mode.PARITY:
                assert bits_equal([j, obj.last_distance(), obj.last_regularizer()], [J, D, S])
                assert bits_equal(g, grad) and bits_equal(q, hv)
            else:
                assert max_rel(j, J) <= FAST_TOL and max_rel(g, grad) <= FAST_TOL and max_rel(q, hv) <= FAST_TOL


def test_device_pointer_path_matches_host(P):
    import torch
    m, h = (32, 28, 24), (1.0, 1.0, 1.0)
    img = P.make_image_grid(m, h)
    dg = P.deformation_grid_for(img, 4)
    R = P.make_phantom(img) * 1000.0
    T = P.warp_sinusoid(R, img, 3.0, 42)
    for mode in (P.Mode.PARITY, P.Mode.FAST):
        oh = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, mode)
        od = P.Objective(torch.from_numpy(R).cuda(), torch.from_numpy(T).cuda(), img, dg, P.NgfParams(), 1.0, mode)
        y = oh.identity() + np.random.default_rng(1).uniform(-0.3, 0.3, oh.dof())
        gh = np.empty(oh.dof())
        jh = oh.eval(y, gh)
        yd = torch.from_numpy(y).cuda()
        gd = torch.empty_like(yd)
        jd = od.eval(yd, gd)
        assert bits_equal(jh, jd) and bits_equal(gh, gd.cpu().numpy())
        p = np.random.default_rng(2).uniform(-1, 1, oh.dof())
        assert bits_equal(oh.gn_hessian_vec(p), od.gn_hessian_vec(torch.from_numpy(p).cuda()).cpu().numpy())


def test_full_size_properties(P):
    """128^3 (C2 finest): fast vs parity within tolerance, GN symmetry/PSD,
    run-to-run determinism (bitwise) for both modes."""
    import torch
    img = P.make_image_grid((128, 128, 128))
    dg = P.deformation_grid_for(img, 4)
    R = P.make_phantom(img, device=True)
    R.mul_(1000.0)
    T = P.warp_sinusoid(R, img, 3.0, 42)
    objs = {md: P.Objective(R, T, img, dg, P.NgfParams(), 1.0, md) for md in (P.Mode.PARITY, P.Mode.FAST)}
    gen = torch.Generator(device="cuda").manual_seed(0)
    y = objs[0].identity(like=R) + (torch.rand(objs[0].dof(), generator=gen, device="cuda", dtype=torch.float64) - 0.5) * 0.6
    p = torch.rand(objs[0].dof(), generator=gen, device="cuda", dtype=torch.float64) - 0.5
    q2 = torch.rand(objs[0].dof(), generator=gen, device="cuda", dtype=torch.float64) - 0.5
    res = {}
    for md, o in objs.items():
        g1, g2 = torch.empty_like(y), torch.empty_like(y)
        j1 = o.eval(y, g1)
        h1 = o.gn_hessian_vec(p).clone()
        j2 = o.eval(y, g2)
        h2 = o.gn_hessian_vec(p).clone()
        assert j1 == j2 and torch.equal(g1, g2) and torch.equal(h1, h2)  # deterministic
        hq = o.gn_hessian_vec(q2)
        a, b = float(h1 @ q2), float(p @ hq)
        assert abs(a - b) <= 1e-10 * max(1.0, abs(a))  # symmetric
        assert float(h1 @ p) >= -1e-10 * float(p @ p)  # PSD
        res[md] = (j1, g1.cpu().numpy(), h1.cpu().numpy())
    assert max_rel(res[1][0], res[0][0]) <= FAST_TOL
    assert max_rel(res[1][1], res[0][1]) <= FAST_TOL
    assert max_rel(res[1][2], res[0][2]) <= FAST_TOL


def test_invalid_arguments_raise(P):
    img = P.make_image_grid((8, 8, 8))
    dg = P.make_deform_grid(img, (3, 3, 3))
    with pytest.raises(ValueError, match="rho must be > 0"):
        P.Objective(np.zeros(512), np.zeros(512), img, dg, P.NgfParams(10.0, 0.0))
    with pytest.raises(ValueError, match="too many levels"):
        P.register_multilevel(np.zeros(512), np.zeros(512), img, P.MultilevelConfig(levels=4))
