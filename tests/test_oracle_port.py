"""CPU: pin the oracle before trusting it.

The C restatement (oracle/mfreg_oracle.c, "port") must reproduce the golden
fixtures generated from the unmodified reference library bit for bit, and —
when the reference library is compiled here (oracle/_ref) — match it bitwise on
fresh inputs. Known-answer tests restate the reference's own unit tests
(tests/test_ngf.cpp, test_transfer.cpp, test_curvature.cpp, test_optimizer.cpp).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import bits_equal, golden_files, load, max_rel, tup
from oracle.oracle import Oracle, OptConfig, available, build


@pytest.fixture(scope="module")
def port():
    if not available("port"):
        build(ref=False)
    return Oracle("port")


@pytest.fixture(scope="module")
def ref():
    if not available("ref"):
        pytest.skip("reference library not built here (needs /root/reference)")
    return Oracle("ref")


@pytest.mark.parametrize("path", golden_files("op"), ids=lambda p: p.split("/")[-1])
def test_port_operators_match_golden(port, path):
    g = load(path)
    m, h, my, hy = tup(g["m"]), tup(g["h"], float), tup(g["my"]), tup(g["hy"], float)
    tau, rho, alpha = float(g["tau"]), float(g["rho"]), float(g["alpha"])
    assert bits_equal(port.make_deform_grid(m, h, my), g["hy"])
    base, rem = port.transfer_plan(my, hy, m, h)
    assert np.array_equal(base, g["plan_base"]) and bits_equal(rem, g["plan_rem"])
    assert bits_equal(port.transfer_apply(my, hy, m, h, g["y"]), g["yhat"])
    assert bits_equal(port.transfer_apply_transpose(my, hy, m, h, g["w_img"]), g["ptw"])
    ngf = port.ngf(g["ref"], m, h, tau, rho)
    ngf.populate(g["tpl"], g["yhat"])
    ws = ngf.workspace()
    for k in ("values", "partials", "residual", "inv1", "inv2", "tpl_grads", "ref_grads"):
        assert bits_equal(ws[k], g[k]), k
    n = int(np.prod(m))
    rh = np.concatenate([[ngf.rho(i, k) for i in range(n)] for k in range(7)])
    assert bits_equal(rh, g["rho_hat"])
    assert bits_equal(ngf.value(), g["D"])
    assert bits_equal(ngf.gradient(), g["g_img"])
    assert bits_equal(ngf.hessian_vec(g["p_img"]), g["hv_img"])
    obj = port.objective(g["ref"], g["tpl"], m, h, my, tau, rho, alpha)
    J, D, S, grad = obj.eval(g["y"])
    assert bits_equal([J, D, S], [g["J"], g["Dobj"], g["S"]]) and bits_equal(grad, g["grad"])
    assert bits_equal(obj.eval(g["y"], want_grad=False)[0], g["Jv"])
    assert bits_equal(obj.gn_hessian_vec(g["p_nod"]), g["gn_hv"])
    assert bits_equal(obj.seed_hessian_vec(g["p_nod"], 1e-3), g["seed_hv"])
    assert bits_equal(port.curvature_value(g["u"], my, hy), g["curv_val"])
    assert bits_equal(port.curvature_gradient(g["u"], my, hy), g["curv_grad"])
    ny = int(np.prod(my))
    assert bits_equal(port.laplacian_apply(g["u"][:ny], my, hy), g["lap"])
    x, it, rr, bd = obj.cg_solve(-g["grad"], 50, 1e-2)
    assert it == int(g["cg_iters"]) and bits_equal(x, g["cg_x"]) and bits_equal(rr, g["cg_relres"])


@pytest.mark.parametrize("path", golden_files("solve"), ids=lambda p: p.split("/")[-1])
def test_port_solvers_match_golden(port, path):
    g = load(path)
    m, h, my = tup(g["m"]), tup(g["h"], float), tup(g["my"])
    obj = port.objective(g["ref"], g["tpl"], m, h, my, float(g["tau"]), float(g["rho"]), float(g["alpha"]))
    y, trace, lsf = obj.minimize(obj.identity(), str(g["method"]), OptConfig.defaults(max_iters=int(g["max_iters"])))
    assert bits_equal(y, g["y"])
    assert bits_equal(np.array(trace, dtype=np.float64), g["trace"])
    assert lsf == bool(g["lsf"])


@pytest.mark.parametrize("path", golden_files("ml"), ids=lambda p: p.split("/")[-1])
def test_port_multilevel_matches_golden(port, path):
    g = load(path)
    m, h = tup(g["m"]), tup(g["h"], float)
    y, my, traces, lsf = port.register_multilevel(g["ref"], g["tpl"], m, h, levels=int(g["levels"]),
                                                  method=str(g["method"]),
                                                  cfg=OptConfig.defaults(max_iters=int(g["max_iters"])))
    assert tuple(my) == tup(g["my"])
    assert bits_equal(y, g["y"])
    assert bits_equal(np.array([r for t in traces for r in t], dtype=np.float64), g["trace"])


@pytest.mark.parametrize("case", [((11, 9, 7), (0.97, 0.97, 2.5), 3), ((13, 12, 5), (0.7, 0.7, 0.7), 4),
                                  ((6, 1, 5), (1.0, 1.0, 1.0), 2)])
def test_port_equals_reference_library(port, ref, case):
    m, h, ratio = case
    R = ref.make_phantom(m, h) * 1000.0
    T = ref.warp_sinusoid(R, m, h, 2.0, 7)
    assert bits_equal(port.make_phantom(m, h) * 1000.0, R)
    assert bits_equal(port.warp_sinusoid(R, m, h, 2.0, 7), T)
    my, hy = ref.deformation_grid_for(m, h, ratio)
    rng = np.random.default_rng(3)
    oR = ref.objective(R, T, m, h, my)
    oP = port.objective(R, T, m, h, my)
    y = oR.identity() + rng.uniform(-0.3, 0.3, oR.dof)
    a, b = oR.eval(y), oP.eval(y)
    assert bits_equal(a[:3], b[:3]) and bits_equal(a[3], b[3])
    p = rng.uniform(-1, 1, oR.dof)
    assert bits_equal(oR.gn_hessian_vec(p), oP.gn_hessian_vec(p))


def test_port_random_volume_and_warp_terms(port, ref):
    assert bits_equal(port.make_random_volume((5, 4, 3), (1, 1, 1), 99, 2), ref.make_random_volume((5, 4, 3), (1, 1, 1), 99, 2))
    for s in (1, 42, 12345):
        a, b = port.sinusoid_terms((64.0, 50.0, 30.0), 3.0, s), ref.sinusoid_terms((64.0, 50.0, 30.0), 3.0, s)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


# ---- known-answer tests restated from the reference's unit suites -----------------

def identity_points(m, h):
    ax = [(np.arange(m[a]) + 0.5) * h[a] for a in range(3)]
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return np.concatenate([x.ravel(), y.ravel(), z.ravel()])


def test_identical_images_zero_distance(port):  # test_ngf.cpp:72-90
    m, h = (6, 6, 6), (1.0, 1.0, 1.0)
    r = port.make_phantom(m, h)
    ngf = port.ngf(r, m, h, 10.0, 10.0)
    ngf.populate(r, identity_points(m, h))
    assert np.allclose(ngf.workspace()["residual"], 1.0, rtol=1e-12)
    assert abs(ngf.value()) < 1e-10


def test_constant_images_unit_residual_zero_gradient(port):  # test_ngf.cpp:92-117
    m, h = (4, 4, 4), (1.0, 1.0, 1.0)
    ngf = port.ngf(np.full(64, 2.0), m, h, 3.0, 7.0)
    ngf.populate(np.full(64, 5.0), identity_points(m, h))
    assert np.allclose(ngf.workspace()["residual"], 1.0)
    assert np.all(ngf.gradient() == 0.0)


def test_transfer_partition_of_unity_and_adjoint(port):  # test_transfer.cpp:42-127
    m, h, my = (7, 6, 5), (1.0, 2.0, 1.5), (4, 3, 3)
    hy = port.make_deform_grid(m, h, my)
    ny, n = int(np.prod(my)), int(np.prod(m))
    ones = np.ones(3 * ny)
    assert np.allclose(port.transfer_apply(my, hy, m, h, ones), 1.0, atol=1e-14)
    ax = [np.arange(my[a]) * hy[a] for a in range(3)]
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    xy = np.concatenate([x.ravel(), y.ravel(), z.ravel()])
    assert np.allclose(port.transfer_apply(my, hy, m, h, xy), identity_points(m, h), atol=1e-13)
    rng = np.random.default_rng(0)
    for _ in range(5):
        p, w = rng.uniform(-1, 1, 3 * ny), rng.uniform(-1, 1, 3 * n)
        a = port.transfer_apply(my, hy, m, h, p) @ w
        b = p @ port.transfer_apply_transpose(my, hy, m, h, w)
        assert abs(a - b) <= 1e-12 * max(1.0, abs(a))


def test_curvature_spike_and_value(port):  # test_curvature.cpp:40-85
    m, h = (5, 5, 5), (1.0, 1.0, 1.0)
    u = np.zeros(125)
    u[62] = 1.0  # centre
    lap = port.laplacian_apply(u, m, h)
    assert lap[62] == -6.0 and lap[61] == 1.0 and lap[63] == 1.0
    u3 = np.concatenate([u, np.zeros(125), np.zeros(125)])
    assert port.curvature_value(u3, m, h) == pytest.approx(42.0)  # 36 + 6*1
    u3c = np.concatenate([np.full(125, 1.0), np.full(125, -2.5), np.full(125, 0.75)])
    assert port.curvature_value(u3c, m, h) == 0.0


def test_gn_hessian_symmetric_psd(port):  # acceptance.cpp:209-286
    m, h, my = (7, 7, 7), (1.0, 1.0, 1.0), (4, 4, 4)
    R = port.make_random_volume(m, h, 4001, 1)
    T = port.make_random_volume(m, h, 4002, 1)
    obj = port.objective(R, T, m, h, my, 1.0, 1.0, 0.5)
    rng = np.random.default_rng(4003)
    y = obj.identity() + rng.uniform(-0.3, 0.3, obj.dof)
    obj.eval(y, want_grad=False)
    for _ in range(10):
        p, q = rng.uniform(-0.3, 0.3, obj.dof), rng.uniform(-0.3, 0.3, obj.dof)
        hp, hq = obj.gn_hessian_vec(p), obj.gn_hessian_vec(q)
        assert abs(hp @ q - p @ hq) <= 1e-12 * max(1.0, abs(hp @ q))
        assert hp @ p >= -1e-10 * (p @ p)


def test_objective_gradient_finite_difference(port):  # acceptance.cpp:164-207
    m, my = (8, 8, 8), (5, 5, 5)
    R = port.make_random_volume(m, (1, 1, 1), 3001, 2)
    T = port.make_random_volume(m, (1, 1, 1), 3002, 2)
    obj = port.objective(R, T, m, (1.0, 1.0, 1.0), my, 1.0, 1.0, 1.0)
    rng = np.random.default_rng(3003)
    y0 = obj.identity() + rng.uniform(-0.2, 0.2, obj.dof)
    g = obj.eval(y0)[3]
    worst = 0.0
    for _ in range(5):
        v = rng.uniform(-0.2, 0.2, obj.dof)
        gv = g @ v
        best = min(abs((obj.eval(y0 + e * v, False)[0] - obj.eval(y0 - e * v, False)[0]) / (2 * e) - gv)
                   / max(1e-12, abs(gv)) for e in (1e-4, 3e-5, 1e-5, 3e-6, 1e-6))
        worst = max(worst, best)
    assert worst <= 1e-6


def test_ngf_against_sparse_chain(ref):  # acceptance.cpp:91-162 (oracle.cpp:223-293)
    m, h, my = (7, 6, 8), (1.0, 1.0, 1.0), (4, 5, 4)
    R = ref.make_random_volume(m, h, 2000, 1)
    T = ref.make_random_volume(m, h, 2001, 1)
    hy = ref.make_deform_grid(m, h, my)
    rng = np.random.default_rng(2002)
    ax = [np.arange(my[a]) * hy[a] for a in range(3)]
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    yv = np.concatenate([x.ravel(), y.ravel(), z.ravel()]) + rng.uniform(-0.4, 0.4, 3 * int(np.prod(my)))
    ngf = ref.ngf(R, m, h, 1.0, 1.0)
    ngf.populate(T, ref.transfer_apply(my, hy, m, h, yv))
    p = rng.uniform(-1, 1, 3 * int(np.prod(m)))
    g_or, hv_or = ngf.oracle_image(my, p)
    assert max_rel(ngf.gradient(), g_or) <= 1e-12
    assert max_rel(ngf.hessian_vec(p), hv_or) <= 1e-12
