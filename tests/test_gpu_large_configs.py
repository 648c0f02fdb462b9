"""Operator parity at the geometry of the large BASELINE configs, against the unmodified
reference library run live on the host (oracle/_ref, built in-tree):

* C4 (512x512x900 thorax-abdomen, h = 0.7 — the interpolation-tie spacing of SURVEY H1): the
  full 512x512 x-y extent on a z sub-volume of 48 planes, nodal ratio 4 (129x129x13);
* C5 (1024^3 derivative sweep, h = 1): the full 1024x1024 x-y extent on 16 planes (257x257x5).

Inputs come from the reference's own generators (synthetic.cpp: phantom x1000, sinusoid warp
amp 3 seed 42); y = identity + U(-0.3, 0.3), p ~ U(-1, 1). Checked: J and the value-only J,
the gradient and the GN Hv — bitwise in parity mode, max-rel <= 1e-9 in fast mode and
<= 1e-4 in FAST32 (metric of tests/acceptance.cpp:40-50)."""
import numpy as np
import pytest

from conftest import bits_equal, max_rel

pytestmark = pytest.mark.gpu

CASES = {
    "c4_subvolume": ((512, 512, 48), (0.7, 0.7, 0.7)),
    "c5_subslab": ((1024, 1024, 16), (1.0, 1.0, 1.0)),
}


@pytest.fixture(scope="module", params=sorted(CASES))
def case(request, oracle):
    m, h = CASES[request.param]
    import os
    oracle.set_threads(os.cpu_count() or 1)
    R = oracle.make_phantom(m, h) * 1000.0
    T = oracle.warp_sinusoid(R, m, h, 3.0, 42)
    my, _ = oracle.deformation_grid_for(m, h, 4)
    ref = oracle.objective(R, T, m, h, my, 10.0, 10.0, 1.0)
    rng = np.random.default_rng(17)
    y = ref.identity() + rng.uniform(-0.3, 0.3, ref.dof)
    p = rng.uniform(-1.0, 1.0, ref.dof)
    Jv = ref.eval(y, want_grad=False)[0]
    J, D, S, grad = ref.eval(y)
    hv = ref.gn_hessian_vec(p)
    return dict(name=request.param, m=m, h=h, my=my, R=R, T=T, y=y, p=p, J=J, Jv=Jv, grad=grad, hv=hv)


@pytest.mark.parametrize("mode", ["PARITY", "FAST", "FAST32"])
def test_large_config_operators(P, case, mode):
    import torch
    img = P.make_image_grid(case["m"], case["h"])
    dg = P.deformation_grid_for(img, 4)
    assert dg.m == tuple(case["my"])
    R, T = torch.from_numpy(case["R"]).cuda(), torch.from_numpy(case["T"]).cuda()
    obj = P.Objective(R, T, img, dg, P.NgfParams(), 1.0, getattr(P.Mode, mode))
    y, p = torch.from_numpy(case["y"]).cuda(), torch.from_numpy(case["p"]).cuda()
    Jv = obj.eval(y)
    g = torch.empty_like(y)
    J = obj.eval(y, g)
    q = obj.gn_hessian_vec(p, torch.empty_like(p))
    g, q = g.cpu().numpy(), q.cpu().numpy()
    if mode == "PARITY":
        assert J == case["J"] and Jv == case["Jv"]
        assert bits_equal(g, case["grad"]) and bits_equal(q, case["hv"])
    else:
        tol = 1e-9 if mode == "FAST" else 1e-4
        assert abs(J - case["J"]) <= tol * abs(case["J"]) and abs(Jv - case["Jv"]) <= tol * abs(case["Jv"])
        assert max_rel(g, case["grad"]) <= tol, max_rel(g, case["grad"])
        assert max_rel(q, case["hv"]) <= tol, max_rel(q, case["hv"])
