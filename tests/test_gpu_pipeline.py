"""Host-buffer calls with pipelined copies (DeviceObjective::eval_host / hv_host):
the operand is copied in nodal z chunks ahead of the warp / Hv pass, which run in z groups, and
each group's nodes are finalized and copied out while the next group runs. The results must be
those of the same objective called with device buffers (same per-tile arithmetic, fixed-order
gathers and D ticket; the pipeline's own plan caps z chunks at 128 planes, so on grids where the
device plan chunks longer the sums group differently in the last bits), in fast and FAST32 mode;
the pipeline is forced on at these small grids with MFREG_PIPE_MIN_MB=0 and checked to have run
(it launches per z group)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [((128, 96, 120), (0.7, 0.7, 0.7), 4, 1.0), ((96, 64, 80), (0.97, 0.97, 2.5), 3, 1.0),
          ((160, 128, 64), (1.0, 1.0, 1.0), 4, 0.0), ((160, 160, 64), (1.0, 1.0, 1.0), 4, 1.0),
          ((64, 64, 260), (1.0, 1.0, 1.0), 4, 0.5)]


def _run(P, torch, R, T, m, h, ratio, alpha, mode, y, p, host, pipe):
    env = {"MFREG_PIPE_MIN_MB": "0", "MFREG_NO_PIPE": "0" if pipe else "1"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        img = P.make_image_grid(m, h)
        dg = P.deformation_grid_for(img, ratio)
        obj = P.Objective(torch.from_numpy(R).cuda(), torch.from_numpy(T).cuda(), img, dg, P.NgfParams(), alpha, mode)
        n0 = P.launch_count()
        if host:
            g = np.empty_like(y)
            j = obj.eval(y.copy(), g)
            q = np.empty_like(p)
            obj.gn_hessian_vec(p.copy(), q)
        else:
            yd, pd = torch.from_numpy(y).cuda(), torch.from_numpy(p).cuda()
            gd, qd = torch.empty_like(yd), torch.empty_like(pd)
            j = obj.eval(yd, gd)
            obj.gn_hessian_vec(pd, qd)
            torch.cuda.synchronize()
            g, q = gd.cpu().numpy(), qd.cpu().numpy()
        return j, g, q, P.launch_count() - n0
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("mode", ["fast", "fast32"])
@pytest.mark.parametrize("case", SHAPES, ids=lambda c: "x".join(map(str, c[0])) + f"_r{c[2]}_a{c[3]}")
def test_host_pipeline_bitwise(P, oracle, case, mode):
    import torch

    m, h, ratio, alpha = case
    md = P.Mode.FAST if mode == "fast" else P.Mode.FAST32
    if md == P.Mode.FAST32 and m[0] % 4:
        pytest.skip("FAST32 needs mx % 4 == 0")
    R = oracle.make_phantom(m, h) * 1000.0
    T = oracle.warp_sinusoid(R, m, h, 3.0, 42)
    img = P.make_image_grid(m, h)
    dg = P.deformation_grid_for(img, ratio)
    rng = np.random.default_rng(5)
    y = dg.point_coords() + rng.uniform(-0.4, 0.4, 3 * dg.count())
    p = rng.uniform(-1.0, 1.0, 3 * dg.count())
    jd, gd, qd, _ = _run(P, torch, R, T, m, h, ratio, alpha, md, y, p, host=False, pipe=False)
    jh, gh, qh, n_pipe = _run(P, torch, R, T, m, h, ratio, alpha, md, y, p, host=True, pipe=True)
    js, gs, qs, n_staged = _run(P, torch, R, T, m, h, ratio, alpha, md, y, p, host=True, pipe=False)
    assert n_pipe > n_staged, "the pipelined host path did not run (no z groups)"
    # the staged host path runs the device calls' plan: bitwise
    for a, b in ((gs, gd), (qs, qd)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert js == jd
    # the pipeline runs its own plan (z chunks of <= 128 planes): bitwise where the chunkings
    # coincide (these grids), else the same sums grouped per other plane ranges (last bits)
    for a, b in ((gh, gd), (qh, qd)):
        assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))
    assert abs(jh - jd) <= 1e-13 * abs(jd)
