"""f3/f4 measurement: MetaImage ingest (MET_SHORT payload -> fp64 on the GPU), the CLI warp
and landmark errors, timed beside the reference library on the host cores (oracle/_ref).
Writes one JSON line. Files live in a temporary directory (page cache warm: the second
read of each file is timed)."""
import json, os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1804_10541_b200 as P
from oracle.oracle import Oracle, available
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_io import write_mha  # noqa: E402

m = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (512, 512, 225)
h = (0.7, 0.7, 0.7)
n = int(np.prod(m))
o = Oracle("ref") if available("ref") else None
if o:
    o.set_threads(os.cpu_count() or 1)
res = {"volume": list(m), "threads": os.cpu_count()}
with tempfile.TemporaryDirectory() as d:
    path = os.path.join(d, "v.mha")
    data = np.random.default_rng(0).integers(-1024, 3000, n).astype(np.int16)
    write_mha(path, data, m, h, "MET_SHORT")
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        vol, img = P.io.read_volume(path, device=True)
        torch.cuda.synchronize(); t_ours = time.perf_counter() - t0
    res["read_volume_ours_s"] = t_ours
    res["read_volume_ours_GBps_payload"] = 2 * n / t_ours / 1e9
    if o:
        o.io_read_volume(path)
        t0 = time.perf_counter(); o.io_read_volume(path); t_ref = time.perf_counter() - t0
        res["read_volume_ref_s"] = t_ref
    dg = P.deformation_grid_for(img, 4)
    y = dg.point_coords() + np.random.default_rng(1).uniform(-1.5, 1.5, 3 * dg.count())
    yd = torch.from_numpy(y).cuda()
    P.io.warp_volume(vol, img, yd, dg); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        out = P.io.warp_volume(vol, img, yd, dg)
    torch.cuda.synchronize()
    t_w = (time.perf_counter() - t0) / 5
    res["warp_ours_s"] = t_w
    res["warp_ours_Gvox_s"] = n / t_w / 1e9
    if o:
        sub = (m[0], m[1], 16)  # bounded CPU sample: 16 planes, rate scaled per voxel
        subimg = P.make_image_grid(sub, h)
        sdg = P.deformation_grid_for(subimg, 4)
        sy = sdg.point_coords()
        sv = np.random.default_rng(2).standard_normal(subimg.count())
        t0 = time.perf_counter()
        pts = o.transfer_apply(sdg.m, sdg.h, sub, h, sy)
        o.sample_deformed(sv, sub, h, pts)
        t_rs = time.perf_counter() - t0
        res["warp_ref_Gvox_s"] = subimg.count() / t_rs / 1e9
        res["warp_ref_sample"] = f"{sub} volume"
    rng = np.random.default_rng(3)
    k = 100000
    fx = (rng.integers(0, m, (k, 3)) + 0.5) * np.array(h)
    mv = fx + rng.uniform(-2, 2, (k, 3))
    P.io.landmark_error(fx, mv, yd, dg)
    t0 = time.perf_counter(); st = P.io.landmark_error(fx, mv, yd, dg); t_l = time.perf_counter() - t0
    res["landmark_error_ours_s_100k"] = t_l
    if o:
        t0 = time.perf_counter(); rst = o.io_landmark_error(fx, mv, y, dg.m, dg.h); t_lr = time.perf_counter() - t0
        res["landmark_error_ref_s_100k"] = t_lr
        res["landmark_error_bitwise_equal"] = bool(st[0] == rst[0] and st[1] == rst[1])
print(json.dumps(res))
