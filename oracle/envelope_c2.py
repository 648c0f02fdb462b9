"""Test infrastructure: the reference's own 1-ulp envelope at BASELINE C2 (128^3, 3-level GN).

Runs the unmodified reference library (oracle/_ref) on the C2 pair with the template moved by
one ulp (every voxel, toward +inf and toward -inf) and reports how far each final displacement
field lands from the unperturbed run (tests/golden/c2_gn.npz), in image voxels. Fast mode's
rounding differs from the reference's at the 1e-16 level per operation, so its final field can be
held to no tighter bound than this: tests/test_gpu_configs.py::test_c2_multilevel_gn uses the
envelope this script writes to tests/golden/c2_envelope.json. About 9 min per run on 8 threads.

    python oracle/envelope_c2.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle.oracle import Oracle  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")


def main():
    g = np.load(os.path.join(GOLDEN, "c2_gn.npz"))
    o = Oracle("ref")
    o.set_threads(os.cpu_count() or 1)
    m, h = tuple(int(v) for v in g["m"]), tuple(float(v) for v in g["h"])
    ref = o.make_phantom(m, h) * 1000.0
    tpl = o.warp_sinusoid(ref, m, h, 3.0, 42)
    out = {"config": "C2 128^3 3-level GN, reference library (oracle/_ref)", "runs": []}
    for name, direction in (("tpl+1ulp", np.inf), ("tpl-1ulp", -np.inf)):
        t = np.nextafter(tpl, direction)
        y, _, traces, _ = o.register_multilevel(ref, t, m, h, levels=3, method="gn")
        d = np.abs(y - g["y"]).reshape(3, -1) / np.array(h)[:, None]
        run = {"perturbation": name, "max_voxel": float(d.max()), "mean_voxel": float(d.mean()),
               "level_iters": [len(tr) for tr in traces]}
        print(run, flush=True)
        out["runs"].append(run)
    out["max_voxel"] = max(r["max_voxel"] for r in out["runs"])
    out["mean_voxel"] = max(r["mean_voxel"] for r in out["runs"])
    with open(os.path.join(GOLDEN, "c2_envelope.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(out)


if __name__ == "__main__":
    main()
