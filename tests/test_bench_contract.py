"""bench.py contract checks that need no GPU: the reference arm (`--impl reference`) prints one
JSON line with the keys the driver reads, runs the driver's K / W steps, describes the same
workload as our arm (`config`), and maps only the checker libraries — never libmfreg_cuda.so."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)


def test_bench_config_nodal_grid_matches_reference_rule():
    """config.nodal is deformation_grid_for(image, RATIO) (multilevel.cpp:39-49) for every workload;
    checked against the oracle's restatement of the reference function."""
    import bench
    from oracle.oracle import Oracle, available

    if not available("port"):
        pytest.skip("oracle port not built")
    o = Oracle("port")
    for name, wl in bench.WORKLOADS.items():
        cfg = bench.bench_config(wl, "fast", 1, False)
        my, _ = o.deformation_grid_for(wl["m"], wl["h"], bench.RATIO)
        assert cfg["nodal"] == [int(v) for v in my], name
        assert cfg["image"] == list(wl["m"]) and cfg["spacing"] == list(wl["h"])
        assert cfg["parallelism"] == "single GPU"
    assert bench.bench_config(bench.WORKLOADS["c4"], "fast", 4, False)["parallelism"].startswith("z slabs x4")


_RUN = r"""
import json, runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--workload", "c2", "--steps", "2", "--warmup", "1"]
try:
    runpy.run_path("bench.py", run_name="__main__")
finally:
    maps = open("/proc/self/maps").read()
    print(json.dumps({"mapped_cuda_lib": "libmfreg_cuda" in maps, "mapped_ref": "libmfreg_ref" in maps}))
"""


@pytest.mark.timeout(600)
def test_reference_arm_line():
    from oracle.oracle import available

    if not available("ref") and not available("port"):
        pytest.skip("no checker library built")
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "4"))
    out = subprocess.run([sys.executable, "-c", _RUN], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 2, out.stdout
    line, maps = json.loads(lines[0]), json.loads(lines[1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    import bench
    assert line["config"] == bench.bench_config(bench.WORKLOADS["c2"], "fast", 1, False)
    assert not maps["mapped_cuda_lib"]
    assert maps["mapped_ref"] == (line["cpu_baseline"]["kind"] == "reference")
