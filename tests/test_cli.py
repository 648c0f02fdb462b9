"""The command line (python -m paper_1804_10541_b200) against the reference CLI's
behaviour (tools/mfreg_cli.cpp:26-158): same options and printed keys; in parity
mode the printed trace and the written files equal what the reference library
produces for the same inputs."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1804_10541_b200", *map(str, args)], cwd=ROOT,
                          capture_output=True, text=True)


def test_cli_parses_and_reports_errors(tmp_path):
    r = run_cli("--help")
    assert r.returncode == 0 and "register" in r.stdout and "eval-landmarks" in r.stdout
    r = run_cli("register", "--fixed", tmp_path / "none.mha", "--moving", tmp_path / "none.mha",
                "--out-deformation", tmp_path / "y.def")
    assert r.returncode == 1 and r.stderr.startswith("error: cannot open ")


@pytest.mark.gpu
def test_cli_register_warp_landmarks_match_reference(oracle, tmp_path):
    from test_io import write_mha
    m, h = (24, 20, 18), (0.97, 0.97, 2.5)
    R = oracle.make_phantom(m, h) * 1000.0
    T = oracle.warp_sinusoid(R, m, h, 3.0, 42)
    write_mha(str(tmp_path / "f.mha"), R, m, h, "MET_DOUBLE")
    write_mha(str(tmp_path / "m.mha"), T, m, h, "MET_DOUBLE")
    r = run_cli("register", "--fixed", tmp_path / "f.mha", "--moving", tmp_path / "m.mha", "--out-deformation",
                tmp_path / "y.def", "--out-warped", tmp_path / "w.mha", "--levels", 2, "--optimizer", "gn",
                "--max-iters", 4)
    assert r.returncode == 0, r.stderr
    lines = dict(l.split(": ", 1) for l in r.stdout.splitlines())
    assert int(lines["peak-derivative-buffer-bytes"]) > 0  # the reference's key (mfreg_cli.cpp:88-89)
    from oracle.gen_golden import nodal_coords
    from oracle.oracle import OptConfig
    y_ref, my, traces, _ = oracle.register_multilevel(R, T, m, h, levels=2, method="gn",
                                                      cfg=OptConfig.defaults(max_iters=4))
    for l, tr in enumerate(traces):
        assert lines[f"level.{l}.iterations"] == str(len(tr))
        for rec in tr:
            it, cg, j, d, s, g, st = rec
            assert lines[f"level.{l}.iter.{int(it)}"] == (f"J={j:.10e} D={d:.10e} aS={s:.10e} grad={g:.4e} "
                                                         f"step={st:.3g} cg={int(cg)}")
    hy = oracle.make_deform_grid(m, h, my)
    oracle.io_write_deformation(tmp_path / "ref.def", y_ref, my, hy)
    assert (tmp_path / "y.def").read_bytes() == (tmp_path / "ref.def").read_bytes()
    assert (tmp_path / "y.def.meta").read_bytes() == (tmp_path / "ref.def.meta").read_bytes()
    pts = oracle.transfer_apply(my, hy, m, h, y_ref)
    warped, _ = oracle.sample_deformed(T, m, h, pts)
    oracle.io_write_volume(tmp_path / "ref_w.mha", warped, m, h)
    assert (tmp_path / "w.mha").read_bytes() == (tmp_path / "ref_w.mha").read_bytes()
    # warp command on the written files
    r = run_cli("warp", "--input", tmp_path / "m.mha", "--deformation", tmp_path / "y.def", "--out", tmp_path / "w2.mha")
    assert r.returncode == 0 and r.stdout == f"command: warp\nwrote: {tmp_path / 'w2.mha'}\n"
    assert (tmp_path / "w2.mha").read_bytes() == (tmp_path / "ref_w.mha").read_bytes()
    # eval-landmarks
    rng = np.random.default_rng(0)
    idx = rng.integers(0, m, (50, 3))
    (tmp_path / "lf.txt").write_text("\n".join(" ".join(map(str, r_)) for r_ in idx) + "\n")
    (tmp_path / "lm.txt").write_text("\n".join(" ".join(map(str, r_ + 1)) for r_ in idx) + "\n")
    r = run_cli("eval-landmarks", "--fixed-landmarks", tmp_path / "lf.txt", "--moving-landmarks", tmp_path / "lm.txt",
                "--deformation", tmp_path / "y.def", "--spacing", *h)
    assert r.returncode == 0, r.stderr
    fx = oracle.io_read_landmarks(tmp_path / "lf.txt", h)
    mv = oracle.io_read_landmarks(tmp_path / "lm.txt", h)
    b = oracle.io_landmark_error(fx, mv, nodal_coords(my, hy), my, hy)
    a = oracle.io_landmark_error(fx, mv, y_ref, my, hy)
    assert r.stdout == (f"command: eval-landmarks\nlandmarks: 50\nerror-before: {b[0]:.6f} +- {b[1]:.6f}\n"
                        f"error-after: {a[0]:.6f} +- {a[1]:.6f}\n")


@pytest.mark.gpu
def test_cli_selftest():
    r = run_cli("selftest")
    assert r.returncode == 0, r.stdout + r.stderr
    for name in ("parity-gradient", "parity-hvp", "transfer-adjoint", "gn-symmetry", "gn-psd", "gradient-fd"):
        assert f"selftest.{name}: pass" in r.stdout
    assert r.stdout.endswith("selftest.failures: 0\n")
