"""Volume / deformation / landmark files: the library's
io API (paper_1804_10541_b200.io over the C ABI) against the unmodified
reference library's io:: functions (oracle fixture) on the same files —
bit-identical data, byte-identical written files, identical error types and
messages. GPU tests: payload conversion, landmark errors and the warp run on
the device."""
import os

import numpy as np
import pytest

from conftest import bits_equal

TYPES = {"MET_SHORT": np.int16, "MET_USHORT": np.uint16, "MET_FLOAT": np.float32, "MET_DOUBLE": np.float64}


def write_mha(path, data, m, h, etype, local=True, crlf=False, extra=None):
    nl = "\r\n" if crlf else "\n"
    lines = ["ObjectType = Image", "NDims = 3", f"DimSize = {m[0]} {m[1]} {m[2]}",
             f"ElementSpacing = {h[0]!r} {h[1]!r} {h[2]!r}", f"ElementType = {etype}"] + (extra or [])
    raw = np.ascontiguousarray(data, dtype=TYPES.get(etype, np.float64)).astype("<" + np.dtype(TYPES.get(etype, np.float64)).str[1:]).tobytes()
    if local:
        lines.append("ElementDataFile = LOCAL")
        with open(path, "wb") as f:
            f.write((nl.join(lines) + nl).encode() + raw)
    else:
        rawname = os.path.basename(path) + ".raw"
        lines.append(f"ElementDataFile = {rawname}")
        with open(path, "wb") as f:
            f.write((nl.join(lines) + nl).encode())
        with open(os.path.join(os.path.dirname(path), rawname), "wb") as f:
            f.write(raw)


def need_ref(oracle):
    if oracle.kind != "ref":
        pytest.skip("reference library not built")


def test_reference_io_wrappers_roundtrip(oracle, tmp_path):
    """CPU: the oracle's io wrappers (checker infrastructure) read what they write."""
    need_ref(oracle)
    m, h = (5, 4, 3), (1.0, 0.5, 2.0)
    v = np.random.default_rng(0).standard_normal(60)
    oracle.io_write_volume(tmp_path / "a.mha", v, m, h)
    d, mm, hh = oracle.io_read_volume(tmp_path / "a.mha")
    assert bits_equal(d, v) and mm == m and hh == h


@pytest.mark.gpu
@pytest.mark.parametrize("etype", list(TYPES))
@pytest.mark.parametrize("local", [True, False])
def test_read_volume_matches_reference(P, oracle, tmp_path, etype, local):
    need_ref(oracle)
    rng = np.random.default_rng(1)
    m, h = (37, 23, 11), (0.97, 0.97, 2.5)
    n = int(np.prod(m))
    if etype in ("MET_SHORT", "MET_USHORT"):
        info = np.iinfo(TYPES[etype])
        data = rng.integers(info.min, info.max, n, endpoint=True)
    else:
        data = rng.standard_normal(n) * 1e3
    path = str(tmp_path / "v.mha")
    write_mha(path, data, m, h, etype, local=local, crlf=not local)
    ref, rm, rh = oracle.io_read_volume(path)
    got, g = P.io.read_volume(path)
    assert g.m == rm and g.h == rh and bits_equal(got, ref)
    dev, g2 = P.io.read_volume(path, device=True)
    assert bits_equal(dev.cpu().numpy(), ref)


BAD_HEADERS = [
    ("missing_datafile", lambda p: open(p, "wb").write(b"NDims = 3\nDimSize = 2 2 2\n")),
    ("malformed_line", lambda p: open(p, "wb").write(b"NDims = 3\nthis line has no equals\nElementDataFile = LOCAL\n")),
    ("ndims", lambda p: write_mha(p, np.zeros(8), (2, 2, 2), (1, 1, 1), "MET_DOUBLE", extra=[]) or
     open(p, "r+b").write(b"ObjectType = Image\nNDims = 2")),
    ("payload_size", lambda p: write_mha(p, np.zeros(7), (2, 2, 2), (1, 1, 1), "MET_DOUBLE")),
    ("two_dims", lambda p: open(p, "wb").write(b"NDims = 3\nDimSize = 2 2\nElementSpacing = 1 1 1\n"
                                               b"ElementType = MET_DOUBLE\nElementDataFile = LOCAL\n")),
    ("unknown_type", lambda p: write_mha(p, np.zeros(8), (2, 2, 2), (1, 1, 1), "MET_UCHAR")),
    ("missing_raw", lambda p: open(p, "wb").write(b"NDims = 3\nDimSize = 2 2 2\nElementSpacing = 1 1 1\n"
                                                  b"ElementType = MET_DOUBLE\nElementDataFile = nowhere.raw\n")),
    ("bad_spacing", lambda p: write_mha(p, np.zeros(8), (2, 2, 2), (1, 0, 1), "MET_DOUBLE")),
    ("no_file", None),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,make", BAD_HEADERS, ids=[b[0] for b in BAD_HEADERS])
def test_read_volume_errors_match_reference(P, oracle, tmp_path, name, make):
    need_ref(oracle)
    path = str(tmp_path / "bad.mha")
    if make is not None:
        make(path)
    with pytest.raises((RuntimeError, ValueError)) as ref_e:
        oracle.io_read_volume(path)
    with pytest.raises(type(ref_e.value)) as our_e:
        P.io.read_volume(path)
    assert str(our_e.value) == str(ref_e.value)


@pytest.mark.gpu
def test_write_volume_byte_identical(P, oracle, tmp_path):
    need_ref(oracle)
    m, h = (19, 7, 5), (0.1, 1.0 / 3.0, 2.5)
    img = P.make_image_grid(m, h)
    v = np.random.default_rng(2).standard_normal(img.count())
    oracle.io_write_volume(tmp_path / "ref.mha", v, m, h)
    P.io.write_volume(tmp_path / "ours.mha", v, img)
    import torch
    P.io.write_volume(tmp_path / "ours_dev.mha", torch.from_numpy(v).cuda(), img)
    ref = (tmp_path / "ref.mha").read_bytes()
    assert (tmp_path / "ours.mha").read_bytes() == ref and (tmp_path / "ours_dev.mha").read_bytes() == ref
    back, g = P.io.read_volume(tmp_path / "ours.mha")
    assert bits_equal(back, v) and g.m == m and g.h == h


@pytest.mark.gpu
def test_deformation_files_match_reference(P, oracle, tmp_path):
    need_ref(oracle)
    img = P.make_image_grid((40, 36, 32), (0.97, 0.97, 2.5))
    dg = P.deformation_grid_for(img, 4)
    y = dg.point_coords() + np.random.default_rng(3).uniform(-0.5, 0.5, 3 * dg.count())
    oracle.io_write_deformation(tmp_path / "ref.def", y, dg.m, dg.h)
    P.io.write_deformation(tmp_path / "ours.def", y, dg)
    assert (tmp_path / "ours.def").read_bytes() == (tmp_path / "ref.def").read_bytes()
    assert (tmp_path / "ours.def.meta").read_bytes() == (tmp_path / "ref.def.meta").read_bytes()
    g = P.io.read_deformation_grid(tmp_path / "ref.def")
    assert (g.m, g.h) == oracle.io_read_deformation_grid(tmp_path / "ref.def") and g.nodal
    assert bits_equal(P.io.read_deformation(tmp_path / "ref.def", g), oracle.io_read_deformation(tmp_path / "ref.def", g.m, g.h))
    assert bits_equal(P.io.read_deformation(tmp_path / "ref.def", g, device=True).cpu().numpy(), y)
    # errors: wrong length, grid mismatch, missing sidecar
    with pytest.raises(ValueError, match="write_deformation: field length mismatch"):
        P.io.write_deformation(tmp_path / "x.def", y[:-1], dg)
    wrong = P.GridDesc(dg.m, (dg.h[0] * 2, dg.h[1], dg.h[2]), True)
    with pytest.raises(RuntimeError) as ref_e:
        oracle.io_read_deformation(tmp_path / "ref.def", wrong.m, wrong.h)
    with pytest.raises(RuntimeError, match=str(ref_e.value)):
        P.io.read_deformation(tmp_path / "ref.def", wrong)
    with pytest.raises(RuntimeError) as ref_e:
        oracle.io_read_deformation_grid(tmp_path / "none.def")
    with pytest.raises(RuntimeError) as our_e:
        P.io.read_deformation_grid(tmp_path / "none.def")
    assert str(our_e.value) == str(ref_e.value)


@pytest.mark.gpu
def test_landmarks_match_reference(P, oracle, tmp_path):
    need_ref(oracle)
    img = P.make_image_grid((48, 40, 30), (0.97, 0.97, 2.5))
    dg = P.deformation_grid_for(img, 4)
    rng = np.random.default_rng(4)
    idx_f = rng.integers(0, [48, 40, 30], (300, 3))
    idx_m = idx_f + rng.integers(-3, 4, (300, 3))
    for name, idx in (("f.txt", idx_f), ("m.txt", idx_m)):
        lines = [" ".join(str(int(v)) for v in r) for r in idx]
        lines.insert(7, "   ")  # blank lines are skipped
        (tmp_path / name).write_text("\n".join(lines) + "\n")
    sp = img.h
    fx = P.io.read_landmarks(tmp_path / "f.txt", sp)
    mv = P.io.read_landmarks(tmp_path / "m.txt", sp)
    assert bits_equal(fx, oracle.io_read_landmarks(tmp_path / "f.txt", sp))
    assert bits_equal(mv, oracle.io_read_landmarks(tmp_path / "m.txt", sp))
    for y in (dg.point_coords(), dg.point_coords() + rng.uniform(-2, 2, 3 * dg.count())):
        ref = oracle.io_landmark_error(fx, mv, y, dg.m, dg.h)
        ours = P.io.landmark_error(fx, mv, y, dg)
        assert bits_equal(ours[:2], ref[:2]) and ours[2] == ref[2] == 300
        import torch
        ours_d = P.io.landmark_error(fx, mv, torch.from_numpy(y).cuda(), dg)
        assert bits_equal(ours_d[:2], ref[:2])
    assert P.io.landmark_error(np.empty((0, 3)), np.empty((0, 3)), dg.point_coords(), dg) == (0.0, 0.0, 0)
    with pytest.raises(ValueError, match="landmark_error: list sizes differ"):
        P.io.landmark_error(fx, mv[:-1], dg.point_coords(), dg)
    with pytest.raises(ValueError, match="landmark_error: field length mismatch"):
        P.io.landmark_error(fx, mv, dg.point_coords()[:-3], dg)
    (tmp_path / "bad.txt").write_text("1 2 3\n4 5\n")
    with pytest.raises(RuntimeError) as ref_e:
        oracle.io_read_landmarks(tmp_path / "bad.txt", sp)
    with pytest.raises(RuntimeError) as our_e:
        P.io.read_landmarks(tmp_path / "bad.txt", sp)
    assert str(our_e.value) == str(ref_e.value) == "malformed landmark line 2"


@pytest.mark.gpu
def test_warp_volume_matches_reference(P, oracle, tmp_path):
    """CLI warp: T(P y) bit-identical to the reference's transfer_apply + sample_deformed."""
    need_ref(oracle)
    m, h = (40, 36, 32), (0.97, 0.97, 2.5)
    img = P.make_image_grid(m, h)
    dg = P.deformation_grid_for(img, 4)
    vol = oracle.make_phantom(m, h) * 1000.0
    y = dg.point_coords() + np.random.default_rng(5).uniform(-1.5, 1.5, 3 * dg.count())
    pts = oracle.transfer_apply(dg.m, dg.h, m, h, y)
    ref_vals, _ = oracle.sample_deformed(vol, m, h, pts)
    assert bits_equal(P.io.warp_volume(vol, img, y, dg), ref_vals)
    # end to end through files
    write_mha(str(tmp_path / "in.mha"), vol, m, h, "MET_DOUBLE")
    P.io.write_deformation(tmp_path / "y.def", y, dg)
    P.io.warp_files(tmp_path / "in.mha", tmp_path / "y.def", tmp_path / "out.mha")
    oracle.io_write_volume(tmp_path / "ref_out.mha", ref_vals, m, h)
    assert (tmp_path / "out.mha").read_bytes() == (tmp_path / "ref_out.mha").read_bytes()
    bad = P.make_image_grid((40, 36, 33), h)
    with pytest.raises(RuntimeError, match="deformation extent does not match the input volume"):
        P.io.warp_volume(np.zeros(bad.count()), bad, y, dg)
