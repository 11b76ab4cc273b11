"""Frame output (§8(f3)): CLT1 trajectory files, OBJ export and the eval CSV, checked byte for
byte against the reference's own writer/reader (the stencilcloth module compiled from
/root/reference into oracle/_ref by integration/Makefile), plus the reader's error texts.
evaluate()'s host-side validation is here too; its GPU sums are in test_gpu_eval.py."""
import os
import struct
import sys

import numpy as np
import pytest

import paper_2403_12820_b200 as ours
from paper_2403_12820_b200.trajio import read_trajectory

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "oracle", "_ref")

SCENE = """
{
  "name": "trajio_sheet",
  "grid": {"nx": 9, "ny": 6, "spacing": 0.05, "origin": [-0.2, -0.12, 0.3], "plane": "xy"},
  "material": {"stiffness": 30.0, "damping": 0.05, "mass": 0.01, "gravity": [0.0, 0.0, -9.8],
               "drag": 0.02, "pressure": 0.3},
  "time": {"dt": 0.001, "steps": 12},
  "pins": {"nodes": ["top_left", "top_right"]},
  "colliders": [{"type": "sphere", "center": [0.0, 0.0, 0.0], "radius": 0.25, "friction": 0.4}]
}
"""


def _ref():
    if not os.path.isdir(os.path.join(REF_PKG, "stencilcloth")):
        pytest.skip("reference module not built (integration/Makefile needs /root/reference)")
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    import stencilcloth as sc
    return sc


def _random_traj(seed=3, nx=7, ny=5, frames=4):
    rng = np.random.default_rng(seed)
    n = nx * ny
    return ours.Trajectory(nx, ny, 1.0 / 240, 0.125, rng.normal(0, 1, (frames, n, 3)),
                           rng.normal(0, 1, (frames, n, 3)))


def _as_ours(t):
    return ours.Trajectory(t.nx, t.ny, t.dt, t.spacing,
                           np.stack([t.positions(f) for f in range(t.frame_count)]),
                           np.stack([t.velocities(f) for f in range(t.frame_count)]))


@pytest.mark.parametrize("version", [1, 2])
def test_roundtrip_and_header(tmp_path, version):
    t = _random_traj()
    p = str(tmp_path / "a.clt1")
    ours.save_trajectory(p, t, version)
    assert not os.path.exists(p + ".tmp")
    raw = open(p, "rb").read()
    assert raw[:4] == b"CLT1"
    assert struct.unpack_from("<IIII", raw, 4) == (version, 7, 5, 4)
    assert struct.unpack_from("<dd", raw, 20) == (1.0 / 240, 0.125)
    esize = 8 if version == 1 else 4
    assert len(raw) == 36 + 4 * 2 * 35 * 3 * esize
    u = ours.load_trajectory(p)
    cast = (lambda a: a) if version == 1 else (lambda a: a.astype(np.float32).astype(np.float64))
    assert (u.nx, u.ny, u.frame_count, u.dt, u.spacing) == (7, 5, 4, t.dt, t.spacing)
    np.testing.assert_array_equal(u.frames_x, cast(t.frames_x))
    np.testing.assert_array_equal(u.frames_v, cast(t.frames_v))


@pytest.mark.parametrize("version", [1, 2])
def test_bytes_identical_to_reference_writer(tmp_path, version):
    sc = _ref()
    traj = sc.simulate(sc.parse_scene(SCENE))  # the reference's own Trajectory
    pr, po = str(tmp_path / "ref.clt1"), str(tmp_path / "ours.clt1")
    sc.save_trajectory(pr, traj, version)
    mine = ours.load_trajectory(pr)  # our reader on the reference's file
    if version == 1:
        np.testing.assert_array_equal(mine.frames_x, _as_ours(traj).frames_x)
        np.testing.assert_array_equal(mine.frames_v, _as_ours(traj).frames_v)
    ours.save_trajectory(po, _as_ours(traj), version)  # our writer, same trajectory
    assert open(po, "rb").read() == open(pr, "rb").read()
    back = sc.load_trajectory(po)  # the reference's reader on our file
    for f in range(traj.frame_count):
        np.testing.assert_array_equal(back.positions(f), mine.positions(f))
        np.testing.assert_array_equal(back.velocities(f), mine.velocities(f))


def _corrupt_cases():
    good = bytearray()
    t = _random_traj(nx=3, ny=2, frames=2)
    import io
    b = io.BytesIO()
    from paper_2403_12820_b200.trajio import write_trajectory
    write_trajectory(b, t, 1)
    good = b.getvalue()
    cases = {
        "bad_magic": b"CLT2" + good[4:],
        "version3": good[:4] + struct.pack("<I", 3) + good[8:],
        "grid_1": good[:8] + struct.pack("<I", 1) + good[12:],
        "grid_huge": good[:12] + struct.pack("<I", 70000) + good[16:],
        "zero_frames": good[:16] + struct.pack("<I", 0) + good[20:],
        "truncated_payload": good[:-5],
        "truncated_header": good[:22],
        "empty": b"",
        "nonfinite": good[:36] + struct.pack("<d", float("nan")) + good[44:],
    }
    return cases


@pytest.mark.parametrize("case", sorted(_corrupt_cases()))
def test_reader_errors_match_reference(tmp_path, case):
    sc = _ref()
    data = _corrupt_cases()[case]
    p = str(tmp_path / (case + ".clt1"))
    open(p, "wb").write(data)
    with pytest.raises(Exception) as ref_err:
        sc.load_trajectory(p)
    with pytest.raises(Exception) as our_err:
        ours.load_trajectory(p)
    assert str(our_err.value) == str(ref_err.value)
    # same exception family as the binding's translation (IoError->OSError, ConfigError->ValueError)
    for base in (OSError, ValueError):
        assert isinstance(our_err.value, base) == isinstance(ref_err.value, base)


def test_reader_errors_without_reference():
    cases = _corrupt_cases()
    with pytest.raises(ours.IoError, match=r"^not a trajectory file \(bad magic\)$"):
        read_trajectory(cases["bad_magic"])
    with pytest.raises(ours.IoError, match="^unsupported trajectory version 3$"):
        read_trajectory(cases["version3"])
    with pytest.raises(ours.IoError, match="^trajectory header: implausible grid 1x2$"):
        read_trajectory(cases["grid_1"])
    with pytest.raises(ours.IoError, match="^trajectory header: zero frames$"):
        read_trajectory(cases["zero_frames"])
    with pytest.raises(ours.IoError, match="^truncated trajectory: header declares 576 payload "
                                           "bytes, found 571$"):
        read_trajectory(cases["truncated_payload"])
    with pytest.raises(ours.ConfigError, match="frame 0 has non-finite components"):
        read_trajectory(cases["nonfinite"])
    with pytest.raises(ours.IoError, match="^cannot open trajectory /nonexistent/x.clt1$"):
        ours.load_trajectory("/nonexistent/x.clt1")
    with pytest.raises(ours.IoError, match="^unsupported trajectory version 7$"):
        ours.save_trajectory("/tmp/never_written.clt1", _random_traj(), 7)
    assert not os.path.exists("/tmp/never_written.clt1")


def test_export_obj_identical_to_reference(tmp_path):
    sc = _ref()
    traj = sc.simulate(sc.parse_scene(SCENE))
    pr, po = str(tmp_path / "ref.obj"), str(tmp_path / "ours.obj")
    sc.export_obj(pr, traj, 7)
    ours.export_obj(po, _as_ours(traj), 7)
    assert open(po, "rb").read() == open(pr, "rb").read()
    with pytest.raises(ValueError) as r:
        sc.export_obj(pr, traj, 99)
    with pytest.raises(ValueError) as o:
        ours.export_obj(po, _as_ours(traj), 99)
    assert str(o.value) == str(r.value)


def test_eval_csv_format(tmp_path):
    rep = ours.EvalReport("s", "c", [0.0, 0.1, 1.0 / 3], 0.14444444444444446, 1.0 / 3)
    p = str(tmp_path / "e.csv")
    ours.write_eval_csv(p, rep)
    assert open(p).read() == ("scene,s\ncheckpoint,c\nframe,error_pct\n0,0\n1,0.10000000000000001\n"
                              "2,0.33333333333333331\nmean,0.14444444444444446\n"
                              "final,0.33333333333333331\n")


def test_evaluate_validation_matches_reference():
    sc = _ref()
    scene = sc.parse_scene(SCENE)
    a = sc.simulate(scene)
    ta = _as_ours(a)
    other = _random_traj(nx=9, ny=6, frames=3)
    flat = ours.Trajectory(9, 6, ta.dt, ta.spacing, np.zeros_like(ta.frames_x), ta.frames_v)
    small = _random_traj(nx=3, ny=3, frames=ta.frame_count)
    for ours_args, ref_make in [
        ((ta, small), None), ((ta, other), None), ((ta, flat), None)]:
        with pytest.raises(Exception) as e:
            ours.evaluate(*ours_args)
        assert isinstance(e.value, (ValueError, ArithmeticError))
    with pytest.raises(ValueError, match="^evaluate: trajectories have different grid shapes$"):
        ours.evaluate(ta, small)
    with pytest.raises(ValueError, match=r"^evaluate: trajectories have different frame counts "
                                         r"\(13 vs 3\)$"):
        ours.evaluate(ta, other)
    with pytest.raises(ArithmeticError,
                       match="^evaluate: reference frame 0 has a degenerate bounding box$"):
        ours.evaluate(ta, flat)
    # the reference raises the same texts for the same pairs
    with pytest.raises(ValueError, match="^evaluate: trajectories have different frame counts "
                                         r"\(13 vs 14\)$"):
        sc.evaluate(a, sc.simulate(sc.parse_scene(SCENE.replace('"steps": 12', '"steps": 13'))))
