"""CKP1 checkpoints and the loss CSV (io.cpp:495-606): byte-identical to the reference's writer,
readable by its reader and vice versa, same reader errors. CPU only (the reference module in
oracle/_ref is the checker)."""
import os
import struct
import sys

import numpy as np
import pytest

import paper_2403_12820_b200 as ours

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "oracle", "_ref")

SCENE = """
{
  "name": "ckp_sheet",
  "grid": {"nx": 8, "ny": 6, "spacing": 0.05, "origin": [-0.2, -0.12, 0.3], "plane": "xy"},
  "material": {"stiffness": 30.0, "damping": 0.05, "mass": 0.01, "gravity": [0.0, 0.0, -9.8],
               "drag": 0.02, "pressure": 0.0},
  "time": {"dt": 0.001, "steps": 24},
  "pins": {"nodes": ["top_left", "top_right"]}
}
"""


def _ref():
    if not os.path.isdir(os.path.join(REF_PKG, "stencilcloth")):
        pytest.skip("reference module not built")
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    import stencilcloth as sc
    return sc


@pytest.fixture(scope="module")
def trained():
    sc = _ref()
    scene = sc.parse_scene(SCENE)
    traj = sc.simulate(scene)
    params, hist = sc.train(scene, traj, alpha=0.5, batch_size=4, epochs=3, seed=2,
                            de_population=4, de_generations=1, de_probe=3)
    return sc, params, hist


def test_reference_checkpoint_roundtrip_bytes(tmp_path, trained):
    sc, params, _ = trained
    ck = sc.Checkpoint()
    ck.params = params
    ck.step = 1234
    ck.config_echo = '{"alpha": 0.5, "note": "echo"}'
    pr, po = str(tmp_path / "ref.ckpt"), str(tmp_path / "ours.ckpt")
    sc.save_checkpoint(pr, ck)
    mine = ours.load_checkpoint(pr)
    assert mine.step == 1234 and mine.config_echo == ck.config_echo and mine.opt is None
    assert mine.params.scalars() == list(params.scalars())
    assert mine.params.trainable == [False, True, True, True, True, True, False]
    assert mine.params.fingerprint == params.fingerprint
    ours.save_checkpoint(po, mine)
    assert open(po, "rb").read() == open(pr, "rb").read()
    back = sc.load_checkpoint(po)
    assert list(back.params.scalars()) == mine.params.scalars() and back.step == 1234


def test_optimizer_state_roundtrip(tmp_path, trained):
    sc, params, _ = trained
    p = ours.NetworkParams.from_scalars(list(params.scalars()))
    p.brackets = [(-0.5 - g, 0.25 * g) for g in range(7)]
    opt = ours.AdamState(np.linspace(-1, 1, 53), np.linspace(0, 2, 53), 77)
    path = str(tmp_path / "opt.ckpt")
    ours.save_checkpoint(path, ours.Checkpoint(p, opt, 9, "x"))
    u = ours.load_checkpoint(path)
    assert u.params.brackets == p.brackets and u.opt.step == 77
    assert np.array_equal(u.opt.m, opt.m) and np.array_equal(u.opt.v, opt.v)
    ref = sc.load_checkpoint(path)  # the reference reader accepts the optimizer block
    assert list(ref.params.scalars()) == p.scalars() and ref.step == 9


def _good_bytes(tmp_path):
    p = ours.NetworkParams()
    path = str(tmp_path / "good.ckpt")
    ours.save_checkpoint(path, ours.Checkpoint(p, None, 3, "abc"))
    return open(path, "rb").read()


def _cases(good):
    hdr = 4 + 4 + 8 + 8 + 4 + 3  # magic, version, hash, step, echo len, echo
    g0 = hdr + 4                  # first group record
    return {
        "bad_magic": b"CKPX" + good[4:],
        "version2": good[:4] + struct.pack("<I", 2) + good[8:],
        "hash": good[:8] + struct.pack("<Q", 12345) + good[16:],
        "echo_huge": good[:24] + struct.pack("<I", (1 << 20) + 1) + good[28:],
        "groups6": good[:hdr] + struct.pack("<I", 6) + good[hdr + 4:],
        "group_name": good[:g0 + 1] + b"x" + good[g0 + 2:],
        "group_count": good[:g0 + 1 + 6 + 1 + 16] + struct.pack("<I", 11) + good[g0 + 1 + 6 + 1 + 20:],
        "truncated": good[:-1],
        "header_only": good[:10],
        "empty": b"",
    }


@pytest.mark.parametrize("case", ["bad_magic", "version2", "hash", "echo_huge", "groups6",
                                  "group_name", "group_count", "truncated", "header_only", "empty"])
def test_reader_errors_match_reference(tmp_path, case):
    sc = _ref()
    data = _cases(_good_bytes(tmp_path))[case]
    path = str(tmp_path / (case + ".ckpt"))
    open(path, "wb").write(data)
    with pytest.raises(OSError) as r:
        sc.load_checkpoint(path)
    with pytest.raises(OSError) as o:
        ours.load_checkpoint(path)
    assert str(o.value) == str(r.value)


def test_missing_file_and_alpha(tmp_path):
    with pytest.raises(ours.IoError, match="^cannot open checkpoint /nonexistent/a.ckpt$"):
        ours.load_checkpoint("/nonexistent/a.ckpt")
    p = ours.NetworkParams()
    p.isru_alpha = -1.0
    path = str(tmp_path / "alpha.ckpt")
    ours.save_checkpoint(path, ours.Checkpoint(p))
    with pytest.raises(ours.IoError, match="checkpoint isru_alpha must be > 0$"):
        ours.load_checkpoint(path)


def test_loss_csv_format(tmp_path, trained):
    _, _, hist = trained
    path = str(tmp_path / "loss.csv")
    ours.write_loss_csv(path, hist)
    lines = open(path).read().splitlines()
    assert lines[0] == "step,lr,physics,data,total" and len(lines) == len(hist) + 1
    step, lr, ph, da, to = lines[1].split(",")
    assert int(step) == hist[0][0] and float(lr) == hist[0][1] and float(to) == hist[0][4]
