"""GPU side of §8(f3)/(f4): evaluate()'s device sums against the reference's own evaluate_rollout
(stencilcloth module in oracle/_ref) and against an exactly-rounded host sum at size; frame
streaming (pinned direct / pageable staged) against step-by-step stepping; batched rollout to
CLT1 and back."""
import math
import os
import sys

import numpy as np
import pytest

import paper_2403_12820_b200 as ours
from paper_2403_12820_b200 import configs

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "oracle", "_ref")
EVAL_RTOL = 1e-12  # node-sum order differs from the reference's left-to-right loop

SCENE = """
{
  "name": "eval_sheet",
  "grid": {"nx": 17, "ny": 13, "spacing": 0.04, "origin": [-0.32, -0.24, 0.3], "plane": "xy"},
  "material": {"stiffness": %s, "damping": 0.05, "mass": 0.01, "gravity": [0.0, 0.0, -9.8],
               "drag": 0.02, "pressure": 0.3},
  "time": {"dt": 0.001, "steps": 40},
  "pins": {"nodes": ["top_left", "top_right"]},
  "colliders": [{"type": "sphere", "center": [0.0, 0.0, 0.0], "radius": 0.25, "friction": 0.4}]
}
"""


def _ref():
    if not os.path.isdir(os.path.join(REF_PKG, "stencilcloth")):
        pytest.skip("reference module not built")
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    import stencilcloth as sc
    return sc


def _as_ours(t):
    return ours.Trajectory(t.nx, t.ny, t.dt, t.spacing,
                           np.stack([t.positions(f) for f in range(t.frame_count)]),
                           np.stack([t.velocities(f) for f in range(t.frame_count)]))


def test_evaluate_matches_reference():
    sc = _ref()
    a = sc.simulate(sc.parse_scene(SCENE % "30.0"))
    b = sc.simulate(sc.parse_scene(SCENE % "45.0"))
    ref = sc.evaluate(a, b)
    mine = ours.evaluate(_as_ours(a), _as_ours(b))
    r = np.array(ref.frame_error_pct)
    m = np.array(mine.frame_error_pct)
    assert m.shape == r.shape and r[-1] > 0
    np.testing.assert_allclose(m, r, rtol=EVAL_RTOL, atol=0)
    assert abs(mine.mean_error_pct - ref.mean_error_pct) <= EVAL_RTOL * ref.mean_error_pct
    assert abs(mine.final_error_pct - ref.final_error_pct) <= EVAL_RTOL * ref.final_error_pct
    same = ours.evaluate(_as_ours(a), _as_ours(a))
    assert same.frame_error_pct == [0.0] * a.frame_count


def test_evaluate_large_exact_sum_and_deterministic():
    rng = np.random.default_rng(11)
    nx = ny = 512
    n = nx * ny
    frames = 5
    ref_x = rng.normal(0.0, 1.0, (frames, n, 3))
    test_x = ref_x + rng.normal(0.0, 1e-3, ref_x.shape) * np.arange(frames)[:, None, None]
    v = np.zeros_like(ref_x)
    A = ours.Trajectory(nx, ny, 1e-3, 0.01, test_x, v)
    B = ours.Trajectory(nx, ny, 1e-3, 0.01, ref_x, v)
    rep = ours.evaluate(A, B)
    rep2 = ours.evaluate(A, B)
    assert rep.frame_error_pct == rep2.frame_error_pct  # fixed reduction order
    d = test_x - ref_x
    norms = np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])
    diag = ours.trajio.bbox_diagonal(ref_x[0])
    for f in range(frames):
        exact = 100.0 * math.fsum(norms[f].tolist()) / (float(n) * diag)
        got = rep.frame_error_pct[f]
        assert abs(got - exact) <= EVAL_RTOL * max(exact, 1e-300), (f, got, exact)


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_rollout_frames_streaming(mode):
    cfg, scenes, params, x, v = configs.build(2, batch=3, n=64)
    steps, stride = 12, 4
    with ours.ClothBatch(scenes, params) as ctx:
        fx, fv = ctx.rollout_frames(x, v, steps, stride, mode)  # pageable: staged slots
        shape = fx.shape
        px, pv = ours.pinned_empty(shape, np.float32), ours.pinned_empty(shape, np.float32)
        ctx.rollout_frames(x, v, steps, stride, mode, out=(px, pv))  # pinned: direct D2H
        assert np.array_equal(px, fx) and np.array_equal(pv, fv)
        assert np.array_equal(fx[0], x) and np.array_equal(fv[0], v)
        xs, vs = x, v
        for f in range(1, steps // stride + 1):
            xs, vs = ctx.rollout(xs, vs, stride, (f - 1) * stride, mode)
            assert np.array_equal(fx[f], xs) and np.array_equal(fv[f], vs), f
        # trailing partial chunk: stepped, not stored
        gx, _ = ctx.rollout_frames(x, v, steps + 2, stride, mode)
        assert gx.shape[0] == steps // stride + 1 and np.array_equal(gx, fx)


def test_batched_rollout_to_clt1(tmp_path):
    cfg, scenes, params, x, v = configs.build(2, batch=2, n=32)
    with ours.ClothBatch(scenes, params) as ctx:
        trajs = ctx.rollout_trajectories(10, 2, "fast")
    assert len(trajs) == 2 and trajs[0].frame_count == 6
    for k, t in enumerate(trajs):
        p = str(tmp_path / ("c%d.clt1" % k))
        ours.save_trajectory(p, t, 2)
        u = ours.load_trajectory(p)
        np.testing.assert_array_equal(u.frames_x, t.frames_x)  # f32 values survive v2 exactly
        assert ours.evaluate(u, t).final_error_pct == 0.0
    rep = ours.evaluate(trajs[0], trajs[1])
    assert rep.final_error_pct > 0.0
