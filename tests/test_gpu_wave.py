"""The wavefront temporal-blocking FAST kernel (csrc/wave_kernels.cu) against one streaming
launch per step (csrc/fast_kernels.cu): the same row pass and finish per timestep, so every
rollout must be bit-identical whatever the batch split, pass length or level count; and one
launch must cover the whole advance (the reference's per-step loop, eval.cpp:48-59)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _wave_at_any_batch(monkeypatch):
    """These tests exercise the wavefront kernel itself: take it whatever the batch size (the
    default prefers chunked streaming below 8 cloths per SM, capi.cu wave_preferred)."""
    monkeypatch.setenv("SC_WAVE_MIN_CLOTHS", "1")
    monkeypatch.setenv("SC_WAVE_MIN_STEPS", "1")  # ... and whatever the step count


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


CASES = [
    (5, 128, 300, 37),  # 2-3 cloths per CTA, all three boundary classes, a short last pass
    (5, 128, 148, 24),  # one cloth per CTA
    (5, 64, 40, 13),    # fewer cloths than SMs, half-width strips (lanes 16..31 idle)
    (2, 128, 20, 50),   # top-row pins + wind
    (3, 128, 3, 30),    # sphere collider, corner pins
    (1, 32, 1, 40),     # config 1: 32 x 32, one cloth
    (5, 128, 12, 1),    # a single step (streaming path either way)
]


@pytest.mark.parametrize("cfg_id,n,batch,steps", CASES)
def test_wave_matches_per_step_launches(monkeypatch, cfg_id, n, batch, steps):
    from paper_2403_12820_b200 import ClothBatch, configs
    monkeypatch.setenv("SC_SMALL", "0")  # config 1's 32^2 cloth: the wavefront kernel, not small
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=batch, n=n)
    with ClothBatch(scenes, p) as cb:
        cb.set_persistent(True)
        l0 = cb.launch_count()
        xa, va = cb.rollout(x, v, steps, 0, "fast")
        la = cb.launch_count() - l0
        cb.set_persistent(False)
        l0 = cb.launch_count()
        xb, vb = cb.rollout(x, v, steps, 0, "fast")
        lb = cb.launch_count() - l0
        # continuing time (k0 offsets) through the wave kernel
        cb.set_persistent(True)
        x1, v1 = cb.rollout(x, v, steps // 2, 0, "fast")
        x2, v2 = cb.rollout(x1, v1, steps - steps // 2, steps // 2, "fast")
    assert bits_equal(xa, xb) and bits_equal(va, vb)
    assert bits_equal(x2, xb) and bits_equal(v2, vb)
    assert lb >= steps
    if steps >= 2 and cfg_id != 5:
        assert la <= 3  # layout in + one wavefront launch + layout out
    assert la <= lb


@pytest.mark.parametrize("levels", ["8", "12", "16"])
def test_wave_level_counts_bit_identical(levels):
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(5, batch=200, n=128)
    old = os.environ.get("SC_WAVE_LEVELS")
    os.environ["SC_WAVE_LEVELS"] = levels
    try:
        with ClothBatch(scenes, p) as cb:
            xa, va = cb.rollout(x, v, 29, 3, "fast")
    finally:
        if old is None:
            del os.environ["SC_WAVE_LEVELS"]
        else:
            os.environ["SC_WAVE_LEVELS"] = old
    with ClothBatch(scenes, p) as cb:
        cb.set_persistent(False)
        xb, vb = cb.rollout(x, v, 29, 3, "fast")
    assert bits_equal(xa, xb) and bits_equal(va, vb)


def test_wave_mask_on_last_step():
    """A rollout asking for the contact mask runs all but the last step in the wave kernel and
    the mask-producing last step in the streaming kernel: same state and mask as per-step."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(5, batch=150, n=128)
    with ClothBatch(scenes, p) as cb:
        xa, va, ma = cb.rollout(x, v, 40, 0, "fast", constrained=True)
        cb.set_persistent(False)
        xb, vb, mb = cb.rollout(x, v, 40, 0, "fast", constrained=True)
    assert bits_equal(xa, xb) and bits_equal(va, vb) and np.array_equal(ma, mb)
    assert ma.any()  # plane contacts and pins really happened


def test_wave_health_matches_streaming():
    """Non-finite inputs in a few cloths: the first non-finite impulse (step, node) and state
    frame per cloth are the same as with per-step launches (net.cpp:139-140, eval.cpp:98-99),
    and the cloths next to them in the kernel's row stream stay finite (the zero tail rows
    separate cloths)."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(5, batch=160, n=128)
    x[7, 128 * 60 + 5, 2] = np.inf
    v[30, 128 * 127 + 64, 0] = np.nan
    v[31, 0, 1] = np.nan
    res, states = [], []
    for persistent in (True, False):
        with ClothBatch(scenes, p) as cb:
            cb.set_persistent(persistent)
            cb.set_health_checks(True)
            cb.set_state(x, v)
            cb.advance(40, 0, "fast")
            res.append(cb.health())
            states.append(cb.get_state())
    for a, b in zip(res[0], res[1]):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    bad = np.nonzero(np.asarray(res[0][2]) >= 0)[0].tolist()
    assert bad == [7, 30, 31], bad
    xs, vs = states[0]
    good = [b for b in range(160) if b not in (7, 30, 31)]
    assert np.isfinite(xs[good]).all() and np.isfinite(vs[good]).all()


def test_wave_class_groups_bit_identical(monkeypatch):
    """A batch mixing collider-free and collider cloths runs as two class groups (collider-free
    cloths in the wavefront kernel, plane / sphere cloths in the streaming kernel); grouped,
    ungrouped (SC_GROUP=0: one wavefront launch with the collider finish) and per-step streaming
    give the same bits, odd and even step counts."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(5, batch=301, n=128)
    out = {}
    for group, persistent in (("1", True), ("0", True), ("1", False)):
        monkeypatch.setenv("SC_GROUP", group)
        with ClothBatch(scenes, p) as cb:
            cb.set_persistent(persistent)
            out[(group, persistent)] = [cb.rollout(x, v, s, 2, "fast") for s in (17, 24)]
    ref = out[("1", False)]
    for key, res in out.items():
        for (xa, va), (xb, vb) in zip(res, ref):
            assert bits_equal(xa, xb) and bits_equal(va, vb), key
